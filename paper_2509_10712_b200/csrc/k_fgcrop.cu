// k_fgcrop.cu -- K2: RandomCrop's foreground oversampling (MLPerf 3D-UNet
// RandBalancedCrop; RandomCrop carries the img_seg chain's 68% cost share,
// proj/src/workloads.cpp:149).  Semantics: oracle/lf_oracle.c lfo_fg_offsets.
//
// fg_scan_kernel: one CTA per (label plane, scanned sample); warps walk rows,
// lanes 16-byte chunks (all-background chunks cost one compare), and keep the
// per-class (labels 1..7) x / y extents in registers; warp min/max reductions
// (redux.sync), shared-memory atomics per CTA, then one global atomicMin /
// atomicMax per class and bound.  HBM-bound: the whole label volume is read
// once (D*H*W bytes) -- the genuinely heavy step that makes foreground-biased
// samples the slow tail.
//
// fg_offsets_kernel: one thread per sample of the launch group turns the class
// boxes and the sample's host-drawn uniforms into the window origin, exactly as
// the oracle (fp64 floor of u * span), or marks it "random offsets hold".
#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kScanThreads = 256;
constexpr int kClasses = 8;   // index = label value; 1..7 are foreground classes
constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ void note(int v, uint32_t x, uint32_t xmin[kClasses], uint32_t xmax[kClasses],
                                     uint32_t& seen) {
#pragma unroll
    for (int c = 1; c < kClasses; ++c) {
        if (v == c) {
            xmin[c] = min(xmin[c], x);
            xmax[c] = (xmax[c] == kNone) ? x : max(xmax[c], x);
            seen |= 1u << c;
        }
    }
}

// bytes of q equal to the byte replicated in rep, as a 16-bit mask (byte k -> bit k):
// per word, the match bytes' low bits (0, 8, 16, 24) times 0x10204080 land on bits
// 28..31 with no carries
__device__ __forceinline__ uint32_t byte_mask16(const uint4 q, uint32_t rep) {
    const uint32_t m0 = (__vcmpeq4(q.x, rep) & 0x01010101u) * 0x10204080u;
    const uint32_t m1 = (__vcmpeq4(q.y, rep) & 0x01010101u) * 0x10204080u;
    const uint32_t m2 = (__vcmpeq4(q.z, rep) & 0x01010101u) * 0x10204080u;
    const uint32_t m3 = (__vcmpeq4(q.w, rep) & 0x01010101u) * 0x10204080u;
    return (m0 >> 28) | ((m1 >> 24) & 0xF0u) | ((m2 >> 20) & 0xF00u) | ((m3 >> 16) & 0xF000u);
}

__global__ void __launch_bounds__(kScanThreads) fg_scan_kernel(const __grid_constant__ Img3dLaunch L,
                                                               const __grid_constant__ FgLaunch F,
                                                               int32_t* __restrict__ box) {
    int k = 0;
    while (k + 1 < F.n_scan && (int)blockIdx.x >= F.scan_start[k + 1]) ++k;
    const int i = F.scan_i[k];
    const Img3dDesc& d = L.d[i];
    const int z = (int)blockIdx.x - F.scan_start[k];
    __shared__ uint32_t s_min[kClasses][3], s_max[kClasses][3];
    __shared__ uint32_t s_seen;
    if (threadIdx.x < kClasses * 3) {
        (&s_min[0][0])[threadIdx.x] = kNone;
        (&s_max[0][0])[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) s_seen = 0;
    __syncthreads();
    const int H = d.sdim[1], W = d.sdim[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per lane: the class x extents of its chunks; the y extents are warp-uniform per
    // row, so lane c keeps class c's (ylo, yhi + 1) for the whole warp (2 registers, not 14)
    uint32_t xmin[kClasses], xmax[kClasses];
#pragma unroll
    for (int c = 0; c < kClasses; ++c) xmin[c] = xmax[c] = kNone;
    uint32_t ylo = kNone, yhi1 = 0;
    uint32_t acc[(kClasses) / 2] = {0u, 0u, 0u, 0u};   // (row-vector path) per-class byte masks, 2 per word
    uint32_t seen_all = 0;
    // one 16-B chunk of a label row against the per-class extents
    auto chunk = [&](const uint4 v, int q, uint32_t& seen) {
        if ((v.x | v.y | v.z | v.w) == 0u) return;   // background chunk
        const uint32_t b0 = v.x & 0xFFu;
        if (v.x == v.y && v.y == v.z && v.z == v.w && v.x == 0x01010101u * b0) {
            // uniform chunk (inside a region): one class spans all 16 bytes
            if (b0 >= 1 && b0 < (uint32_t)kClasses) {
#pragma unroll
                for (int c = 1; c < kClasses; ++c) {
                    if ((uint32_t)c > b0) break;
                    if (b0 == (uint32_t)c) {
                        xmin[c] = min(xmin[c], (uint32_t)(16 * q));
                        xmax[c] = (xmax[c] == kNone) ? (uint32_t)(16 * q + 15) : max(xmax[c], (uint32_t)(16 * q + 15));
                    }
                }
                seen |= 1u << b0;
            }
            return;
        }
        // per class: SIMD byte compares give the chunk's match mask (one bit per
        // byte), whose lowest / highest set bits are the class's x extent in the chunk;
        // classes above the chunk's largest label are skipped
        uint32_t mx = __vmaxu4(__vmaxu4(v.x, v.y), __vmaxu4(v.z, v.w));
        mx = __vmaxu4(mx, mx >> 16);
        mx = max(mx & 0xFFu, (mx >> 8) & 0xFFu);
#pragma unroll
        for (int c = 1; c < kClasses; ++c) {
            if ((uint32_t)c > mx) break;
            const uint32_t rep = 0x01010101u * (uint32_t)c;
            const uint32_t m[4] = {__vcmpeq4(v.x, rep), __vcmpeq4(v.y, rep), __vcmpeq4(v.z, rep),
                                   __vcmpeq4(v.w, rep)};
            if ((m[0] | m[1] | m[2] | m[3]) == 0u) continue;
            uint32_t bm = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                bm |= ((m[k] & 0x01u) | ((m[k] >> 7) & 0x02u) | ((m[k] >> 14) & 0x04u) | ((m[k] >> 21) & 0x08u))
                      << (4 * k);
            const uint32_t lo = (uint32_t)(16 * q) + (uint32_t)(__ffs(bm) - 1);
            const uint32_t hi = (uint32_t)(16 * q) + (uint32_t)(31 - __clz(bm));
            xmin[c] = min(xmin[c], lo);
            xmax[c] = (xmax[c] == kNone) ? hi : max(xmax[c], hi);
            seen |= 1u << c;
        }
    };
    const uint8_t* plane = d.lbl + (int64_t)z * d.lbl_pz;
    const int zsk = d.lbl_sk0 + z * d.lbl_skz;
    auto row_ptr = [&](int y) {
        // row start (K0-staged volumes keep the source's 16-B alignment phase: skews)
        return plane + (int64_t)y * d.lbl_py + ((zsk + y * d.lbl_sky) & 15);
    };
    // (warp-uniform call: every lane passes its chunks' classes of row y)
    auto close_row = [&](int y, uint32_t seen) {
        const uint32_t w = __reduce_or_sync(0xFFFFFFFFu, seen);
        if (w == 0u) return;   // all-background row (most of a volume)
        if ((w >> lane) & 1u) {
            ylo = min(ylo, (uint32_t)y);
            yhi1 = max(yhi1, (uint32_t)y + 1u);
        }
        seen_all |= seen;
    };
    constexpr int kRowsInFlight = 8;    // rows per warp with their loads issued together
    constexpr int kWarps = kScanThreads / 32;
    const bool vec = (reinterpret_cast<uintptr_t>(row_ptr(0)) & 15) == 0 && (d.lbl_py & 15) == 0 &&
                     (d.lbl_pz & 15) == 0 && (W & 15) == 0 && (d.lbl_sky & 15) == 0;
    if (vec && (W >> 4) <= 32) {
        // rows of <= 512 B: lane q holds the row's 16-B chunk q, kRowsInFlight rows per
        // warp with their loads issued together.  A row's class extents are found at
        // warp level: ballot of the lanes whose chunk holds class c, then the first /
        // last such lane's byte offsets by shuffle -- O(1) warp instructions per class
        // present, no per-lane extent registers (occupancy, bytes in flight).  Lane c
        // keeps class c's x / y extents for the warp.
        const bool lane_live = lane < (W >> 4);
        const int64_t py = d.lbl_py;
        const uint8_t* base = plane + (zsk & 15);   // aligned rows: no per-row skew
        for (int y0 = warp; y0 < H; y0 += kWarps * kRowsInFlight) {
            uint4 v[kRowsInFlight];
#pragma unroll
            for (int r = 0; r < kRowsInFlight; ++r) {
                const int y = y0 + r * kWarps;
                v[r] = (lane_live && y < H) ? __ldcs(reinterpret_cast<const uint4*>(base + (int64_t)y * py) + lane)
                                            : make_uint4(0u, 0u, 0u, 0u);
            }
            // which of the 8 rows hold any foreground byte: one warp OR for all of them,
            // so an all-background batch of rows (most of a volume) costs no per-row work
            uint32_t anym = 0;
#pragma unroll
            for (int r = 0; r < kRowsInFlight; ++r)
                anym |= ((v[r].x | v[r].y | v[r].z | v[r].w) != 0u ? 1u : 0u) << r;
            const uint32_t rows = __reduce_or_sync(0xFFFFFFFFu, anym);
            if (rows == 0u) continue;
#pragma unroll
            for (int r = 0; r < kRowsInFlight; ++r) {
                if (!((rows >> r) & 1u)) continue;   // warp-uniform
                const uint4 q = v[r];
                uint32_t mx = __vmaxu4(__vmaxu4(q.x, q.y), __vmaxu4(q.z, q.w));
                mx = __vmaxu4(mx, mx >> 16);
                mx = max(mx & 0xFFu, (mx >> 8) & 0xFFu);
                const uint32_t top = __reduce_max_sync(0xFFFFFFFFu, mx);
                const uint32_t y = (uint32_t)(y0 + r * kWarps);
#pragma unroll
                for (int c = 1; c < kClasses; ++c) {
                    if ((uint32_t)c > top) break;   // warp-uniform
                    // the chunk's bytes equal to c as a 16-bit mask (byte k -> bit k), OR-ed
                    // into the lane's per-class accumulator; the row's y once per class
                    const uint32_t bm = (uint32_t)c <= mx ? byte_mask16(q, 0x01010101u * (uint32_t)c) : 0u;
                    acc[(c - 1) >> 1] |= bm << (16 * ((c - 1) & 1));
                    if (__any_sync(0xFFFFFFFFu, bm != 0u) && lane == c) {
                        ylo = min(ylo, y);
                        yhi1 = max(yhi1, y + 1u);
                    }
                }
            }
        }
        // x extents: lane q's accumulated byte masks cover bytes 16q .. 16q + 15
#pragma unroll
        for (int c = 1; c < kClasses; ++c) {
            const uint32_t m = (acc[(c - 1) >> 1] >> (16 * ((c - 1) & 1))) & 0xFFFFu;
            if (__ballot_sync(0xFFFFFFFFu, m != 0u) == 0u) continue;   // warp-uniform
            const uint32_t a = __reduce_min_sync(0xFFFFFFFFu, m ? 16u * lane + __ffs(m) - 1u : kNone);
            const uint32_t b = __reduce_max_sync(0xFFFFFFFFu, m ? 16u * lane + 32u - __clz(m) : 0u);
            if (lane == 0) {
                atomicMin(&s_min[c][2], a);
                atomicMax(&s_max[c][2], b);
                atomicOr(&s_seen, 1u << c);
            }
        }
    } else {
        for (int y = warp; y < H; y += kWarps) {
            const uint8_t* row = row_ptr(y);
            uint32_t seen = 0;
            if (vec) {
                for (int q = lane; q < (W >> 4); q += 32) chunk(__ldcs(reinterpret_cast<const uint4*>(row) + q), q, seen);
            } else {
                for (int x = lane; x < W; x += 32) {
                    const int b = row[x];
                    if (b != 0) note(b, (uint32_t)x, xmin, xmax, seen);
                }
            }
            close_row(y, seen);
        }
    }
    // warp reductions (kNone = absent: min ignores it; max treats it as absent via 0-shift)
    seen_all = __reduce_or_sync(0xFFFFFFFFu, seen_all);
#pragma unroll
    for (int c = 1; c < kClasses; ++c) {
        if (!(seen_all & (1u << c))) continue;   // warp-uniform
        const uint32_t a = __reduce_min_sync(0xFFFFFFFFu, xmin[c]);
        const uint32_t b = __reduce_max_sync(0xFFFFFFFFu, xmax[c] == kNone ? 0u : xmax[c] + 1u);
        if (lane == 0) {
            atomicMin(&s_min[c][2], a);
            atomicMax(&s_max[c][2], b);
            atomicOr(&s_seen, 1u << c);
        }
    }
    if (lane >= 1 && lane < kClasses && yhi1 != 0u) {   // lane c: class c's rows
        atomicMin(&s_min[lane][1], ylo);
        atomicMax(&s_max[lane][1], yhi1);
    }
    __syncthreads();
    if (threadIdx.x < kClasses && (s_seen & (1u << threadIdx.x))) {
        const int c = threadIdx.x;
        int32_t* mins = box + (int64_t)i * kClasses * 3;                  // [kMax3D][8][3] mins,
        int32_t* maxs = box + (int64_t)(kMax3D + i) * kClasses * 3;       // then [kMax3D][8][3] maxs
        atomicMin(&mins[c * 3 + 0], z);
        atomicMax(&maxs[c * 3 + 0], z);
        atomicMin(&mins[c * 3 + 1], (int32_t)s_min[c][1]);
        atomicMax(&maxs[c * 3 + 1], (int32_t)s_max[c][1] - 1);
        atomicMin(&mins[c * 3 + 2], (int32_t)s_min[c][2]);
        atomicMax(&maxs[c * 3 + 2], (int32_t)s_max[c][2] - 1);
    }
}

__global__ void fg_offsets_kernel(const __grid_constant__ Img3dLaunch L, const __grid_constant__ FgLaunch F,
                                  const int32_t* __restrict__ box, int4* __restrict__ offs) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L.n) return;
    const Img3dDesc& d = L.d[i];
    const FgDraw& g = F.d[i];
    int4 o = make_int4(d.off[0], d.off[1], d.off[2], 0);
    if (g.fg) {
        const int32_t* mins = box + (int64_t)i * kClasses * 3;
        const int32_t* maxs = box + (int64_t)(kMax3D + i) * kClasses * 3;
        int cls[7], n = 0;
        for (int c = 1; c < kClasses; ++c)
            if (maxs[c * 3] >= 0) cls[n++] = c;
        if (n > 0) {
            int k = (int)floor(g.u_cls * (double)n);
            if (k >= n) k = n - 1;
            const int cl = cls[k];
            int off[3];
            for (int a = 0; a < 3; ++a) {
                const int64_t patch = d.win[a], lo = mins[cl * 3 + a], hi = (int64_t)maxs[cl * 3 + a] + 1;
                const int64_t dim = d.sdim[a];
                int64_t diff = patch - (hi - lo);
                const int64_t sign = diff < 0 ? -1 : 1;
                if (diff < 0) diff = -diff;
                int64_t ladj = diff > 0 ? (int64_t)floor(g.u_adj[a] * (double)diff) : 0;
                if (ladj >= diff && diff > 0) ladj = diff - 1;
                const int64_t hadj = diff - ladj;
                int64_t low = lo - sign * ladj, high = hi + sign * hadj;
                if (low < 0) low = 0;
                if (high > dim) high = dim;
                const int64_t d2 = patch - (high - low);
                if (d2 > 0) {
                    if (low == 0) high += d2;
                    else low -= d2;
                }
                const int64_t room = dim - patch > 0 ? dim - patch : 0;
                off[a] = (int)(low < 0 ? 0 : (low > room ? room : low));
            }
            o = make_int4(off[0], off[1], off[2], 1);
        }
    }
    offs[i] = o;
}

}  // namespace

cudaError_t launch_fg_scan(const Img3dLaunch& L, const FgLaunch& F, int32_t* box, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    FgLaunch G = F;   // one CTA per plane of each scanned sample (no empty CTAs)
    G.n_scan = 0;
    int planes = 0;
    for (int i = 0; i < L.n; ++i) {
        if (!F.d[i].fg) continue;
        G.scan_i[G.n_scan] = i;
        G.scan_start[G.n_scan++] = planes;
        planes += L.d[i].sdim[0];
    }
    G.scan_start[G.n_scan] = planes;
    if (planes == 0) return cudaSuccess;
    fg_scan_kernel<<<planes, kScanThreads, 0, s>>>(L, G, box);
    return cudaGetLastError();
}

cudaError_t launch_fg_offsets(const Img3dLaunch& L, const FgLaunch& F, const int32_t* box, int4* offs,
                              cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    fg_offsets_kernel<<<1, 32, 0, s>>>(L, F, box, offs);
    return cudaGetLastError();
}

}  // namespace lfg
