// k_stage.cu -- K0: strided-box gather from pinned host memory into HBM staging.
//
// Replaces per-sample cudaMemcpy2D/3DAsync DMA (hundreds of short rows per
// sample) on the end-to-end path: one launch per launch group reads exactly
// the bytes the chain needs (img_seg crop window, obj_det crop box) over PCIe
// with aligned 16-byte loads through the UVA mapping of the pinned buffer.
// A row is copied as the 16-B aligned superset of its byte range, so the
// staging copy keeps the source's alignment phase ("skew"); consumers
// re-derive a row's start as base + z*dst_pz + y*dst_py + (src_row_addr & 15).
#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kWarps = 8;
constexpr int kIlp = 4;   // 16-B chunks in flight per lane (all loads issued before the stores)

// The aligned 16-B chunk at `a` (chunk address) of a row spanning [lo, hi): only the
// bytes inside the range are read (byte loads), the rest of the chunk is zero.  Used
// for the box's first and last chunk, which may extend past the caller's allocation
// (aligned chunks never cross a page, but the bytes outside belong to no allocation).
__device__ __forceinline__ int4 load_chunk_exact(uintptr_t a, uintptr_t lo, uintptr_t hi) {
    // whole 4-B words inside the range by word loads, the rest byte by byte; all loads
    // independent, so a PCIe round trip is paid once, not per byte
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uintptr_t x = a + 4 * q;
        if (x >= lo && x + 4 <= hi) {
            w[q] = *reinterpret_cast<const uint32_t*>(x);
        } else {
            uint32_t v = 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (x + b >= lo && x + b < hi) v |= uint32_t(*reinterpret_cast<const uint8_t*>(x + b)) << (8 * b);
            w[q] = v;
        }
    }
    return make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
}

// The box's 16-B chunks are one flat index space (row-major, nch_max chunks per
// row, the padded staging pitch): consecutive lanes take consecutive chunks, so
// short rows (the 144-B label rows of a crop window) do not idle most of a warp,
// and every lane keeps kIlp PCIe reads in flight.
__global__ void __launch_bounds__(32 * kWarps) stage_kernel(const __grid_constant__ StageLaunch L) {
    const StageDesc& d = L.d[blockIdx.y];
    const int nch_max = (d.row_bytes + 30) >> 4;     // chunks of the aligned superset, upper bound
    const int64_t rows = (int64_t)d.ny * d.nz;
    const int64_t total = rows * nch_max;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kIlp;
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x) * kIlp + threadIdx.x; base < total; base += stride) {
        int4 v[kIlp];
        int4* dst[kIlp];
#pragma unroll
        for (int k = 0; k < kIlp; ++k) {
            dst[k] = nullptr;
            const int64_t item = base + (int64_t)k * blockDim.x;
            if (item >= total) continue;
            const int64_t r = item / nch_max;
            const int c = (int)(item - r * nch_max);
            const int64_t z = r / d.ny, y = r - z * d.ny;
            const uintptr_t s = reinterpret_cast<uintptr_t>(d.src) + z * d.src_pz + y * d.src_py;
            const uintptr_t a = s & ~uintptr_t(15);
            const int nch = (int)((((s + d.row_bytes + 15) & ~uintptr_t(15)) - a) >> 4);
            if (c >= nch) continue;
            // the box's first and last chunk: only the box's own bytes are read
            const bool edge = (r == 0 && c == 0) || (r == rows - 1 && c == nch - 1);
            v[k] = edge ? load_chunk_exact(a + 16 * (uintptr_t)c, s, s + d.row_bytes)
                        : reinterpret_cast<const int4*>(a)[c];
            dst[k] = reinterpret_cast<int4*>(d.dst + z * d.dst_pz + y * d.dst_py) + c;
        }
#pragma unroll
        for (int k = 0; k < kIlp; ++k)
            if (dst[k] != nullptr) *dst[k] = v[k];
    }
}

// Bulk variant: one thread per warp moves whole rows with the TMA engine --
// cp.async.bulk host->smem (the aligned superset of the row), then smem->HBM --
// keeping kBulkDepth rows in flight per warp (ring of smem buffers).
constexpr int kBulkDepth = 8;
constexpr int kBulkBuf = 1600;     // bytes per ring slot (rows longer than this use stage_kernel)

__global__ void __launch_bounds__(32 * kWarps) stage_bulk_kernel(const __grid_constant__ StageLaunch L) {
    extern __shared__ __align__(128) uint8_t sbuf[];
    __shared__ __align__(8) uint64_t bars[kWarps][kBulkDepth];
    const StageDesc& d = L.d[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t rows = (int64_t)d.ny * d.nz;
    if (blockIdx.x == 0 && warp == 0) {
        // the box's first and last row by lanes, their end chunks read exactly (a bulk
        // copy of the aligned superset could read bytes outside the caller's buffer)
        for (int e = 0; e < (rows > 1 ? 2 : 1); ++e) {
            const int64_t r = e == 0 ? 0 : rows - 1;
            const int64_t z = r / d.ny, y = r - z * d.ny;
            const uintptr_t s = reinterpret_cast<uintptr_t>(d.src) + z * d.src_pz + y * d.src_py;
            const uintptr_t a = s & ~uintptr_t(15);
            const int nch = (int)((((s + d.row_bytes + 15) & ~uintptr_t(15)) - a) >> 4);
            int4* out = reinterpret_cast<int4*>(d.dst + z * d.dst_pz + y * d.dst_py);
            for (int c = lane; c < nch; c += 32)
                out[c] = (c == 0 || c == nch - 1) ? load_chunk_exact(a + 16 * (uintptr_t)c, s, s + d.row_bytes)
                                                  : reinterpret_cast<const int4*>(a)[c];
        }
    }
    if (lane != 0) return;
    uint8_t* ring = sbuf + warp * kBulkDepth * kBulkBuf;
    for (int k = 0; k < kBulkDepth; ++k) mbar_init(&bars[warp][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // bulk rows: 1 .. rows - 2 (row index 1 + i)
    const int64_t nbulk = rows > 2 ? rows - 2 : 0;
    const int64_t first = (int64_t)blockIdx.x * kWarps + warp, step = (int64_t)gridDim.x * kWarps;
    const int64_t mine = first < nbulk ? (nbulk - first + step - 1) / step : 0;
    int64_t use[kBulkDepth] = {};
    auto row_src = [&](int64_t i, uint32_t& nb) {
        const int64_t r = 1 + i;
        const int64_t z = r / d.ny, y = r - z * d.ny;
        const uintptr_t s = reinterpret_cast<uintptr_t>(d.src) + z * d.src_pz + y * d.src_py;
        const uintptr_t a = s & ~uintptr_t(15);
        nb = (uint32_t)(((s + d.row_bytes + 15) & ~uintptr_t(15)) - a);
        return a;
    };
    auto row_dst = [&](int64_t i) {
        const int64_t r = 1 + i;
        const int64_t z = r / d.ny, y = r - z * d.ny;
        return d.dst + z * d.dst_pz + y * d.dst_py;
    };
    for (int64_t k = 0; k < mine + kBulkDepth - 1; ++k) {
        if (k < mine) {
            const int b = (int)(k % kBulkDepth);
            // the slot's previous row (k - depth) must have been read out by its store
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBulkDepth - 1) : "memory");
            uint32_t nb;
            const uintptr_t a = row_src(first + k * step, nb);
            mbar_expect_tx(&bars[warp][b], nb);
            bulk_g2s(ring + b * kBulkBuf, reinterpret_cast<const void*>(a), nb, &bars[warp][b]);
        }
        const int64_t j = k - (kBulkDepth - 1);
        if (j >= 0) {
            const int b = (int)(j % kBulkDepth);
            mbar_wait(&bars[warp][b], (uint32_t)(use[b] & 1));
            ++use[b];
            uint32_t nb;
            (void)row_src(first + j * step, nb);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(row_dst(first + j * step)),
                         "r"(smem_u32(ring + b * kBulkBuf)), "r"(nb)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// K0w: one CTA per (window plane z, sample); a warp per window row.  Image rows
// come from host memory as 16-B aligned chunks (lane l holds chunk q0 + l, lane
// 31 also the next group's first chunk) and are realigned to the window's first
// float with a shuffle; label rows come from the staged volume in HBM.
__device__ __forceinline__ float4 shift4w(float4 a, float4 b, int m) {
    switch (m) {   // warp-uniform
        case 0: return a;
        case 1: return make_float4(a.y, a.z, a.w, b.x);
        case 2: return make_float4(a.z, a.w, b.x, b.y);
        default: return make_float4(a.w, b.x, b.y, b.z);
    }
}

__global__ void __launch_bounds__(32 * kWarps) stage_window_kernel(const __grid_constant__ WindowLaunch L) {
    const WindowDesc& d = L.d[blockIdx.y];
    const int z = blockIdx.x;
    if (z >= d.win[0]) return;
    const int4 o = L.offs[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = d.dims[0], H = d.dims[1], W = d.dims[2];
    const int sz = o.x + z;
    const int w2 = d.win[2];
    const int vw = max(0, min(w2, W - o.z));            // window columns inside the volume
    const int nq = (w2 + 3) >> 2;                         // output quads per row
    for (int y = warp; y < d.win[1]; y += kWarps) {
        const int sy = o.y + y;
        float4* out = reinterpret_cast<float4*>(d.dst_img + ((int64_t)z * d.win[1] + y) * d.img_pitch);
        uint8_t* lout = d.dst_lbl + ((int64_t)z * d.win[1] + y) * d.lbl_pitch;
        const bool row_ok = sz < D && sy < H && vw > 0;
        if (!row_ok) {
            for (int q = lane; q < nq; q += 32) out[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int x = lane; x < w2; x += 32) lout[x] = 0;
            continue;
        }
        const float* a = d.img_host + ((int64_t)sz * H + sy) * W + o.z;   // first window float
        const uintptr_t ab = reinterpret_cast<uintptr_t>(a);
        const int m = (int)((ab & 15) >> 2);                               // warp-uniform
        const float4* c0 = reinterpret_cast<const float4*>(ab & ~uintptr_t(15));
        const int nch = (m + vw + 3) >> 2;                                 // chunks holding window data
        // the volume's first and last rows: end chunks read exactly (the aligned chunk
        // may reach outside the caller's buffer); other rows' overreads stay inside it
        const bool vol_edge = (sz == 0 && sy == 0) || (sz == D - 1 && sy == H - 1);
        const uintptr_t row_lo = reinterpret_cast<uintptr_t>(d.img_host + ((int64_t)sz * H + sy) * W);
        const uintptr_t row_hi = row_lo + uintptr_t(4) * W;
        auto chunk = [&](int c) {
            const uintptr_t ca = reinterpret_cast<uintptr_t>(c0 + c);
            if (vol_edge && (ca < row_lo || ca + 16 > row_hi)) {
                const int4 w = load_chunk_exact(ca, row_lo, row_hi);
                return make_float4(__int_as_float(w.x), __int_as_float(w.y), __int_as_float(w.z), __int_as_float(w.w));
            }
            return c0[c];
        };
        for (int q0 = 0; q0 < nq; q0 += 32) {
            const int c = q0 + lane;
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 v = c < nch ? chunk(c) : zero;
            float4 nx = make_float4(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1),
                                    __shfl_down_sync(0xffffffffu, v.z, 1), __shfl_down_sync(0xffffffffu, v.w, 1));
            if (lane == 31) nx = (q0 + 32 < nch) ? chunk(q0 + 32) : zero;
            if (c < nq) {
                float4 x = shift4w(v, nx, m);
                const int keep = vw - 4 * c;                                // valid floats of this quad
                if (keep < 4) x.w = 0.f;
                if (keep < 3) x.z = 0.f;
                if (keep < 2) x.y = 0.f;
                if (keep < 1) x.x = 0.f;
                out[c] = x;
            }
        }
        const uint8_t* lrow = d.lbl + (int64_t)sz * d.lbl_pz + (int64_t)sy * d.lbl_py +
                              ((d.lbl_sk0 + sz * d.lbl_skz + sy * d.lbl_sky) & 15) + o.z;
        for (int x = lane; x < w2; x += 32) lout[x] = x < vw ? lrow[x] : (uint8_t)0;
    }
}

}  // namespace

cudaError_t launch_stage_window(const WindowLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    int planes = 1;
    for (int i = 0; i < L.n; ++i) {
        if ((L.d[i].img_pitch & 3) || (L.d[i].lbl_pitch & 15) || L.d[i].img_pitch < L.d[i].win[2] ||
            L.d[i].lbl_pitch < L.d[i].win[2])
            return cudaErrorInvalidValue;
        planes = planes > L.d[i].win[0] ? planes : L.d[i].win[0];
    }
    stage_window_kernel<<<dim3(planes, L.n), 32 * kWarps, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_stage(const StageLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    int64_t max_chunks = 0;
    for (int i = 0; i < L.n; ++i) {
        const int64_t c = (int64_t)L.d[i].ny * L.d[i].nz * ((L.d[i].row_bytes + 30) >> 4);
        if (c > max_chunks) max_chunks = c;
    }
    const int64_t per_cta = 32 * kWarps * kIlp;
    int64_t g = (max_chunks + per_cta - 1) / per_cta;
    int gx = (int)(g > 4096 ? 4096 : g);
    if (gx < 1) gx = 1;
    // Row-wise bulk copies win on long rows (obj_det crop boxes: +6% PCIe rate), the
    // flat chunk kernel on short ones (img_seg window rows of 512 + 128 B)
    static const int bulk_env = getenv("LFG_STAGE_BULK") ? atoi(getenv("LFG_STAGE_BULK")) : -1;
    bool fits = true;
    int64_t max_rows = 0, rows_all = 0, bytes_all = 0;
    for (int i = 0; i < L.n; ++i) {
        const int64_t r = (int64_t)L.d[i].ny * L.d[i].nz;
        fits = fits && L.d[i].row_bytes + 32 <= kBulkBuf;
        max_rows = max_rows > r ? max_rows : r;
        rows_all += r;
        bytes_all += r * L.d[i].row_bytes;
    }
    const bool bulk = bulk_env >= 0 ? bulk_env != 0 : bytes_all >= 640 * rows_all;
    if (bulk && fits) {
        int64_t gb = (max_rows + kWarps * 4 - 1) / (kWarps * 4);   // ~4 rows per issuing thread
        int gxb = (int)(gb > 4096 ? 4096 : (gb < 1 ? 1 : gb));
        stage_bulk_kernel<<<dim3(gxb, L.n), 32 * kWarps, kWarps * kBulkDepth * kBulkBuf, s>>>(L);
        return cudaGetLastError();
    }
    stage_kernel<<<dim3(gx, L.n), 32 * kWarps, 0, s>>>(L);
    return cudaGetLastError();
}

}  // namespace lfg

namespace lfg {
// Runs on every Context's device at creation (the shared-memory limit is a
// per-device kernel attribute).
cudaError_t warm_stage() {
    cudaError_t e = cudaFuncSetAttribute(stage_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kWarps * kBulkDepth * kBulkBuf);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, stage_kernel);
}
}  // namespace lfg
