// k_img3d.cu -- K1: fused img_seg chain for a launch group of volumes.
//
// Realises the reference transforms RandomCrop (0.0735), RandomFlip,
// RandomBrightness, GaussianNoise, Cast (proj/src/workloads.cpp:142-148) in
// one pass: every output voxel is read once and written once.
//
// Algorithmic HBM bytes per sample: read cd*ch*cw*(4+1) + write cd*ch*cw*(4+1)
// (20,971,520 B at 128^3).
//
// Mapping: grid (ceil(ch / 32), cd, n_samples), block (32, 8).  A warp owns an
// output row (lane = 4 consecutive voxels, 32 lanes = 128 voxels) and each
// thread walks 2 rows (y, y+8), issuing all row loads before any
// math.  A row of the crop window starts at an arbitrary element of the source
// row, so each lane loads the two ALIGNED 16-byte image chunks (two aligned
// 4-byte label words) covering its 4 voxels and realigns them with a
// warp-uniform element shift -- 4 load instructions per 4 voxels instead of 8
// scalar ones; RandomFlip along W reverses the quad (and the lane order).
// Image and label stores are 16-B / 4-B streaming stores.  GaussianNoise draws
// one Philox4x32-10 block per 4 output voxels, so noise-on samples are
// ALU-bound; noise-off samples are HBM-bound.
//
// HBM-resident volumes with 16-B aligned rows take the TMA tile path instead
// (img3d_tma_kernel below); the row kernel serves K0-staged windows (skewed
// rows) and unaligned geometries.
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kRowsY = 8;          // threadIdx.y extent
constexpr int kRowsPerThread = 2;  // rows y, y + 8 (4 rows halves the grid: < 1 wave per volume)
constexpr int kRowsPerCta = kRowsY * kRowsPerThread;

// 4 consecutive floats starting m (0..3) elements into the 8 floats a|b
__device__ __forceinline__ float4 shift4(float4 a, float4 b, int m) {
    switch (m) {   // warp-uniform
        case 0: return a;
        case 1: return make_float4(a.y, a.z, a.w, b.x);
        case 2: return make_float4(a.z, a.w, b.x, b.y);
        default: return make_float4(a.w, b.x, b.y, b.z);
    }
}

__global__ void __launch_bounds__(32 * kRowsY)
img3d_kernel(const __grid_constant__ Img3dLaunch L) {
    const Img3dDesc& d = L.d[blockIdx.z];
    int off[3];
    img3d_offsets(L, blockIdx.z, off);
    const int cd = L.crop[0], ch = L.crop[1], cw = L.crop[2];
    const int cw4 = cw >> 2;
    const int z = blockIdx.y;
    const int fz = (d.flip & 1) ? cd - 1 - z : z;
    const int sz = off[0] + fz;
    const bool z_ok = sz < d.sdim[0];
    const bool flip_w = (d.flip & 4) != 0;
    const int valid_w = d.sdim[2] - off[2];             // window columns inside the source
    const bool noise = d.sigma != 0.0f;
    float A, B;                                           // brightness (+ contrast) affine
    img3d_affine(d, (int64_t)cd * ch * cw, A, B);

    for (int qx = threadIdx.x; qx < cw4; qx += 32) {
        const int qs = flip_w ? cw4 - 1 - qx : qx;         // source quad (logical columns 4qs..4qs+3)
        float4 v[kRowsPerThread];
        uint32_t l[kRowsPerThread];
        int ys[kRowsPerThread];
#pragma unroll
        for (int r = 0; r < kRowsPerThread; ++r) {
            const int y = blockIdx.x * kRowsPerCta + threadIdx.y + r * kRowsY;
            ys[r] = y;
            const int fy = (d.flip & 2) ? ch - 1 - y : y;
            const int sy = off[1] + fy;
            v[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            l[r] = 0u;
            if (!(z_ok && y < ch && sy < d.sdim[1]) || 4 * qs >= valid_w) continue;
            // logical column 0 of this window row (row start + skew + crop offset)
            const float* irow = d.img + sz * d.img_pz + sy * d.img_py +
                                ((d.img_sk0 + sz * d.img_skz + sy * d.img_sky) & 3) + off[2];
            const uint8_t* lrow = d.lbl + sz * d.lbl_pz + sy * d.lbl_py +
                                  ((d.lbl_sk0 + sz * d.lbl_skz + sy * d.lbl_sky) & 15) + off[2];
            const int mi = (int)((reinterpret_cast<uintptr_t>(irow) >> 2) & 3);   // warp-uniform
            const int mb = (int)(reinterpret_cast<uintptr_t>(lrow) & 3);
            const float4* ia = reinterpret_cast<const float4*>(irow - mi) + qs;
            const uint32_t* la = reinterpret_cast<const uint32_t*>(lrow - mb) + qs;
            const bool second_i = mi != 0 && 4 * qs + 4 - mi < valid_w;       // next chunk has data
            const bool second_l = mb != 0 && 4 * qs + 4 - mb < valid_w;
            float4 x;
            uint32_t lb;
            // rows within a chunk of the end of the source (its last row; with tiny rows,
            // the last few): element loads, as an aligned chunk could reach past the
            // caller's buffer
            const int64_t to_end_l = (int64_t)(d.sdim[0] - 1 - sz) * d.lbl_pz + (int64_t)(d.sdim[1] - 1 - sy) * d.lbl_py;
            const int64_t to_end_i = (int64_t)(d.sdim[0] - 1 - sz) * d.img_pz + (int64_t)(d.sdim[1] - 1 - sy) * d.img_py;
            if ((to_end_l < 16 || to_end_i < 4) && 4 * qs + 8 > valid_w) {
                float e[4];
                lb = 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int col = 4 * qs + k;
                    e[k] = col < valid_w ? __ldg(irow + col) : 0.f;
                    lb |= (col < valid_w ? uint32_t(__ldg(lrow + col)) : 0u) << (8 * k);
                }
                x = make_float4(e[0], e[1], e[2], e[3]);
            } else {
                const float4 a = __ldg(ia);
                const float4 b = second_i ? __ldg(ia + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
                const uint32_t wa = __ldg(la), wb = second_l ? __ldg(la + 1) : 0u;
                x = shift4(a, b, mi);
                lb = __funnelshift_r(wa, wb, 8 * mb);
            }
            if (4 * qs + 4 > valid_w) {                    // zero-pad past the source edge
                const int keep = valid_w - 4 * qs;         // 1..3 valid voxels
                if (keep < 4) x.w = 0.f;
                if (keep < 3) x.z = 0.f;
                if (keep < 2) x.y = 0.f;
                lb &= 0xFFFFFFFFu >> (8 * (4 - keep));
            }
            if (flip_w) {
                x = make_float4(x.w, x.z, x.y, x.x);
                lb = __byte_perm(lb, 0, 0x0123);
            }
            v[r] = x;
            l[r] = lb;
        }
#pragma unroll
        for (int r = 0; r < kRowsPerThread; ++r) {
            const int y = ys[r];
            if (y >= ch) continue;
            const int64_t vox = ((int64_t)z * ch + y) * cw + 4 * qx;   // output voxel index
            float o[4] = {fmaf(v[r].x, A, B), fmaf(v[r].y, A, B), fmaf(v[r].z, A, B),
                          fmaf(v[r].w, A, B)};                        // RandomBrightness / Contrast
            if (noise) {                                               // GaussianNoise
                const uint64_t g = (uint64_t)vox >> 2;
                const uint4 rnd = philox4x32_10(
                    make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0u, 0u), d.key0, d.key1);
                const float2 z01 = box_muller(rnd.x, rnd.y);
                const float2 z23 = box_muller(rnd.z, rnd.w);
                o[0] = fmaf(d.sigma, z01.x, o[0]);
                o[1] = fmaf(d.sigma, z01.y, o[1]);
                o[2] = fmaf(d.sigma, z23.x, o[2]);
                o[3] = fmaf(d.sigma, z23.y, o[3]);
            }
            // Cast: f32 image, u8 label
            __stcs(reinterpret_cast<float4*>(d.out_img + vox), make_float4(o[0], o[1], o[2], o[3]));
            __stcs(reinterpret_cast<unsigned int*>(d.out_lbl + vox), l[r]);
        }
    }
    if (L.st.cnt != nullptr) {   // this CTA's rows of the sample are written
        __syncthreads();
        if (threadIdx.x == 0 && threadIdx.y == 0)
            sample_part_done(L.st.cnt + d.slot, L.st.stamp + d.slot, gridDim.x * gridDim.y);
    }
}

// ------------------------------------------------------------------ TMA tile path
// HBM-resident volumes whose rows are 16-B aligned (W % 16 == 0) take this
// path.  A tile is kImg3dTileRows output rows of one z-slice of one sample; the
// crop window's rows for it are two 3-D TMA boxes (image, label; kTR rows each) of the
// source volume -- the copy engine handles the arbitrary crop offset and
// zero-fills boxes hanging over the volume's edge (RandomCrop's padding), so
// the threads issue no global loads and no address arithmetic.
//
// Persistent CTAs, one producer thread and 8 consumer warps.  The producer
// streams tiles into a kTmaStages-deep shared-memory ring and publishes, next
// to each tile, a 64-byte record with everything its consumer needs (output
// addresses, brightness / noise parameters, flips, realignment), so consumers
// never divide, never touch the parameter block and never wait on each other:
// tile k of the CTA belongs to consumer warp k % 8 alone, which keeps 8 tiles
// in flight per CTA (the per-tile latency chain -- barrier wait, record load,
// shared loads, stores -- measured as the bottleneck when all 8 warps shared
// every tile).  Flip = reversed row / quad order; 16-B streaming stores.
constexpr int kTR = kImg3dTileRows;
#ifndef LFG_IMG3D_STAGES
#define LFG_IMG3D_STAGES 16   // (build-time A/B switch)
#endif
constexpr int kTmaStages = LFG_IMG3D_STAGES;
constexpr int kTmaWarps = 8;                       // consumer warps
constexpr int kTmaThreads = 32 * (kTmaWarps + 1);  // + producer warp
// header: full / empty barriers, tile records, the launch's sample descriptors
constexpr int kTmaRecOff = 4 * kTmaStages * 8;
constexpr int kTmaDescOff = kTmaRecOff + kTmaStages * 64;
constexpr int kTmaHdr = (kTmaDescOff + kMax3D * (int)sizeof(Img3dDesc) + 127) / 128 * 128;

// A box must start on a 16-B boundary (an unaligned first byte faults on
// sm_100a), so the image box starts at the crop column rounded down to 4
// elements and is cw + 4 wide, the label box at the column rounded down to 16
// bytes and cw + 16 wide; the consumers realign both by the warp-uniform
// element shift off[2] & 3.  The maps use 64-B L2 sector promotion (img3d_encode_maps):
// 1.20x the window's bytes read, against 1.40x with none or 128-B promotion (measured).
constexpr int kPadImg = 4, kPadLbl = 16;
__host__ __device__ inline int tma_stage_bytes(int cw) { return kTR * ((cw + kPadImg) * 4 + (cw + kPadLbl)); }
__host__ __device__ inline int tma_smem_bytes(int cw) { return kTmaHdr + kTmaStages * tma_stage_bytes(cw); }

struct __align__(16) TileRec {
    float* out_img;          // output voxel (z, y0, 0) of this tile
    uint8_t* out_lbl;
    uint64_t q0;             // Philox group of the tile's first voxel
    float scale, sigma;      // affine A (brightness [x contrast]), noise std (0 = none)
    uint32_t key0, key1;
    int32_t rows;            // valid output rows (y0 + r < ch)
    int32_t flags;           // bit 0 flip_y, bit 1 flip_w
    int32_t wl0, m;          // realignment: first label word inside the box row, element shift
    float bias;              // affine B (contrast; 0 otherwise)
    int32_t slot;            // the sample's completion stamp slot
};
static_assert(sizeof(TileRec) == 64, "tile record is one 64-B slot");

// kDebug: the LFG_IMG3D_DEBUG profiling switches are compiled in (debug launches only),
// so the production tile loop carries no switch tests
template <bool kDebug>
__global__ void __launch_bounds__(kTmaThreads)
img3d_tma_kernel(const __grid_constant__ Img3dLaunch L) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int cd = L.crop[0], ch = L.crop[1], cw = L.crop[2];
    const int nyb = (ch + kTR - 1) / kTR;
    const int per = cd * nyb;
    const int total = L.n * per;
    const uint32_t img_bytes = kTR * (cw + kPadImg) * 4, stage_bytes = tma_stage_bytes(cw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kTmaStages;
    TileRec* rec = reinterpret_cast<TileRec*>(smem + kTmaRecOff);
    Img3dDesc* sdesc = reinterpret_cast<Img3dDesc*>(smem + kTmaDescOff);
    uint8_t* tiles = smem + kTmaHdr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {   // the descriptors the producer reads per tile, staged once (parameter-space
        // loads with a dynamic index are slow and would sit on its critical path)
        const int words = L.n * (int)sizeof(Img3dDesc) / 4;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(L.d);
        uint32_t* dst = reinterpret_cast<uint32_t*>(sdesc);
        for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
    }
    if (L.offs != nullptr) {   // foreground-biased crops: window origins resolved by K2
        __syncthreads();
        if ((int)threadIdx.x < L.n) {
            int off[3];
            img3d_offsets(L, threadIdx.x, off);
            for (int a = 0; a < 3; ++a) sdesc[threadIdx.x].off[a] = off[a];
        }
    }
    __syncthreads();

    if (warp == kTmaWarps) {
        // producer: lane j < kTmaStages owns ring stage j and fills it with this
        // CTA's tiles j, j + 16, ... (16 independent issue chains)
        if (lane < kTmaStages) {
            const int ntiles = (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
            const int s = lane;
            for (int k = lane, use = 0; k < ntiles; k += kTmaStages, ++use) {
                if (use > 0) mbar_wait(empty + s, (use - 1) & 1);
                const int t = (int)blockIdx.x + k * (int)gridDim.x;
                // (debug bit 4: samples interleaved tile by tile instead of one after another)
                const int i = (kDebug && (L.debug & 4)) ? t % L.n : t / per;
                const int rr = (kDebug && (L.debug & 4)) ? t / L.n : t - i * per;
                const int z = rr / nyb, y0 = (rr - z * nyb) * kTR;
                Img3dDesc& d = sdesc[i];
                if (kDebug && (L.debug & 8)) d.off[2] &= ~31;   // (profiling switch: 128-B aligned crop rows; wrong output)
                const int fz = (d.flip & 1) ? cd - 1 - z : z;
                const int fy0 = (d.flip & 2) ? ch - kTR - y0 : y0;   // may be < 0: zero rows, never stored
                const int64_t v0 = ((int64_t)z * ch + y0) * cw;
                TileRec tr;
                tr.out_img = d.out_img + v0;
                tr.out_lbl = d.out_lbl + v0;
                tr.q0 = (uint64_t)v0 >> 2;
                img3d_affine(d, (int64_t)cd * ch * cw, tr.scale, tr.bias);
                tr.sigma = d.sigma;
                tr.key0 = d.key0;
                tr.key1 = d.key1;
                tr.rows = min(kTR, ch - y0);
                tr.flags = ((d.flip >> 1) & 1) | (((d.flip >> 2) & 1) << 1);
                tr.wl0 = (d.off[2] & (kPadLbl - 1)) >> 2;
                tr.m = d.off[2] & 3;
                tr.slot = d.slot;
                rec[s] = tr;
                if (kDebug && (L.debug & 2)) {   // profiling switch: no loads
                    mbar_arrive(full + s);
                } else {
                    uint8_t* st = tiles + s * stage_bytes;
                    mbar_expect_tx(full + s, stage_bytes);
                    tma_load_3d(st, &L.tm_img[i], d.off[2] & ~(kPadImg - 1), d.off[1] + fy0, d.off[0] + fz,
                                full + s);
                    tma_load_3d(st + img_bytes, &L.tm_lbl[i], d.off[2] & ~(kPadLbl - 1), d.off[1] + fy0,
                                d.off[0] + fz, full + s);
                }
            }
        }
        return;
    }

    const int cw4 = cw >> 2, bi4 = (cw + kPadImg) >> 2, bl4 = (cw + kPadLbl) >> 2;
    const int ntiles = (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    for (int k = warp; k < ntiles; k += kTmaWarps) {
        const int s = k % kTmaStages, use = k / kTmaStages;
        mbar_wait(full + s, use & 1);
        const TileRec tr = rec[s];
        const bool flip_y = (tr.flags & 1) != 0, flip_w = (tr.flags & 2) != 0;
        const float4* simg = reinterpret_cast<const float4*>(tiles + s * stage_bytes);
        const uint32_t* slbl = reinterpret_cast<const uint32_t*>(tiles + s * stage_bytes + img_bytes);
#pragma unroll 2
        for (int r = 0; r < tr.rows; ++r) {
            const int sr = flip_y ? kTR - 1 - r : r;
            for (int qx = lane; qx < cw4; qx += 32) {
                const int qs = flip_w ? cw4 - 1 - qx : qx;
                const int wi = sr * bi4 + qs, wl = sr * bl4 + tr.wl0 + qs;
                float4 x = simg[wi];
                uint32_t lb = slbl[wl];
                if (tr.m != 0) {
                    x = shift4(x, simg[wi + 1], tr.m);
                    lb = __funnelshift_r(lb, slbl[wl + 1], 8 * tr.m);
                }
                if (flip_w) {
                    x = make_float4(x.w, x.z, x.y, x.x);
                    lb = __byte_perm(lb, 0, 0x0123);
                }
                const int vo = r * cw + 4 * qx;   // voxel offset inside the tile
                float o[4] = {fmaf(x.x, tr.scale, tr.bias), fmaf(x.y, tr.scale, tr.bias),
                              fmaf(x.z, tr.scale, tr.bias), fmaf(x.w, tr.scale, tr.bias)};
                if (tr.sigma != 0.0f) {
                    const uint64_t g = tr.q0 + (uint64_t)(vo >> 2);
                    const uint4 rnd = philox4x32_10(
                        make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0u, 0u), tr.key0, tr.key1);
                    const float2 z01 = box_muller(rnd.x, rnd.y);
                    const float2 z23 = box_muller(rnd.z, rnd.w);
                    o[0] = fmaf(tr.sigma, z01.x, o[0]);
                    o[1] = fmaf(tr.sigma, z01.y, o[1]);
                    o[2] = fmaf(tr.sigma, z23.x, o[2]);
                    o[3] = fmaf(tr.sigma, z23.y, o[3]);
                }
                if (kDebug && (L.debug & 1)) {   // profiling switch: no stores
                    if (o[0] == 123.f && lb == 7u) tr.out_img[0] = o[1];
                    continue;
                }
                __stcs(reinterpret_cast<float4*>(tr.out_img + vo), make_float4(o[0], o[1], o[2], o[3]));
                __stcs(reinterpret_cast<unsigned int*>(tr.out_lbl + vo), lb);
            }
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(empty + s);
            // one part of per = cd * nyb tiles of the sample is written
            if (L.st.cnt != nullptr) sample_part_done(L.st.cnt + tr.slot, L.st.stamp + tr.slot, (uint32_t)per);
        }
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

}  // namespace

cudaError_t img3d_encode_maps(Img3dLaunch& L, int i, const void* img, const void* lbl, const int64_t dims[3]) {
    EncodeTiledFn fn = encode_fn();
    if (fn == nullptr) return cudaErrorNotSupported;
    // L2 sector promotion of the maps: 64 B.  A crop row's box starts at a random 16-B offset,
    // so its first and last DRAM atoms are partial; without promotion the reads came out at
    // 1.40x the window's bytes (128-B fetches), with 64-B promotion at 1.20x (ncu, 16
    // volumes: 235 -> 201 MB read, 85 -> 80 us).  LFG_TMA_PROMO=0|128|256: A/B switch.
    static const CUtensorMapL2promotion promo = [] {
        const char* e = getenv("LFG_TMA_PROMO");
        const int v = e ? atoi(e) : 64;
        return v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                       : (v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                   : (v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE));
    }();
    const cuuint64_t gdim[3] = {(cuuint64_t)dims[2], (cuuint64_t)dims[1], (cuuint64_t)dims[0]};
    const cuuint32_t box_i[3] = {(cuuint32_t)(L.crop[2] + kPadImg), (cuuint32_t)kTR, 1};
    const cuuint32_t box_l[3] = {(cuuint32_t)(L.crop[2] + kPadLbl), (cuuint32_t)kTR, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint64_t si[2] = {(cuuint64_t)dims[2] * 4, (cuuint64_t)(dims[1] * dims[2]) * 4};
    const cuuint64_t sl[2] = {(cuuint64_t)dims[2], (cuuint64_t)(dims[1] * dims[2])};
    CUresult r = fn(&L.tm_img[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(img), gdim, si, box_i,
                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    r = fn(&L.tm_lbl[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(lbl), gdim, sl, box_l, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_img3d(const Img3dLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    if (L.tma) {
        const int cw = L.crop[2];
        if (cw % 16 != 0 || cw > 240) return cudaErrorInvalidValue;
        const int smem = tma_smem_bytes(cw);
        // resident CTAs per SM, per cw / 16 (same on every B200; a benign race between
        // shard threads: each computes the same value)
        static std::atomic<int> occ[17];
        int o = occ[cw / 16].load(std::memory_order_relaxed);
        if (o == 0) {
            int v = 0;
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, img3d_tma_kernel<false>, kTmaThreads, smem);
            if (e != cudaSuccess) return e;
            o = v > 0 ? v : 1;
            occ[cw / 16].store(o, std::memory_order_relaxed);
        }
        const int64_t total = int64_t(L.n) * L.crop[0] * ((L.crop[1] + kTR - 1) / kTR);
        const int grid = static_cast<int>(std::min<int64_t>(total, int64_t(sm_count()) * o));
        static const int dbg = getenv("LFG_IMG3D_DEBUG") ? atoi(getenv("LFG_IMG3D_DEBUG")) : 0;
        static const int ctas = getenv("LFG_IMG3D_CTAS") ? atoi(getenv("LFG_IMG3D_CTAS")) : 0;
        if (dbg == 0 && ctas == 0) {
            img3d_tma_kernel<false><<<grid, kTmaThreads, smem, s>>>(L);
        } else {
            Img3dLaunch L2 = L;
            L2.debug = dbg;
            const int g2 = ctas ? static_cast<int>(std::min<int64_t>(total, int64_t(sm_count()) * ctas)) : grid;
            img3d_tma_kernel<true><<<g2, kTmaThreads, smem, s>>>(L2);
        }
        return cudaGetLastError();
    }
    dim3 grid((L.crop[1] + kRowsPerCta - 1) / kRowsPerCta, L.crop[0], L.n);
    dim3 block(32, kRowsY);
    img3d_kernel<<<grid, block, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t warm_img3d() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, img3d_kernel);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(img3d_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem_bytes(240));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(img3d_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem_bytes(240));
    if (e != cudaSuccess) return e;
    sm_count();
    encode_fn();
    return cudaFuncGetAttributes(&a, img3d_tma_kernel<false>);
}

}  // namespace lfg
