// k_img3d_zoom.cu -- K4: the img_seg chain with RandomZoom3D (trilinear
// resample of a zoomed crop window), and K5: the per-sample crop mean that
// RandomContrast needs.
//
// Neither op is in the reference's img_seg chain (RandomCrop, RandomFlip,
// RandomBrightness, GaussianNoise, Cast -- proj/src/workloads.cpp:142-148);
// they are the north_star's "trilinear resize" and "brightness/contrast"
// transforms, added as optional ops.  Semantics: oracle/lf_oracle.c
// lfo_draw3d / lfo_apply3d.
//
// K4 mapping: grid (ceil(ch / 8), ceil(cd / 8), n), block (32, 8): a warp per
// output row (for 8 consecutive output planes), a lane per 4 consecutive output
// voxels (one Philox block, as K1).  The
// CTA's per-column taps (source columns, fp32 weights, nearest label column)
// are computed once into shared memory in fp64 with the oracle's exact
// (non-contracted) operations, so tap indices always agree with the oracle;
// z / y taps are per-row scalars.  The 8 image taps of a voxel come through
// the read-only path (__ldg): neighbouring voxels share source lines, so HBM
// sees the window about once.  Output: f32 image with the brightness/contrast
// affine and Philox noise of K1, u8 label (nearest), 16-B / 4-B streaming
// stores.
//
// K5: sum over the crop of the resampled image R, computed from the source
// window without materialising R: sum(R) = sum_z,y,x cz[z] cy[y] cx[x] src,
// where c_a[i] = sum over output positions of the linear weight on source i
// (separable).  One CTA per (window plane, sample); fp32 row partials, fp64
// CTA reduction and one fp64 atomicAdd per CTA.
#include <algorithm>

#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kZRows = 8;          // output rows per CTA (threadIdx.y)
constexpr int kZPlanes = 8;        // output planes per CTA
constexpr int kMaxCrop = 1024;

// PyTorch area_pixel_compute_source_index (align_corners=False) + linear taps,
// fp64 with _rn intrinsics (no FMA contraction): identical to linear_taps() of
// the oracle.
// `scale` is (double)in / (double)out, divided once on the host (IEEE, as the oracle).
__device__ __forceinline__ void taps(int dst, int in, double scale, int& i0, int& i1, double& l0, double& l1) {
    double src = __dadd_rn(__dmul_rn(scale, __dadd_rn((double)dst, 0.5)), -0.5);
    if (src < 0.0) src = 0.0;
    int a = (int)floor(src);
    if (a > in - 1) a = in - 1;
    i0 = a;
    i1 = a < in - 1 ? a + 1 : a;
    l1 = __dadd_rn(src, -(double)a);
    l0 = __dadd_rn(1.0, -l1);
}

// start of source row (z, y) of the window (window coordinates), or null if the
// row lies outside the source's valid extent (zero padding)
__device__ __forceinline__ const float* img_row(const Img3dDesc& d, const int off[3], int z, int y) {
    const int sz = off[0] + z, sy = off[1] + y;
    if (sz >= d.sdim[0] || sy >= d.sdim[1]) return nullptr;
    return d.img + sz * d.img_pz + sy * d.img_py + ((d.img_sk0 + sz * d.img_skz + sy * d.img_sky) & 3) + off[2];
}
__device__ __forceinline__ const uint8_t* lbl_row(const Img3dDesc& d, const int off[3], int z, int y) {
    const int sz = off[0] + z, sy = off[1] + y;
    if (sz >= d.sdim[0] || sy >= d.sdim[1]) return nullptr;
    return d.lbl + sz * d.lbl_pz + sy * d.lbl_py + ((d.lbl_sk0 + sz * d.lbl_skz + sy * d.lbl_sky) & 15) + off[2];
}

__global__ void __launch_bounds__(32 * kZRows) img3d_zoom_kernel(const __grid_constant__ Img3dLaunch L) {
    __shared__ int2 sx_tap[kMaxCrop];     // per output column (after flip): source columns x0, x1
    __shared__ float2 sx_w[kMaxCrop];     // weights l0, l1
    __shared__ int sx_near[kMaxCrop];     // nearest label column
    const Img3dDesc& d = L.d[blockIdx.z];
    int off[3];
    img3d_offsets(L, blockIdx.z, off);
    const int cd = L.crop[0], ch = L.crop[1], cw = L.crop[2];
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const bool flip_w = (d.flip & 4) != 0;
    const int valid_w = d.sdim[2] - off[2];      // window columns inside the source
    for (int x = tid; x < cw; x += 32 * kZRows) {
        const int wx = flip_w ? cw - 1 - x : x;
        int i0, i1;
        double l0, l1;
        taps(wx, d.win[2], d.zscale[2], i0, i1, l0, l1);
        // taps past the source edge read zero: fold that into the weights
        sx_tap[x] = make_int2(i0 < valid_w ? i0 : 0, i1 < valid_w ? i1 : 0);
        sx_w[x] = make_float2(i0 < valid_w ? (float)l0 : 0.f, i1 < valid_w ? (float)l1 : 0.f);
        const int nx = min(wx * d.win[2] / cw, d.win[2] - 1);
        sx_near[x] = nx < valid_w ? nx : -1;
    }
    float A, B;
    img3d_affine(d, (int64_t)cd * ch * cw, A, B);
    const bool noise = d.sigma != 0.0f;
    __syncthreads();

    const int y = blockIdx.x * kZRows + threadIdx.y;
    if (y >= ch) return;
    const int wy = (d.flip & 2) ? ch - 1 - y : y;
    int y0, y1;
    double ly0d, ly1d;
    taps(wy, d.win[1], d.zscale[1], y0, y1, ly0d, ly1d);
    const float ly0 = (float)ly0d, ly1 = (float)ly1d;
    const int ny = min(wy * d.win[1] / ch, d.win[1] - 1);
    const int cw4 = cw >> 2;
    // the CTA's rows, for kZPlanes consecutive output planes (amortises the column table)
    const int z_end = min(cd, (int)(blockIdx.y + 1) * kZPlanes);
    for (int z = blockIdx.y * kZPlanes; z < z_end; ++z) {
        const int wz = (d.flip & 1) ? cd - 1 - z : z;
        int z0, z1;
        double lz0d, lz1d;
        taps(wz, d.win[0], d.zscale[0], z0, z1, lz0d, lz1d);
        const float lz0 = (float)lz0d, lz1 = (float)lz1d;
        const int nz = min(wz * d.win[0] / cd, d.win[0] - 1);
        const float* r00 = img_row(d, off, z0, y0);
        const float* r01 = img_row(d, off, z0, y1);
        const float* r10 = img_row(d, off, z1, y0);
        const float* r11 = img_row(d, off, z1, y1);
        const uint8_t* rl = lbl_row(d, off, nz, ny);
        auto tap_row = [&](const float* r, int2 t, float2 w) -> float {
            if (r == nullptr) return 0.0f;
            return fmaf(w.x, __ldg(r + t.x), w.y * __ldg(r + t.y));
        };
        for (int q = threadIdx.x; q < cw4; q += 32) {
            float o[4];
            uint32_t lb = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int x = 4 * q + k;
                const int2 t = sx_tap[x];
                const float2 w = sx_w[x];
                const float a = fmaf(ly0, tap_row(r00, t, w), ly1 * tap_row(r01, t, w));
                const float b = fmaf(ly0, tap_row(r10, t, w), ly1 * tap_row(r11, t, w));
                o[k] = fmaf(A, fmaf(lz0, a, lz1 * b), B);
                const int nx = sx_near[x];
                if (rl != nullptr && nx >= 0) lb |= (uint32_t)__ldg(rl + nx) << (8 * k);
            }
            const int64_t vox = ((int64_t)z * ch + y) * cw + 4 * q;
            if (noise) {
                const uint64_t g = (uint64_t)vox >> 2;
                const uint4 rnd =
                    philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0u, 0u), d.key0, d.key1);
                const float2 z01 = box_muller(rnd.x, rnd.y);
                const float2 z23 = box_muller(rnd.z, rnd.w);
                o[0] = fmaf(d.sigma, z01.x, o[0]);
                o[1] = fmaf(d.sigma, z01.y, o[1]);
                o[2] = fmaf(d.sigma, z23.x, o[2]);
                o[3] = fmaf(d.sigma, z23.y, o[3]);
            }
            __stcs(reinterpret_cast<float4*>(d.out_img + vox), make_float4(o[0], o[1], o[2], o[3]));
            __stcs(reinterpret_cast<unsigned int*>(d.out_lbl + vox), lb);
        }
    }
}

// c_a[i]: total linear weight source index i receives over all output positions
// (deterministic: thread i walks the output positions that can tap it)
__device__ __forceinline__ float axis_weight(int i, int win, int crop, double scale) {
    if (win == crop) return 1.0f;
    const double inv = (double)crop / (double)win;
    int lo = (int)floor(((double)i - 0.5) * inv - 0.5) - 1;
    int hi = (int)ceil(((double)i + 1.5) * inv - 0.5) + 1;
    lo = max(lo, 0);
    hi = min(hi, crop - 1);
    double c = 0.0;
    for (int dst = lo; dst <= hi; ++dst) {
        int i0, i1;
        double l0, l1;
        taps(dst, win, scale, i0, i1, l0, l1);
        if (i0 == i) c += l0;
        if (i1 == i) c += l1;
    }
    return (float)c;
}

constexpr int kMeanThreads = 256;

__global__ void __launch_bounds__(kMeanThreads) img3d_mean_kernel(const __grid_constant__ Img3dLaunch L) {
    __shared__ float cx[kMaxCrop * 2];
    __shared__ float cy[kMaxCrop * 2];
    __shared__ double red[kMeanThreads / 32];
    const Img3dDesc& d = L.d[blockIdx.y];
    if (d.csum == nullptr) return;                 // not a contrasted sample
    int off[3];
    img3d_offsets(L, blockIdx.y, off);
    const int z = blockIdx.x;                      // window plane
    if (z >= d.win[0]) return;
    const int ww = min(d.win[2], d.sdim[2] - off[2]);   // window extent inside the source
    const int wh = min(d.win[1], d.sdim[1] - off[1]);
    if (off[0] + z >= d.sdim[0] || ww <= 0 || wh <= 0) return;
    for (int i = threadIdx.x; i < ww; i += kMeanThreads) cx[i] = axis_weight(i, d.win[2], L.crop[2], d.zscale[2]);
    for (int i = threadIdx.x; i < wh; i += kMeanThreads) cy[i] = axis_weight(i, d.win[1], L.crop[1], d.zscale[1]);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int y = warp; y < wh; y += kMeanThreads / 32) {
        const float* r = img_row(d, off, z, y);
        float s = 0.0f;
        for (int x = lane; x < ww; x += 32) s = fmaf(cx[x], __ldg(r + x), s);
        acc += (double)cy[y] * (double)s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kMeanThreads / 32; ++w) t += red[w];
        atomicAdd(const_cast<double*>(d.csum), t * (double)axis_weight(z, d.win[0], L.crop[0], d.zscale[0]));
    }
}

}  // namespace

cudaError_t launch_img3d_zoom(const Img3dLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    if (L.crop[2] > kMaxCrop || (L.crop[2] & 3)) return cudaErrorInvalidValue;
    dim3 grid((L.crop[1] + kZRows - 1) / kZRows, (L.crop[0] + kZPlanes - 1) / kZPlanes, L.n);
    img3d_zoom_kernel<<<grid, dim3(32, kZRows), 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_img3d_mean(const Img3dLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    int planes = 1;
    for (int i = 0; i < L.n; ++i) {
        if (L.d[i].win[1] > 2 * kMaxCrop || L.d[i].win[2] > 2 * kMaxCrop) return cudaErrorInvalidValue;
        planes = std::max(planes, L.d[i].win[0]);
    }
    img3d_mean_kernel<<<dim3(planes, L.n), kMeanThreads, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t warm_img3d_zoom() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, img3d_zoom_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, img3d_mean_kernel);
    return e;
}

}  // namespace lfg
