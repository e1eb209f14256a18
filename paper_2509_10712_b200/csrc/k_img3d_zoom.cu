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
// voxels (one Philox block, as K1).  The CTA's per-column taps (source columns,
// fp32 weights, nearest label column) and per-plane z taps are computed once into
// shared memory in fp64 with the oracle's exact (non-contracted) operations, so
// tap indices always agree with the oracle; y taps are per-warp scalars.  Source
// taps come through the read-only path (__ldg): neighbouring voxels share source
// lines, so HBM sees the window about once; each source plane is x/y-blended once
// per output row (separable form, below).  Output: f32 image with the
// brightness/contrast affine and Philox noise of K1, u8 label (nearest), 16-B /
// 4-B streaming stores.
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

// per output plane of the CTA: z taps and the source planes' offsets (the plane
// part of img_row's address; -1 = outside the source, zero padding)
struct ZPlane {
    int64_t io0, io1, lo;      // image planes z0, z1 and label plane nz: element / byte offsets
    int32_t ik0, ik1, lk;      // their skew terms (the z part of the row skew)
    int32_t z0, z1;
    float lz0, lz1;
};

// Trilinear in separable form: H(s) = ly0 * X(s, y0) + ly1 * X(s, y1) is the
// y-blended, x-interpolated source plane s of this output row and
// out = lz0 * H(z0) + lz1 * H(z1) -- the per-voxel formula's operations in the same
// order, so bit-identical to it.  Consecutive output planes share source planes,
// so each H(s) is built once and kept in the register set of its parity (z0 and
// z0 + 1 never collide: K3's row trick along z): ~zoom H builds (8 taps + 12 FMA
// per lane) per output plane instead of 8 taps + 7 FMA per voxel.  A lane owns 4
// consecutive output columns across the CTA's planes; z taps and the planes'
// offsets come from a per-CTA table, the row part of the offsets is per warp.
// 64 registers (4 CTAs per SM): the per-voxel form measured 210 us per 16 zoomed
// 128^3 crops, this one 135 us (ncu: 99 M -> 67 M instructions).
__global__ void __launch_bounds__(32 * kZRows, 4) img3d_zoom_kernel(const __grid_constant__ Img3dLaunch L) {
    __shared__ __align__(16) int2 sx_tap[kMaxCrop];
    __shared__ __align__(16) float2 sx_w[kMaxCrop];
    __shared__ __align__(16) int sx_near[kMaxCrop];
    __shared__ ZPlane sz_tab[kZPlanes];
    const Img3dDesc& d = L.d[blockIdx.z];
    int off[3];
    img3d_offsets(L, blockIdx.z, off);
    const int cd = L.crop[0], ch = L.crop[1], cw = L.crop[2];
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const bool flip_w = (d.flip & 4) != 0;
    const int valid_w = d.sdim[2] - off[2];
    for (int x = tid; x < cw; x += 32 * kZRows) {
        const int wx = flip_w ? cw - 1 - x : x;
        int i0, i1;
        double l0, l1;
        taps(wx, d.win[2], d.zscale[2], i0, i1, l0, l1);
        sx_tap[x] = make_int2(i0 < valid_w ? i0 : 0, i1 < valid_w ? i1 : 0);
        sx_w[x] = make_float2(i0 < valid_w ? (float)l0 : 0.f, i1 < valid_w ? (float)l1 : 0.f);
        const int nx = min(wx * d.win[2] / cw, d.win[2] - 1);
        sx_near[x] = nx < valid_w ? nx : -1;
    }
    const int z_begin = blockIdx.y * kZPlanes, z_end = min(cd, z_begin + kZPlanes);
    if (tid >= 32 * kZRows - kZPlanes) {
        const int z = z_begin + tid - (32 * kZRows - kZPlanes);
        if (z < z_end) {
            const int wz = (d.flip & 1) ? cd - 1 - z : z;
            ZPlane e;
            double lz0d, lz1d;
            taps(wz, d.win[0], d.zscale[0], e.z0, e.z1, lz0d, lz1d);
            e.lz0 = (float)lz0d;
            e.lz1 = (float)lz1d;
            const int nz = min(wz * d.win[0] / cd, d.win[0] - 1);
            auto plane = [&](int zz, int64_t& io, int32_t& ik) {
                const int sz = off[0] + zz;
                io = sz < d.sdim[0] ? sz * d.img_pz + off[2] : -1;
                ik = d.img_sk0 + sz * d.img_skz;
            };
            plane(e.z0, e.io0, e.ik0);
            plane(e.z1, e.io1, e.ik1);
            const int szn = off[0] + nz;
            e.lo = szn < d.sdim[0] ? szn * d.lbl_pz + off[2] : -1;
            e.lk = d.lbl_sk0 + szn * d.lbl_skz;
            sz_tab[z - z_begin] = e;
        }
    }
    float A, B;
    img3d_affine(d, (int64_t)cd * ch * cw, A, B);
    const bool noise = d.sigma != 0.0f;
    __syncthreads();

    const int y = blockIdx.x * kZRows + threadIdx.y;
    if (y < ch) {
        const int wy = (d.flip & 2) ? ch - 1 - y : y;
        int y0, y1;
        double ly0d, ly1d;
        taps(wy, d.win[1], d.zscale[1], y0, y1, ly0d, ly1d);
        const float ly0 = (float)ly0d, ly1 = (float)ly1d;
        const int ny = min(wy * d.win[1] / ch, d.win[1] - 1);
        // the row part of img_row / lbl_row (-1: outside the source)
        const int sy0 = off[1] + y0, sy1 = off[1] + y1, syn = off[1] + ny;
        const int64_t yo0 = sy0 < d.sdim[1] ? sy0 * d.img_py : -1;
        const int64_t yo1 = sy1 < d.sdim[1] ? sy1 * d.img_py : -1;
        const int64_t ylo = syn < d.sdim[1] ? syn * d.lbl_py : -1;
        const int yk0 = sy0 * d.img_sky, yk1 = sy1 * d.img_sky, ylk = syn * d.lbl_sky;
        const int cw4 = cw >> 2;
        for (int q = threadIdx.x; q < cw4; q += 32) {
            float H0[4], H1[4];            // H of the even / odd source plane held
            int held0 = -1, held1 = -1;
            // the quad's column taps are re-read from shared memory (4 x 16 B) per build
            // rather than held across the plane loop: registers decide the occupancy here
            auto build = [&](int64_t io, int ik, float h[4]) {
                const float* r0 = (io >= 0 && yo0 >= 0) ? d.img + io + yo0 + ((ik + yk0) & 3) : nullptr;
                const float* r1 = (io >= 0 && yo1 >= 0) ? d.img + io + yo1 + ((ik + yk1) & 3) : nullptr;
                const int4 ta = reinterpret_cast<const int4*>(sx_tap)[2 * q];
                const int4 tb = reinterpret_cast<const int4*>(sx_tap)[2 * q + 1];
                const float4 wa = reinterpret_cast<const float4*>(sx_w)[2 * q];
                const float4 wb = reinterpret_cast<const float4*>(sx_w)[2 * q + 1];
                const int2 t[4] = {make_int2(ta.x, ta.y), make_int2(ta.z, ta.w), make_int2(tb.x, tb.y),
                                   make_int2(tb.z, tb.w)};
                const float2 w[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w), make_float2(wb.x, wb.y),
                                     make_float2(wb.z, wb.w)};
    #pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float a = r0 ? fmaf(w[k].x, __ldg(r0 + t[k].x), w[k].y * __ldg(r0 + t[k].y)) : 0.0f;
                    const float b = r1 ? fmaf(w[k].x, __ldg(r1 + t[k].x), w[k].y * __ldg(r1 + t[k].y)) : 0.0f;
                    h[k] = fmaf(ly0, a, ly1 * b);
                }
            };
            for (int z = z_begin; z < z_end; ++z) {
                const ZPlane& e = sz_tab[z - z_begin];
                const int z0 = e.z0, z1 = e.z1;
                // the plane's nearest labels first, so their latency overlaps the builds'
                const uint8_t* rl = (e.lo >= 0 && ylo >= 0) ? d.lbl + e.lo + ylo + ((e.lk + ylk) & 15) : nullptr;
                const int4 n4 = reinterpret_cast<const int4*>(sx_near)[q];
                const int nx[4] = {n4.x, n4.y, n4.z, n4.w};
                uint32_t lbk[4];
    #pragma unroll
                for (int k = 0; k < 4; ++k) lbk[k] = (rl != nullptr && nx[k] >= 0) ? (uint32_t)__ldg(rl + nx[k]) : 0u;
                // warp-uniform: every lane of the warp is on the same (z, y)
                if (z0 & 1) {
                    if (held1 != z0) { build(e.io0, e.ik0, H1); held1 = z0; }
                    if (z1 != z0 && held0 != z1) { build(e.io1, e.ik1, H0); held0 = z1; }
                } else {
                    if (held0 != z0) { build(e.io0, e.ik0, H0); held0 = z0; }
                    if (z1 != z0 && held1 != z1) { build(e.io1, e.ik1, H1); held1 = z1; }
                }
                const bool odd0 = (z0 & 1) != 0, odd1 = (z1 & 1) != 0;
                const float lz0 = e.lz0, lz1 = e.lz1;
                float o[4];
                const uint32_t lb = lbk[0] | (lbk[1] << 8) | (lbk[2] << 16) | (lbk[3] << 24);
    #pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float a = odd0 ? H1[k] : H0[k];
                    const float b = odd1 ? H1[k] : H0[k];
                    o[k] = fmaf(A, fmaf(lz0, a, lz1 * b), B);
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
    if (L.st.cnt != nullptr) {   // this CTA's rows of the sample are written
        __syncthreads();
        if (threadIdx.x == 0 && threadIdx.y == 0)
            sample_part_done(L.st.cnt + d.slot, L.st.stamp + d.slot, gridDim.x * gridDim.y);
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
