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
    const int cd = L.crop[0], ch = L.crop[1], cw = L.crop[2];
    const int cw4 = cw >> 2;
    const int z = blockIdx.y;
    const int fz = (d.flip & 1) ? cd - 1 - z : z;
    const int sz = d.off[0] + fz;
    const bool z_ok = sz < d.sdim[0];
    const bool flip_w = (d.flip & 4) != 0;
    const int valid_w = d.sdim[2] - d.off[2];             // window columns inside the source
    const bool noise = d.sigma != 0.0f;

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
            const int sy = d.off[1] + fy;
            v[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            l[r] = 0u;
            if (!(z_ok && y < ch && sy < d.sdim[1]) || 4 * qs >= valid_w) continue;
            // logical column 0 of this window row (row start + skew + crop offset)
            const float* irow = d.img + sz * d.img_pz + sy * d.img_py +
                                ((d.img_sk0 + sz * d.img_skz + sy * d.img_sky) & 3) + d.off[2];
            const uint8_t* lrow = d.lbl + sz * d.lbl_pz + sy * d.lbl_py +
                                  ((d.lbl_sk0 + sz * d.lbl_skz + sy * d.lbl_sky) & 15) + d.off[2];
            const int mi = (int)((reinterpret_cast<uintptr_t>(irow) >> 2) & 3);   // warp-uniform
            const int mb = (int)(reinterpret_cast<uintptr_t>(lrow) & 3);
            const float4* ia = reinterpret_cast<const float4*>(irow - mi) + qs;
            const uint32_t* la = reinterpret_cast<const uint32_t*>(lrow - mb) + qs;
            const bool second_i = mi != 0 && 4 * qs + 4 - mi < valid_w;       // next chunk has data
            const bool second_l = mb != 0 && 4 * qs + 4 - mb < valid_w;
            const float4 a = __ldg(ia);
            const float4 b = second_i ? __ldg(ia + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
            const uint32_t wa = __ldg(la), wb = second_l ? __ldg(la + 1) : 0u;
            float4 x = shift4(a, b, mi);
            uint32_t lb = __funnelshift_r(wa, wb, 8 * mb);
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
            float o[4] = {v[r].x * d.scale, v[r].y * d.scale, v[r].z * d.scale,
                          v[r].w * d.scale};                          // RandomBrightness
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
}

}  // namespace

cudaError_t launch_img3d(const Img3dLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    dim3 grid((L.crop[1] + kRowsPerCta - 1) / kRowsPerCta, L.crop[0], L.n);
    dim3 block(32, kRowsY);
    img3d_kernel<<<grid, block, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t warm_img3d() {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, img3d_kernel);
}

}  // namespace lfg
