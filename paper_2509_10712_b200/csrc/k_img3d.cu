// k_img3d.cu -- K1: fused img_seg chain for a launch group of volumes.
//
// Realises the reference transforms RandomCrop (0.0735), RandomFlip,
// RandomBrightness, GaussianNoise, Cast (proj/src/workloads.cpp:142-148) in
// one pass: every output voxel is read once and written once.
//
// Algorithmic HBM bytes per sample: read cd*ch*cw*(4+1) + write cd*ch*cw*(4+1)
// (20,971,520 B at 128^3).  Mapping: grid (ch/16, cd, n_samples); a warp
// owns one output row (32 lanes x 4 voxels = 128), each thread does 2 rows
// (y and y+8) so 16 scalar loads are in flight before the math; img and
// label stores are 16-B / 4-B vector stores.  GaussianNoise uses one
// Philox4x32-10 call per 4 output voxels (the 4 voxels a thread owns), so
// noise-on samples are ALU-bound while noise-off samples are HBM-bound.
#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kRowsY = 8;          // threadIdx.y extent
constexpr int kRowsPerThread = 2;  // rows y, y + kRowsY
constexpr int kRowsPerCta = kRowsY * kRowsPerThread;

__global__ void __launch_bounds__(32 * kRowsY)
img3d_kernel(const __grid_constant__ Img3dLaunch L) {
    const Img3dDesc& d = L.d[blockIdx.z];
    const int cd = L.crop[0], ch = L.crop[1], cw = L.crop[2];
    const int cw4 = cw >> 2;
    const int z = blockIdx.y;
    const int fz = (d.flip & 1) ? cd - 1 - z : z;
    const int sz = d.off[0] + fz;
    const bool z_ok = sz < d.sdim[0];
    const bool noise = d.sigma != 0.0f;

    for (int qx = threadIdx.x; qx < cw4; qx += 32) {
        float v[kRowsPerThread][4];
        uint8_t l[kRowsPerThread][4];
        int ys[kRowsPerThread];
#pragma unroll
        for (int r = 0; r < kRowsPerThread; ++r) {
            const int y = blockIdx.x * kRowsPerCta + threadIdx.y + r * kRowsY;
            ys[r] = y;
            const int fy = (d.flip & 2) ? ch - 1 - y : y;
            const int sy = d.off[1] + fy;
            const bool row_ok = z_ok && y < ch && sy < d.sdim[1];
            // row start (see kernels.h): pitch + alignment-phase skew
            const float* irow = d.img + sz * d.img_pz + sy * d.img_py +
                                ((d.img_sk0 + sz * d.img_skz + sy * d.img_sky) & 3);
            const uint8_t* lrow = d.lbl + sz * d.lbl_pz + sy * d.lbl_py +
                                  ((d.lbl_sk0 + sz * d.lbl_skz + sy * d.lbl_sky) & 15);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int x = 4 * qx + j;
                const int fx = (d.flip & 4) ? cw - 1 - x : x;
                const int sx = d.off[2] + fx;
                const bool ok = row_ok && sx < d.sdim[2];
                v[r][j] = ok ? __ldg(irow + sx) : 0.0f;
                l[r][j] = ok ? __ldg(lrow + sx) : (uint8_t)0;
            }
        }
#pragma unroll
        for (int r = 0; r < kRowsPerThread; ++r) {
            const int y = ys[r];
            if (y >= ch) continue;
            const int64_t vox = ((int64_t)z * ch + y) * cw + 4 * qx;   // output voxel index
            float o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = v[r][j] * d.scale;        // RandomBrightness
            if (noise) {                                                  // GaussianNoise
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
            *reinterpret_cast<float4*>(d.out_img + vox) = make_float4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uchar4*>(d.out_lbl + vox) =
                make_uchar4(l[r][0], l[r][1], l[r][2], l[r][3]);
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

}  // namespace lfg

namespace lfg {
cudaError_t warm_img3d() {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, img3d_kernel);
}
}  // namespace lfg
