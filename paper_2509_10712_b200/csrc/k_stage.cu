// k_stage.cu -- K0: strided-box gather from pinned host memory into HBM staging.
//
// Replaces per-sample cudaMemcpy2D/3DAsync DMA (hundreds of short rows per
// sample) on the end-to-end path: one launch per launch group reads exactly
// the bytes the chain needs (img_seg crop window, obj_det crop box) over PCIe
// with aligned 16-byte loads through the UVA mapping of the pinned buffer.
// A row is copied as the 16-B aligned superset of its byte range, so the
// staging copy keeps the source's alignment phase ("skew"); consumers
// re-derive a row's start as base + z*dst_pz + y*dst_py + (src_row_addr & 15).
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kWarps = 8;

__global__ void __launch_bounds__(32 * kWarps) stage_kernel(const __grid_constant__ StageLaunch L) {
    const StageDesc& d = L.d[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t rows = (int64_t)d.ny * d.nz;
    for (int64_t r = (int64_t)blockIdx.x * kWarps + warp; r < rows; r += (int64_t)gridDim.x * kWarps) {
        const int64_t z = r / d.ny, y = r - z * d.ny;
        const uintptr_t s = reinterpret_cast<uintptr_t>(d.src) + z * d.src_pz + y * d.src_py;
        const uintptr_t a = s & ~uintptr_t(15);
        const int nch = (int)(((s + d.row_bytes + 15) & ~uintptr_t(15)) - a) >> 4;
        const int4* src = reinterpret_cast<const int4*>(a);
        int4* dst = reinterpret_cast<int4*>(d.dst + z * d.dst_pz + y * d.dst_py);
        for (int c = lane; c < nch; c += 32) dst[c] = src[c];
    }
}

}  // namespace

cudaError_t launch_stage(const StageLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    int64_t max_rows = 0;
    for (int i = 0; i < L.n; ++i) {
        const int64_t r = (int64_t)L.d[i].ny * L.d[i].nz;
        if (r > max_rows) max_rows = r;
    }
    int64_t g = (max_rows + kWarps - 1) / kWarps;
    int gx = (int)(g > 4096 ? 4096 : g);
    if (gx < 1) gx = 1;
    stage_kernel<<<dim3(gx, L.n), 32 * kWarps, 0, s>>>(L);
    return cudaGetLastError();
}

}  // namespace lfg

namespace lfg {
cudaError_t warm_stage() {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, stage_kernel);
}
}  // namespace lfg
