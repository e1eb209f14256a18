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
constexpr int kIlp = 4;   // 16-B chunks in flight per lane (all loads issued before the stores)

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
            v[k] = reinterpret_cast<const int4*>(a)[c];
            dst[k] = reinterpret_cast<int4*>(d.dst + z * d.dst_pz + y * d.dst_py) + c;
        }
#pragma unroll
        for (int k = 0; k < kIlp; ++k)
            if (dst[k] != nullptr) *dst[k] = v[k];
    }
}

}  // namespace

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
