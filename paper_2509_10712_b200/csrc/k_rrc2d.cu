// k_rrc2d.cu -- K3: fused obj_det / ImageNet chain for a launch group of images.
//
// Realises Resize (RandomResizedCrop, bilinear, align_corners=False,
// antialias=False), RandomHorizontalFlip, ToTensor and Normalize
// (proj/src/workloads.cpp:151-156): u8 HWC crop box -> f32 CHW [3, oh, ow].
//
// Source coordinates and weights are computed in fp64 with the same
// (non-contracted) operations as the oracle (PyTorch
// area_pixel_compute_source_index), then rounded to fp32 for the blend, so
// tap indices always agree with the oracle and only the fp32 arithmetic
// differs (~1e-7 relative).
//
// Mapping: grid (ceil(oh / kRows), n_samples), 256 threads.  A CTA owns kRows
// output rows of one sample:
//   1. the source rows those outputs touch (<= (kRows-1)*h/oh + 3) are copied
//      from HBM into shared memory with aligned 16-byte loads; row taps are
//      computed once per CTA;
//   2. one thread per output column reads its two horizontal taps (6 bytes
//      per source row) with three 32-bit shared loads and two funnel shifts,
//      converts bytes to floats with PRMT into the 2^23 mantissa (exact), and
//      writes 3 coalesced f32 planes with streaming stores.
// The per-launch dynamic shared memory is the largest row window of the group
// (computed on the host with the same formula); crops whose window exceeds the
// budget (sources taller than ~2.6x oh) fall back to direct L2 byte loads.
#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kRows = 8;
constexpr int kThreads = 256;
constexpr int kMaxSmem = 64 * 1024;

// PyTorch area_pixel_compute_source_index (align_corners=False, linear), fp64,
// written with _rn intrinsics so nvcc cannot contract it into an FMA.
__device__ __forceinline__ void src_index(int dst, int in, double scale, int& i0, int& i1,
                                          float& l0, float& l1) {
    double src = __dadd_rn(__dmul_rn(__dadd_rn((double)dst, 0.5), scale), -0.5);
    if (src < 0.0) src = 0.0;
    int a = (int)floor(src);
    if (a > in - 1) a = in - 1;
    i0 = a;
    i1 = a < in - 1 ? a + 1 : a;
    const double w1 = __dadd_rn(src, -(double)a);
    l1 = (float)w1;
    l0 = (float)__dadd_rn(1.0, -w1);
}

__device__ __forceinline__ const uint8_t* row_ptr(const RrcDesc& d, int y) {
    return d.src + (int64_t)y * d.pitch + ((d.sk0 + y * d.sky) & 15);
}

// exact u8 -> f32: place byte k of w in the low mantissa of 2^23, subtract 2^23
__device__ __forceinline__ float ubyte(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7650u | (uint32_t)k)) - 8388608.0f;
}

__global__ void __launch_bounds__(kThreads)
rrc2d_kernel(const __grid_constant__ RrcLaunch L, int smem_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int row_off[64];           // byte offset of each staged row's first pixel
    __shared__ int ty[kRows][2];
    __shared__ float wy[kRows][2];
    const RrcDesc& d = L.d[blockIdx.y];
    const int oh = L.oh, ow = L.ow;
    const int y_begin = blockIdx.x * kRows;
    const int y_end = min(y_begin + kRows, oh);
    const double sy = __ddiv_rn((double)d.h, (double)oh);
    if (threadIdx.x < y_end - y_begin) {
        int a, b;
        float l0, l1;
        src_index(y_begin + threadIdx.x, d.h, sy, a, b, l0, l1);
        ty[threadIdx.x][0] = a;
        ty[threadIdx.x][1] = b;
        wy[threadIdx.x][0] = l0;
        wy[threadIdx.x][1] = l1;
    }
    __syncthreads();
    const int ylo = ty[0][0];
    const int nrows = ty[y_end - y_begin - 1][1] - ylo + 1;
    const int row_bytes = d.w * 3;
    const int spitch = ((row_bytes + 30) >> 4) << 4;        // 16-B chunks + alignment phase
    const bool staged = nrows <= 64 && nrows * spitch <= smem_bytes;

    // 1. stage the touched source rows (aligned 16-byte superset of each row)
    if (staged) {
        const int chunks = spitch >> 4;
        for (int i = threadIdx.x; i < nrows * chunks; i += kThreads) {
            const int r = i / chunks, c = i - r * chunks;
            const uintptr_t s = reinterpret_cast<uintptr_t>(row_ptr(d, ylo + r));
            const uintptr_t a = s & ~uintptr_t(15);
            const uintptr_t e = (s + row_bytes + 15) & ~uintptr_t(15);
            if (a + 16u * c < e) {
                *reinterpret_cast<int4*>(smem + r * spitch + 16 * c) =
                    __ldg(reinterpret_cast<const int4*>(a) + c);
            }
            if (c == 0) row_off[r] = r * spitch + (int)(s & 15);
        }
        __syncthreads();
    }

    const int x = threadIdx.x;
    if (x >= ow) return;
    int x0, x1;
    float lx0, lx1;
    src_index(x, d.w, __ddiv_rn((double)d.w, (double)ow), x0, x1, lx0, lx1);
    const bool edge = x1 == x0;                                     // right border: tap 1 = tap 0
    const int xo = d.flip ? ow - 1 - x : x;                         // RandomHorizontalFlip
    const int64_t plane = (int64_t)oh * ow;
    const float a0 = L.a[0], a1 = L.a[1], a2 = L.a[2];
    const float b0 = L.b[0], b1 = L.b[1], b2 = L.b[2];

    // horizontal blend of one source row at this thread's column (3 channels)
    auto hrow = [&](int y, float h[3]) {
        float p[6];   // R0 G0 B0 R1 G1 B1
        if (staged) {
            const int off = row_off[y - ylo] + 3 * x0;
            const uint32_t* w = reinterpret_cast<const uint32_t*>(smem + (off & ~3));
            const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
            const uint32_t sh = (off & 3) * 8;
            const uint32_t lo = __funnelshift_r(w0, w1, sh);        // bytes 0..3
            const uint32_t hi = __funnelshift_r(w1, w2, sh);        // bytes 4..7
            p[0] = ubyte(lo, 0);
            p[1] = ubyte(lo, 1);
            p[2] = ubyte(lo, 2);
            p[3] = edge ? p[0] : ubyte(lo, 3);
            p[4] = edge ? p[1] : ubyte(hi, 0);
            p[5] = edge ? p[2] : ubyte(hi, 1);
        } else {
            const uint8_t* row = row_ptr(d, y);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                p[c] = __ldg(row + 3 * x0 + c);
                p[3 + c] = __ldg(row + 3 * x1 + c);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) h[c] = fmaf(lx0, p[c], lx1 * p[3 + c]);
    };
    // Two-entry cache of blended rows: consecutive output rows share source
    // rows (y0(j) == y1(j-1) when downscaling < 2x, y0(j) == y0(j-1) when
    // upscaling).  Row indices are CTA-uniform, so the branches do not diverge.
    int ra = -1, rb = -1;
    float ha[3] = {0, 0, 0}, hb[3] = {0, 0, 0};
    for (int j = 0; j < y_end - y_begin; ++j) {
        const int y0 = ty[j][0], y1 = ty[j][1];
        const float ly0 = wy[j][0], ly1 = wy[j][1];
        float top[3], bot[3];
        if (y0 == rb) {
            top[0] = hb[0]; top[1] = hb[1]; top[2] = hb[2];
        } else if (y0 == ra) {
            top[0] = ha[0]; top[1] = ha[1]; top[2] = ha[2];
        } else {
            hrow(y0, top);
        }
        if (y1 == y0) {
            bot[0] = top[0]; bot[1] = top[1]; bot[2] = top[2];
        } else if (y1 == rb) {
            bot[0] = hb[0]; bot[1] = hb[1]; bot[2] = hb[2];
        } else {
            hrow(y1, bot);
        }
        ra = y0;
        ha[0] = top[0]; ha[1] = top[1]; ha[2] = top[2];
        rb = y1;
        hb[0] = bot[0]; hb[1] = bot[1]; hb[2] = bot[2];
        float out[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) out[c] = fmaf(ly0, top[c], ly1 * bot[c]);   // Resize (bilinear)
        float* o = d.out + (int64_t)(y_begin + j) * ow + xo;
        __stcs(o, fmaf(out[0], a0, b0));                           // ToTensor + Normalize
        __stcs(o + plane, fmaf(out[1], a1, b1));
        __stcs(o + 2 * plane, fmaf(out[2], a2, b2));
    }
}

}  // namespace

// Shared-memory window a group needs: max over its samples of
// (touched rows of one CTA) x (padded row bytes), bounded by kMaxSmem.
int rrc2d_smem_bytes(const RrcLaunch& L) {
    int need = 0;
    for (int i = 0; i < L.n; ++i) {
        const RrcDesc& d = L.d[i];
        const int rows = (int)((double)(kRows - 1) * d.h / L.oh) + 4;
        const int spitch = ((d.w * 3 + 30) >> 4) << 4;
        need = max(need, min(rows, 64) * spitch);
    }
    return min(need, kMaxSmem);
}

cudaError_t launch_rrc2d(const RrcLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    if (L.ow > kThreads) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(rrc2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kMaxSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int smem = rrc2d_smem_bytes(L);
    dim3 grid((L.oh + kRows - 1) / kRows, L.n);
    rrc2d_kernel<<<grid, kThreads, smem, s>>>(L, smem);
    return cudaGetLastError();
}

cudaError_t warm_rrc2d() {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, rrc2d_kernel);
}

}  // namespace lfg
