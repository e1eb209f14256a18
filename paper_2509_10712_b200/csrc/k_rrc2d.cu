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
// Mapping: grid (ceil(oh / kRows), n_samples), 128 threads.  A CTA owns kRows
// output rows of one sample:
//   1. the source rows those outputs touch (<= (kRows-1)*h/oh + 4) land in
//      shared memory by cp.async.bulk (one bulk copy per row, the 16-B aligned
//      superset, all on one mbarrier) while the threads compute their taps; the
//      row schedule (which source row to blend into which register, vertical
//      weights with Normalize's scale folded in) is built once per CTA;
//   2. each thread owns two ADJACENT output columns, carried as the two lanes of
//      float2 values through Blackwell's paired FP32 instructions (FFMA2 / FMUL2
//      / FADD2); it reads each horizontal tap pair (6 bytes) with three 32-bit
//      shared loads and two funnel shifts, converts bytes with PRMT into the 2^23
//      mantissa (exact), blends each source row once into the register of its
//      parity (even / odd: the taps y0, y0 + 1 never collide, so no register
//      moves), and writes 3 planes with 8-byte streaming stores (RandomHorizontal
//      Flip swaps the lanes' roles, not the data).
// The per-launch dynamic shared memory is the largest row window of the group
// (computed on the host with the same formula); crops whose window exceeds the
// budget (sources taller than ~2.6x oh) fall back to direct L2 byte loads.
#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

constexpr int kRows = 8;        // 16 measured slower (larger windows cut occupancy)
constexpr int kThreads = 128;
constexpr int kMaxSmem = 64 * 1024;
// load6 reads 12 bytes from (off & ~3): up to 5 bytes past the last staged
// row's slot, so every window is allocated with this much slack behind it
constexpr int kSmemSlack = 16;

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

// an image's descriptor, unpacked once per CTA
struct RrcView {
    const uint8_t* src;
    float* out;
    int pitch, h, w, sk0, sky, flip, slot;
};
__device__ __forceinline__ RrcView unpack(const RrcLaunch& L, int i) {
    const RrcDesc p = L.d[i];
    RrcView v;
    v.src = rrc_src(p);
    v.sk0 = rrc_sk0(p);
    v.sky = rrc_sky(p);
    v.pitch = rrc_pitch(p);
    v.h = rrc_h(p);
    v.w = rrc_w(p);
    v.flip = rrc_flip(p);
    v.out = L.out_tab[rrc_buf(p)] + (int64_t)rrc_pos(p) * L.out_stride;
    v.slot = L.slot_base + i;
    return v;
}

__device__ __forceinline__ const uint8_t* row_ptr(const RrcView& d, int y) {
    return d.src + (int64_t)y * d.pitch + ((d.sk0 + y * d.sky) & 15);
}

// byte offset of staged row y's first pixel: the row sits at (y - ylo) * spitch
// with its 16-byte alignment phase preserved (only the low 4 address bits matter)
__device__ __forceinline__ int staged_off(const RrcView& d, int y, int ylo, int spitch) {
    const uint32_t lo = (uint32_t)reinterpret_cast<uintptr_t>(d.src) + (uint32_t)y * (uint32_t)d.pitch +
                        (uint32_t)((d.sk0 + y * d.sky) & 15);
    return (y - ylo) * spitch + (int)(lo & 15u);
}

// exact u8 -> f32: place byte k of w in the low mantissa of 2^23, subtract 2^23
__device__ __forceinline__ float ubyte(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7650u | (uint32_t)k)) - 8388608.0f;
}

// The two output columns a thread owns (2t, 2t + 1) travel as the .x / .y
// lanes of float2 values, so the blend runs on Blackwell's paired FP32 units
// (FFMA2 / FMUL2 / FADD2: two IEEE fp32 results per instruction, each rounded
// exactly like fmaf / fmul / fadd).
struct ColPair {
    int off_a, off_b;       // byte offset of tap 0 within a source row (3 * x0)
    int x0_a, x0_b;         // (fallback path only)
    float2 w0, w1;          // tap weights; at the right border tap 1 aliases tap 0,
                            // folded as w0 = l0 + l1, w1 = 0
};

// bytes k of (wa, wb) -> exact (float, float)
__device__ __forceinline__ float2 ubyte2(uint32_t wa, uint32_t wb, int k) {
    const float2 m = make_float2(__uint_as_float(__byte_perm(wa, 0x4B000000u, 0x7650u | (uint32_t)k)),
                                 __uint_as_float(__byte_perm(wb, 0x4B000000u, 0x7650u | (uint32_t)k)));
    return __fadd2_rn(m, make_float2(-8388608.0f, -8388608.0f));
}

__device__ __forceinline__ void load6(const uint8_t* smem, int off, uint32_t& lo, uint32_t& hi) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(smem + (off & ~3));
    const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
    const uint32_t sh = (off & 3) * 8;
    lo = __funnelshift_r(w0, w1, sh);    // bytes 0..3: R0 G0 B0 R1
    hi = __funnelshift_r(w1, w2, sh);    // bytes 4..7: G1 B1 . .
}

__device__ __forceinline__ void blend_row(const uint8_t* smem, int row_off, const ColPair& c, float2 h[3]) {
    uint32_t la, ha, lb, hb;
    load6(smem, row_off + c.off_a, la, ha);
    load6(smem, row_off + c.off_b, lb, hb);
    h[0] = __ffma2_rn(c.w0, ubyte2(la, lb, 0), __fmul2_rn(c.w1, ubyte2(la, lb, 3)));
    h[1] = __ffma2_rn(c.w0, ubyte2(la, lb, 1), __fmul2_rn(c.w1, ubyte2(ha, hb, 0)));
    h[2] = __ffma2_rn(c.w0, ubyte2(la, lb, 2), __fmul2_rn(c.w1, ubyte2(ha, hb, 1)));
}

__device__ __forceinline__ void blend_row_l2(const RrcView& d, int y, const ColPair& c, float2 h[3]) {
    const uint8_t* row = row_ptr(d, y);
    const int x1a = min(c.x0_a + 1, d.w - 1), x1b = min(c.x0_b + 1, d.w - 1);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float2 p0 = make_float2(__ldg(row + 3 * c.x0_a + k), __ldg(row + 3 * c.x0_b + k));
        const float2 p1 = make_float2(__ldg(row + 3 * x1a + k), __ldg(row + 3 * x1b + k));
        h[k] = __ffma2_rn(c.w0, p0, __fmul2_rn(c.w1, p1));
    }
}

// the row loop of one CTA (defined below the kernel)
__device__ __forceinline__ void blend_rows(const RrcLaunch& L, const RrcView& d, const ColPair& cp, int y_begin,
                                           int n_rows_out, bool staged, int xa, const uint8_t* smem,
                                           uint64_t* stage_bar, const int2* sched_rows,
                                           const float (*sched_w)[6]);

__global__ void __launch_bounds__(kThreads, 12)   // 40 registers (one 8-B spill): shared memory, not registers, sets the CTAs / SM
rrc2d_kernel(const __grid_constant__ RrcLaunch L, int smem_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t stage_bar;   // staged rows landed
    // Per output row j: which source rows to blend into the two row registers
    // (row r always lives in register r & 1 -- the two taps y0, y0 + 1 of a
    // row never collide) and the vertical weights with Normalize's scale folded
    // in: out_c = wE_c * E_c + (wO_c * O_c + b_c).
    __shared__ int2 sched_rows[kRows];            // {even row, odd row} to blend (-1: kept) as a
                                                  // staged byte offset (or a row index, unstaged)
    __shared__ float sched_w[kRows][6];           // {wE * a_c (c = 0..2), wO * a_c}
    __shared__ int yspan[2];                      // [0]: the block's rows are staged
    const RrcView d = unpack(L, blockIdx.y);
    const int oh = L.oh, ow = L.ow;
    const int y_begin = blockIdx.x * kRows;
    const int n_rows_out = min(kRows, oh - y_begin);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row_bytes = d.w * 3;
    const int spitch = ((row_bytes + 30) >> 4) << 4;        // 16-B chunks + alignment phase
    // Warp 0, lane j < n_rows_out: output row j's vertical taps.  The block's source
    // row span (first tap of row 0 .. last tap of the last row) is known after one
    // shuffle, so the bulk copies go out before the rest of the schedule is built;
    // the other warps derive their column taps meanwhile.
    bool staged = false;
    int ylo = 0;
    if (warp == 0) {
        const int j = lane;
        const double sy = __ddiv_rn((double)d.h, (double)oh);   // IEEE: as the oracle / host
        int y0 = 0, y1 = 0;
        float l0 = 0.f, l1 = 0.f;
        if (j < n_rows_out) src_index(y_begin + j, d.h, sy, y0, y1, l0, l1);
        ylo = __shfl_sync(0xffffffffu, y0, 0);
        const int yhi = __shfl_sync(0xffffffffu, y1, n_rows_out - 1);
        const int nrows = yhi - ylo + 1;
        staged = nrows * spitch + kSmemSlack <= smem_bytes;
        if (staged) {
            if (lane == 0) {
                mbar_init(&stage_bar, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncwarp();
            // stage the touched source rows (aligned 16-byte superset of each row) with
            // bulk async copies, one per row (a lane per row), all on one mbarrier.  The
            // window's first chunk and last chunk are copied byte by byte instead when they
            // are partial: the superset there may reach past the caller's buffer.
            auto span = [&](int r, uintptr_t& sa, uintptr_t& b0, uintptr_t& b1) {
                sa = reinterpret_cast<uintptr_t>(row_ptr(d, ylo + r));
                const uintptr_t al = sa & ~uintptr_t(15), ae = (sa + row_bytes + 15) & ~uintptr_t(15);
                b0 = (r == 0 && (sa & 15) != 0) ? al + 16 : al;
                b1 = (r == nrows - 1 && ((sa + row_bytes) & 15) != 0) ? ae - 16 : ae;
                if (b1 < b0) b1 = b0;
            };
            int bytes = 0;
            for (int r = lane; r < nrows; r += 32) {
                uintptr_t sa, b0, b1;
                span(r, sa, b0, b1);
                bytes += (int)(b1 - b0);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
            if (lane == 0) mbar_expect_tx(&stage_bar, (uint32_t)bytes);
            __syncwarp();
            for (int r = lane; r < nrows; r += 32) {
                uintptr_t sa, b0, b1;
                span(r, sa, b0, b1);
                const uintptr_t al = sa & ~uintptr_t(15);
                uint8_t* srow = smem + r * spitch;
                if (b1 > b0) bulk_g2s(srow + (b0 - al), reinterpret_cast<const void*>(b0), (uint32_t)(b1 - b0), &stage_bar);
            }
            {
                // the exact parts, one byte per lane (one round trip): lanes 0-15 the
                // window's first chunk [sa, b0), lanes 16-31 its last chunk [b1, end)
                // (visible to the other warps after the CTA barrier below)
                const int r = lane < 16 ? 0 : nrows - 1;
                uintptr_t sa, b0, b1;
                span(r, sa, b0, b1);
                const uintptr_t al = sa & ~uintptr_t(15), end = sa + row_bytes;
                const uintptr_t x = lane < 16 ? al + lane : (((end - 1) & ~uintptr_t(15)) + (lane - 16));
                const bool in = x >= sa && x < end && (lane < 16 ? x < b0 : x >= b1);
                if (in) smem[r * spitch + (x - al)] = *reinterpret_cast<const uint8_t*>(x);
            }
        }
        // the previous output row's taps (row j - 1 is lane j - 1)
        int p0 = __shfl_up_sync(0xffffffffu, y0, 1), p1 = __shfl_up_sync(0xffffffffu, y1, 1);
        if (j == 0) p0 = p1 = -1;
        if (j < n_rows_out) {
            // a row is already in its register iff the previous output row used it
            // (rows are non-decreasing and adjacent taps differ by at most one)
            const bool new0 = y0 != p0 && y0 != p1;
            const bool new1 = y1 != y0 && y1 != p0 && y1 != p1;
            const bool odd0 = (y0 & 1) != 0;   // y1 (if distinct) has the other parity
            int ld_e = odd0 ? (new1 ? y1 : -1) : (new0 ? y0 : -1);
            int ld_o = odd0 ? (new0 ? y0 : -1) : (new1 ? y1 : -1);
            if (staged) {   // resolve rows to their byte offsets in the staged window once, here
                if (ld_e >= 0) ld_e = staged_off(d, ld_e, ylo, spitch);
                if (ld_o >= 0) ld_o = staged_off(d, ld_o, ylo, spitch);
            }
            float w_e, w_o;
            if (y1 == y0) {
                w_e = odd0 ? 0.f : l0 + l1;
                w_o = odd0 ? l0 + l1 : 0.f;
            } else {
                w_e = odd0 ? l1 : l0;
                w_o = odd0 ? l0 : l1;
            }
            sched_rows[j] = make_int2(ld_e, ld_o);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                sched_w[j][c] = w_e * L.a[c];
                sched_w[j][3 + c] = w_o * L.a[c];
            }
        }
        if (lane == 0) yspan[0] = staged ? 1 : 0;
    }

    const int xa = 2 * threadIdx.x;                         // columns xa, xa + 1 (ow is even)
    ColPair cp;
    if (xa < ow) {
        const double sx = __ddiv_rn((double)d.w, (double)ow);
        int x1a, x1b;
        float l0a, l1a, l0b, l1b;
        src_index(xa, d.w, sx, cp.x0_a, x1a, l0a, l1a);
        src_index(xa + 1, d.w, sx, cp.x0_b, x1b, l0b, l1b);
        cp.off_a = 3 * cp.x0_a;
        cp.off_b = 3 * cp.x0_b;
        // right border (tap 1 == tap 0): fold both weights onto tap 0
        cp.w0 = make_float2(x1a == cp.x0_a ? l0a + l1a : l0a, x1b == cp.x0_b ? l0b + l1b : l0b);
        cp.w1 = make_float2(x1a == cp.x0_a ? 0.0f : l1a, x1b == cp.x0_b ? 0.0f : l1b);
        // RandomHorizontalFlip: the pair lands at (ow-2-xa, ow-1-xa), so the
        // lanes swap roles (.x = column xa + 1) and every store stays a plain float2
        if (d.flip) {
            const int t0 = cp.off_a, t1 = cp.x0_a;
            cp.off_a = cp.off_b, cp.x0_a = cp.x0_b;
            cp.off_b = t0, cp.x0_b = t1;
            cp.w0 = make_float2(cp.w0.y, cp.w0.x);
            cp.w1 = make_float2(cp.w1.y, cp.w1.x);
        }
    }
    __syncthreads();   // schedule visible; the mbarrier was initialised before the copies
    staged = yspan[0] != 0;
    if (xa < ow) blend_rows(L, d, cp, y_begin, n_rows_out, staged, xa, smem, &stage_bar, sched_rows, sched_w);
    if (L.st.cnt != nullptr) {   // this CTA's rows of the sample are written
        __syncthreads();
        if (threadIdx.x == 0) sample_part_done(L.st.cnt + d.slot, L.st.stamp + d.slot, gridDim.x);
    }
}

__device__ __forceinline__ void blend_rows(const RrcLaunch& L, const RrcView& d, const ColPair& cp, int y_begin,
                                           int n_rows_out, bool staged, int xa, const uint8_t* smem,
                                           uint64_t* stage_bar, const int2* sched_rows,
                                           const float (*sched_w)[6]) {
    const int oh = L.oh, ow = L.ow;
    const int64_t plane = (int64_t)oh * ow;
    float2* o = reinterpret_cast<float2*>(d.out + (int64_t)y_begin * ow + (d.flip ? ow - 2 - xa : xa));
    const int ow2 = ow >> 1;
    const int64_t plane2 = plane >> 1;
    const float2 nb[3] = {make_float2(L.b[0], L.b[0]), make_float2(L.b[1], L.b[1]), make_float2(L.b[2], L.b[2])};

    // Horizontally blended source rows, even rows in E, odd rows in O (no
    // register moves: each row is blended once, straight into its register).
    float2 E[3], O[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) E[k] = O[k] = make_float2(0.f, 0.f);
    if (staged) mbar_wait(stage_bar, 0);
    for (int j = 0; j < n_rows_out; ++j) {
        const int2 lr = sched_rows[j];   // CTA-uniform: no divergence
        if (lr.x >= 0) {
            if (staged) blend_row(smem, lr.x, cp, E);
            else blend_row_l2(d, lr.x, cp, E);
        }
        if (lr.y >= 0) {
            if (staged) blend_row(smem, lr.y, cp, O);
            else blend_row_l2(d, lr.y, cp, O);
        }
        // Resize (vertical blend) + ToTensor + Normalize; 8-byte streaming stores
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float we = sched_w[j][k], wo = sched_w[j][3 + k];
            __stcs(o + k * plane2,
                   __ffma2_rn(make_float2(we, we), E[k], __ffma2_rn(make_float2(wo, wo), O[k], nb[k])));
        }
        o += ow2;
    }
}

}  // namespace

// Shared-memory window a group needs: max over its samples of
// (touched rows of one CTA) x (padded row bytes), bounded by kMaxSmem.
int rrc2d_smem_bytes(const RrcLaunch& L) {
    int need = 0;
    for (int i = 0; i < L.n; ++i) {
        const RrcDesc& d = L.d[i];
        const int rows = (int)((double)(kRows - 1) * rrc_h(d) / L.oh) + 4;
        const int spitch = ((rrc_w(d) * 3 + 30) >> 4) << 4;
        need = max(need, rows * spitch);
    }
    return min(need, kMaxSmem) + kSmemSlack;
}

cudaError_t launch_rrc2d(const RrcLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    if (L.ow > 2 * kThreads || (L.ow & 1)) return cudaErrorInvalidValue;
    // (the raised shared-memory limit is set per device by warm_rrc2d at context creation)
    const int smem = rrc2d_smem_bytes(L);
    dim3 grid((L.oh + kRows - 1) / kRows, L.n);
    rrc2d_kernel<<<grid, kThreads, smem, s>>>(L, smem);
    return cudaGetLastError();
}

// Runs on every Context's device at creation: the dynamic shared-memory limit
// is a per-device (per CUDA context) attribute of the kernel.
cudaError_t warm_rrc2d() {
    cudaError_t e = cudaFuncSetAttribute(rrc2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kMaxSmem + kSmemSlack);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, rrc2d_kernel);
}

}  // namespace lfg
