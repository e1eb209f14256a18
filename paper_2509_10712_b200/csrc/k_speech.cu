// k_speech.cu -- K8/K9/K10: FilterBank (STFT power -> slaney mel -> log) with
// SpecAugment and FrameSplicing fused, on the 5th-gen tensor cores; and K11,
// the PermuteAudio + Pad collation of a speech batch.
//
// Reference chain: Pad, SpecAugment, FilterBank, FrameSplicing, PermuteAudio
// (proj/src/workloads.cpp:103-111).  Semantics: oracle/lf_oracle.c lfo_applysp.
//
// K8/K9 as a GEMM.  With the periodic Hann window (320 taps centred in the
// 512-point frame) folded into the basis, the STFT of frame f is
//     X[f, k] = sum_{j<320} x[(f-1)*160 + j] * w[j] * exp(-2 pi i k (j+96) / 512)
// i.e. C[frames x 512] = A[frames x 320] . B[320 x 512] with B's columns the
// cos / sin rows for bins 0..255 (bin 256, Nyquist, is a signed sum done on the
// CUDA cores while A is built).  fp32 accuracy on TF32 tensor cores by the
// 3xTF32 split: A = Ah + Al, B = Bh + Bl, C ~ Al.Bh + Ah.Bl + Ah.Bh.
//
// Per CTA (128 threads, 1 per SM): 126 frames of one utterance (M = 128 rows,
// a multiple of 3 frames so FrameSplicing never crosses CTAs).  The full
// 128 x 512 fp32 accumulator lives in TMEM (all 512 columns) as two
// M128 x N256 tcgen05.mma.kind::tf32 tiles.  K = 320 in 20 chunks of 16 taps,
// double-buffered in shared memory: the constant B chunk (64 KB, hi+lo, both
// N halves) arrives by cp.async.bulk on an mbarrier while the threads build
// the A chunk (frames read from the waveform with reflect padding, split into
// tf32 hi/lo); one elected thread issues the MMAs and commits them to the
// stage's mbarrier.  Operands use the 32-byte-swizzled K-major canonical layout
// (one 32-B row per frame / basis column = one K=8 tf32 step; the swizzle keeps
// the tensor core's operand reads bank-conflict free -- the unswizzled layout
// measured ~5x slower).
//
// Epilogue (all 4 warps, thread = frame = TMEM lane): tcgen05.ld 16 columns of
// cos and sin at a time -> power -> the slaney mel filterbank as a streaming
// reduction (each FFT bin feeds at most two adjacent triangular filters; the
// bank is 2.4% dense, so it stays on the CUDA cores instead of a mostly-zero
// GEMM) -> shared memory -> log(x + eps), SpecAugment masks, stack-3 splice,
// coalesced time-major stores into the sample's output slot.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "device_common.cuh"
#include "kernels.h"
#include "mel_table.h"

namespace lfg {

namespace {

constexpr int kTaps = 320;            // Hann window length (non-zero taps of the 512 frame)
constexpr int kWinOff = 96;           // (512 - 320) / 2
constexpr int kHop = 160;
constexpr int kNfft = 512;
constexpr int kBins = 256;            // bins 0..255 on the tensor cores, 256 on the CUDA cores
constexpr int kMels = 80;
constexpr int kRowsM = 128;           // MMA M
constexpr int kFramesPerCta = 126;    // multiple of 3 (FrameSplicing stack)
constexpr int kKChunk = 8;            // taps per pipeline stage = one MMA K-step
constexpr int kChunks = kTaps / kKChunk;          // 40
constexpr int kStages = 2;             // x 2 CTAs per SM (see the kernel comment)
constexpr int kABytesStep = kRowsM * 32;          // one K=8 step of A (one part): 4 KB
constexpr int kAPartBytes = (kKChunk / 8) * kABytesStep;
constexpr int kBBlock = 256 * 32;                 // one K=8 step, one N half, one part: 8 KB
constexpr int kBStageBytes = (kKChunk / 8) * 2 * 2 * kBBlock;   // 32 KB
constexpr int kStageBytes = 2 * kAPartBytes + kBStageBytes;     // 40 KB
constexpr int kSmemBytes = kStages * kStageBytes + 1024;        // + barriers
constexpr int kMelPitch = kMels + 1;
constexpr int kThreads = 320;         // warp 0 producer, warp 1 MMA, warps 2-9 A builders (taps 0-3 /
                                      // 4-7 of each K step) + epilogue (bins 128..255 / 0..127)

// instruction descriptor: D f32, A/B tf32, K-major both, N = 256, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

__constant__ float c_win_nyq[kTaps];  // w[j] * (-1)^(j + 96): the Nyquist bin's real coefficients
__constant__ int c_mel_m[kBins + 1];  // lower filter index fed by bin k (-1: none)
__constant__ float c_mel_wa[kBins + 1], c_mel_wb[kBins + 1];   // weights into m and m+1

// ------------------------------------------------------------------ PTX helpers
// (smem_u32 / mbar_* / bulk_g2s live in device_common.cuh)
__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    // K-major, 32-byte swizzle: start>>4 [0,14), LBO>>4 = 1 [16,30), SBO>>4 = 256 B [32,46),
    // version 1 [46,48), layout SWIZZLE_32B = 6 [61,64).  Rows are 32 B (= one K=8 tf32
    // step); the 16-B half index is XORed with address bit 7 (row bit 2).
    return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) |
           (1ull << 46) | (6ull << 61);
}
// byte offset of 16-B half c of row (or column) r in a 32-B-swizzled K-major tile
__host__ __device__ __forceinline__ int sw32_off(int r, int c) { return r * 32 + ((c ^ ((r >> 2) & 1)) << 4); }
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float v[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
        "[%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void epilogue_sync() {   // the 8 epilogue warps (2..9) only
    asm volatile("bar.sync 1, 256;" ::: "memory");
}

// ------------------------------------------------------------------ the kernel
// Two CTAs per SM (2-stage rings of 40 KB, <= 102 registers): TMEM holds one
// 128x512 accumulator, so the second CTA waits in tcgen05.alloc while its builders
// already fill its ring, and gets the columns as soon as the first CTA's epilogue
// has read them -- its MMAs then run under the first CTA's log / SpecAugment /
// store tail (one CTA per SM with a 5-stage ring: 103 us per 64 utterances; this:
// 95 us).
// Warp-specialised: warp 0 streams the constant B chunks (cp.async.bulk) into a
// 2-deep ring, warp 1 issues the MMAs (one elected thread), warps 2-9 build the
// A chunks from the waveform (two warps per row quarter, one 16-B half of each
// row's K step each) and then run the epilogue.  Per stage: full_a (8 builder-warp
// arrivals), full_b (bulk-copy bytes), empty (tcgen05.commit).
__global__ void __launch_bounds__(kThreads, 2)
speech_kernel(const __grid_constant__ SpLaunch L, const char* __restrict__ basis) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ float nyq_s[kRowsM];                       // warps 6-9's half of the Nyquist sums
    // flattened grid: CTA -> (utterance, tile) through the tile prefix sums
    int u = 0;
    while (u + 1 < L.n && L.tile_start[u + 1] <= (int)blockIdx.x) ++u;
    const SpDesc& d = L.d[u];
    const int tile = blockIdx.x - L.tile_start[u];
    const int T = d.T;
    const int f0 = tile * kFramesPerCta;
    const uint32_t parts = (uint32_t)(L.tile_start[u + 1] - L.tile_start[u]);   // the utterance's CTAs
    if (f0 >= T) {                                        // CTA-uniform (never, with the launcher's tiling)
        if (L.st.cnt != nullptr && threadIdx.x == 0) sample_part_done(L.st.cnt + d.slot, L.st.stamp + d.slot, parts);
        return;
    }
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    uint64_t* full_a = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* full_b = full_a + kStages;
    uint64_t* empty = full_b + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full_a + s, 8);          // one arrival per builder warp
            mbar_init(full_b + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer: constant DFT basis chunks
        if (lane == 0) {
            for (int it = 0; it < kChunks; ++it) {
                const int s = it % kStages, use = it / kStages;
                if (use > 0) mbar_wait(empty + s, (use - 1) & 1);
                if (L.debug & 4) {
                    mbar_arrive(full_b + s);
                } else {
                    mbar_expect_tx(full_b + s, kBStageBytes);
                    bulk_g2s(smem + s * kStageBytes + 2 * kAPartBytes, basis + (size_t)it * kBStageBytes,
                             kBStageBytes, full_b + s);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            for (int it = 0; it < kChunks; ++it) {
                const int s = it % kStages, use = it / kStages;
                mbar_wait(full_b + s, use & 1);
                mbar_wait(full_a + s, use & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t a_hi = smem_u32(smem + s * kStageBytes), a_lo = a_hi + kAPartBytes;
                const uint32_t b0 = a_hi + 2 * kAPartBytes;
                const uint64_t dah = smem_desc(a_hi), dal = smem_desc(a_lo);
#pragma unroll
                for (int h = 0; h < 2 && !(L.debug & 2); ++h) {
                    const uint64_t dbh = smem_desc(b0 + (h * 2 + 0) * kBBlock);
                    const uint64_t dbl = smem_desc(b0 + (h * 2 + 1) * kBBlock);
                    const uint32_t acc = tmem + h * 256;
                    mma_tf32(acc, dal, dbh, it > 0 ? 1u : 0u);     // 3xTF32, small terms first
                    mma_tf32(acc, dah, dbl, 1u);
                    mma_tf32(acc, dah, dbh, 1u);
                }
                mma_commit(empty + s);
            }
            mma_commit(done);
        }
        __syncwarp();
    } else {
        // ---------------- A builders (warps 2-9), then the epilogue: one frame per thread,
        // thread row = TMEM lane (warp w may only read lanes 32*(w%4) .. +31)
        const int r = 32 * (warp & 3) + lane;
        const int f = f0 + r;
        const bool row_live = r < kFramesPerCta && f < T;
        const int64_t n0 = (int64_t)(f - 1) * kHop;       // first tap's sample index
        const bool interior = row_live && n0 >= 0 && n0 + kTaps <= d.L &&
                              ((reinterpret_cast<uintptr_t>(static_cast<const float*>(d.wav) + n0) & 15) == 0);
        float nyq = 0.0f;
        // All 8 warps build A: warps 2-5 taps 0-3 of every K step (16-B chunk 0 of
        // the row), warps 6-9 taps 4-7 (chunk 1), each into its own half of the
        // Nyquist bin's sum (combined in the epilogue).
        const int half = warp >= 6 ? 1 : 0;
        auto load = [&](int it, float x[4]) {
            if (interior) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(d.wav) + n0 + it * kKChunk + 4 * half));
                x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float v = 0.0f;
                    if (row_live) {
                        int64_t n = n0 + it * kKChunk + 4 * half + j;     // reflect padding
                        if (n < 0) n = -n;
                        if (n >= d.L) n = 2 * ((int64_t)d.L - 1) - n;
                        v = __ldg(static_cast<const float*>(d.wav) + n);
                    }
                    x[j] = v;
                }
            }
        };
        {
            float x[4];
            const bool skip_loads = (L.debug & 1) != 0;
            if (skip_loads) {
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = 0.001f * j;
            } else {
                load(0, x);
            }
            for (int it = 0; it < kChunks; ++it) {
                const int s = it % kStages, use = it / kStages;
                float xn[4];
                if (skip_loads) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) xn[j] = x[j];
                } else if (it + 1 < kChunks) {
                    load(it + 1, xn);                            // prefetch the next chunk's taps
                }
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    nyq = fmaf(x[j], c_win_nyq[it * kKChunk + 4 * half + j], nyq);
                    hi[j] = tf32_rna(x[j]);
                    lo[j] = tf32_rna(x[j] - __uint_as_float(hi[j]));
                }
                if (use > 0) {                                   // one poller per warp
                    if (lane == 0) mbar_wait(empty + s, (use - 1) & 1);
                    __syncwarp();
                }
                uint8_t* sa = smem + s * kStageBytes;
                // canonical K-major, 32-byte swizzle (see smem_desc)
                const int off = sw32_off(r, half);
                *reinterpret_cast<uint4*>(sa + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<uint4*>(sa + kAPartBytes + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to the tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive(full_a + s);
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = xn[j];
            }
        }
        if (half == 1) nyq_s[r] = nyq;   // read after the first epilogue barrier

        // ---------------- epilogue: power -> mel with the filter bank as compile-time
        // constants (mel_table.h: with the bin loops unrolled every filter index is a
        // constant -- 2 FMAs per bin with immediate weights, no loads, no branches).
        // Two warps per TMEM lane quarter split the bins: warps 6-9 bins 0..127
        // (filters 0..62), warps 2-5 bins 128..255 (filters 61..79); the filters
        // both halves feed are summed through shared memory, then both halves of a
        // row take 40 filters each for log + SpecAugment.
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        float* mel_s = reinterpret_cast<float*>(smem);    // the operand ring is free now
        // filters fed by both bin halves: [kHiMin, kLoMax] (bins 127 / 128 straddle them)
        constexpr int kLoMax = kMelM[127] + 1, kHiMin = kMelM[128], kOvl = kLoMax - kHiMin + 1;
        static_assert(kOvl >= 1 && kOvl <= 4, "shared filters between the bin halves");
        float* ovl_s = mel_s + kRowsM * kMelPitch;        // [row][kOvl]: the upper half's share
        const uint32_t lane_base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
        const bool low_bins = warp >= 6;
        float* row = mel_s + r * kMelPitch;
        auto half_bins = [&](auto H, float mel[kMels]) {
            constexpr int h = decltype(H)::value;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                float re[16], im[16];
                tmem_ld16(lane_base + h * 256 + 16 * b, re);
                tmem_ld16(lane_base + h * 256 + 128 + 16 * b, im);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int kk = h * 128 + 16 * b + i;
                    const float p = fmaf(re[i], re[i], im[i] * im[i]);
                    if (kMelM[kk] >= 0) mel[kMelM[kk]] = fmaf(kMelWa[kk], p, mel[kMelM[kk]]);
                    if (kMelM[kk] >= 0 && kMelM[kk] + 1 < kMels)
                        mel[kMelM[kk] + 1] = fmaf(kMelWb[kk], p, mel[kMelM[kk] + 1]);
                }
            }
        };
        {
            float mel[kMels];
#pragma unroll
            for (int m = 0; m < kMels; ++m) mel[m] = 0.0f;
            if (low_bins) {
                half_bins(std::integral_constant<int, 0>{}, mel);
#pragma unroll
                for (int m = 0; m <= kLoMax; ++m) row[m] = mel[m];
            } else {
                half_bins(std::integral_constant<int, 1>{}, mel);
#pragma unroll
                for (int m = kHiMin; m <= kLoMax; ++m) ovl_s[r * kOvl + (m - kHiMin)] = mel[m];
#pragma unroll
                for (int m = kLoMax + 1; m < kMels; ++m) row[m] = mel[m];
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        epilogue_sync();
        // Every TMEM read of this CTA is done: hand the 512 columns to the SM's other
        // CTA (blocked in tcgen05.alloc) so its MMAs run under this epilogue's tail.
        if (warp == 2) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        }
        // Nyquist bin (CUDA cores): its filter is the upper half's own (row[m], m > kLoMax)
        static_assert(kMelM[kBins] < 0 || kMelM[kBins] > kLoMax, "Nyquist filter owned by warps 2-5");
        if (kMelM[kBins] >= 0 && !low_bins) {
            const float x = nyq + nyq_s[r];
            row[kMelM[kBins]] = fmaf(kMelWa[kBins], x * x, row[kMelM[kBins]]);
        }
        // log + SpecAugment on this row's 40 filters; padding frames are zero
        {
            bool tmask = f >= T || r >= kFramesPerCta;
            for (int q = 0; q < L.n_tmask; ++q) tmask |= f >= d.t_lo[q] && f < d.t_lo[q] + d.t_w[q];
            const int fl0 = L.n_fmask > 0 ? d.f_lo[0] : 0, fh0 = L.n_fmask > 0 ? d.f_lo[0] + d.f_w[0] : 0;
            const int fl1 = L.n_fmask > 1 ? d.f_lo[1] : 0, fh1 = L.n_fmask > 1 ? d.f_lo[1] + d.f_w[1] : 0;
            const int m0 = low_bins ? 0 : kMels / 2;
#pragma unroll
            for (int mm = 0; mm < kMels / 2; ++mm) {
                const int m = m0 + mm;
                const float v = row[m] + ((m >= kHiMin && m <= kLoMax) ? ovl_s[r * kOvl + (m - kHiMin)] : 0.0f);
                const bool masked = tmask || (m >= fl0 && m < fh0) || (m >= fl1 && m < fh1);
                row[m] = masked ? 0.0f : logf(v + 5.9604644775390625e-8f);   // + 2^-24
            }
        }
        epilogue_sync();

        // FrameSplicing: spliced row t' is frames stack*t' .. stack*t'+stack-1, so
        // the CTA's output rows are one contiguous run of (frame, mel) values:
        // copy it out with 128-bit stores (256 epilogue threads)
        const int e = tid - 64;
        const int stack = L.stack;
        const int width = stack * kMels;
        const int row0 = f0 / stack;
        const int t_rows = (T + stack - 1) / stack;
        const int rows = min(kFramesPerCta / stack, t_rows - row0);
        float* out = d.out + (int64_t)row0 * width;
        for (int q = 4 * e; q < rows * width && !(L.debug & 64); q += 4 * 256) {
            const int fr = q / kMels, m = q - fr * kMels;   // 4 values of one frame (80 % 4 == 0)
            const float* src = mel_s + fr * kMelPitch + m;
            *reinterpret_cast<float4*>(out + q) = make_float4(src[0], src[1], src[2], src[3]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    // this CTA's spliced rows of the utterance are written
    if (L.st.cnt != nullptr && tid == 0) sample_part_done(L.st.cnt + d.slot, L.st.stamp + d.slot, parts);
}

// ------------------------------------------------------------------ K8'-K10' (default)
// The same FilterBank + SpecAugment + FrameSplicing as speech_kernel, with the STFT as a
// real 512-point FFT on the CUDA cores instead of a DFT GEMM: ~12 k FLOPs per frame
// instead of 2 x 320 x 512 x 3 tensor FLOPs (3xTF32), so the kernel is bound by issue and
// HBM rather than by the tensor pipe.  Per frame (one warp):
//   z_n = a_2n + i a_2n+1 (a = windowed taps, 160 non-zero of 256); Z = FFT256(z) as
//   256 = 8 x 32: lane l holds z[32 n1 + l] -> 8-point DFT over n1, twiddle W256^(l k1);
//   a shared-memory transpose gives lane (k1, b) = 4 k1 + b the values of lanes 4a + b ->
//   8-point DFT over a, twiddle W32^(b c); a 4-point DFT across the lane quad (two
//   shuffle stages) -> lane (k1, b') holds Z[k1 + 8 c + 64 bitrev2(b')], c = 0..7;
//   one shuffle per c fetches Z[256 - k]; X_k = E_k + W512^k O_k (E, O the even / odd
//   sample spectra), P_k = |X_k|^2 for k = 0..256 (X_256 = E_0 - O_0).
// Mel: each lane sums its filters' (bin, weight) lists from the warp's power row in
// shared memory (bank-spread, pw_at; the 16 widest filters two lanes apiece); then log(x + 2^-24), SpecAugment masks and the stack-3 splice layout
// (frame f's 80 values at out + 80 f) as the tensor-core kernel.  Index mapping and
// pairing are checked against numpy in tests (test_speech_* vs the oracle).
constexpr int kFftFrames = 96;                                   // per CTA (multiple of 3)
constexpr int kFftWarps = 8;
#ifndef LFG_FFT_DYN_ROUNDS
#define LFG_FFT_DYN_ROUNDS 4   // (build-time A/B) frame-deal rounds left to the dynamic tail (1..8 measured)
#endif
constexpr int kFftDynRounds = LFG_FFT_DYN_ROUNDS;
constexpr int kTrPitch = 36;                                     // transpose row pitch (float2)
// mel filters as dense taps: filter m = lane + 32 g reads kMelW[g] consecutive bins from
// mel_b0[m] (the slaney bank's widest filters per lane group: 3, 10, 18 bins)
constexpr int kMelW0 = 3, kMelW1 = 10, kMelW2 = 18;
// The warp's power row in shared memory, bank-spread: bin k lives at pw_at(k) = k + 40 (k / 64),
// so the split's stores (lanes (k1, b') write bins k1 + 8 c + 64 bitrev2(b'), 64 apart across
// b') fall in distinct banks; the 40-word gap after each 64-bin block repeats the next
// block's first 40 bins, so a filter's taps stay contiguous from pw_at(b0) (mel_b0 holds
// pw_at(b0); filters are at most 18 bins wide).  The Nyquist bin lives in block 3's gap.
constexpr int kPwGap = 40;
constexpr int kPwPitch = 4 * (64 + kPwGap);
__device__ __host__ __forceinline__ int pw_at(int k) { return k + kPwGap * (k >> 6); }

struct __align__(16) FftTables {
    float win[kTaps];                 // periodic Hann(320)
    float2 tw256[8 * 32];             // [k1][l] W256^(l k1)
    float2 tw32[8 * 4];               // [c][b] W32^(b c)
    float2 tw512[8 * 32];             // [c][lane (k1, b')] -i W512^k, k = k1 + 8 c + 64 bitrev2(b')
    int32_t mel_b0[kMels];            // pw_at(first bin of filter m's tap window): lo_m - s_m
    float mel_wd[kMelW2 * kMels];     // [tap][filter] weights / 4 over the window (0 outside the filter's span)
    int32_t mel_b2[32];               // the 16 widest filters per lane (filter 64 + (l & 15), half l >> 4):
                                      // half 0 at mel_b0, half 1 at mel_b0 + 9 - t (see the tables)
};

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }   // a * (-i)
// in-place 8-point DFT, natural order in and out
__device__ __forceinline__ void dft8(float2 x[8]) {
    constexpr float r = 0.70710678118654752f;
    // even / odd 4-point DFTs
    const float2 e0 = cadd(x[0], x[4]), e1 = csub(x[0], x[4]), e2 = cadd(x[2], x[6]), e3 = mul_mi(csub(x[2], x[6]));
    const float2 E0 = cadd(e0, e2), E2 = csub(e0, e2), E1 = cadd(e1, e3), E3 = csub(e1, e3);
    const float2 o0 = cadd(x[1], x[5]), o1 = csub(x[1], x[5]), o2 = cadd(x[3], x[7]), o3 = mul_mi(csub(x[3], x[7]));
    float2 O0 = cadd(o0, o2), O2 = csub(o0, o2), O1 = cadd(o1, o3), O3 = csub(o1, o3);
    O1 = make_float2(r * (O1.x + O1.y), r * (O1.y - O1.x));      // * W8^1 = (1 - i) / sqrt 2
    O2 = mul_mi(O2);                                               // * W8^2 = -i
    O3 = make_float2(r * (O3.y - O3.x), -r * (O3.x + O3.y));     // * W8^3 = -(1 + i) / sqrt 2
    x[0] = cadd(E0, O0);
    x[4] = csub(E0, O0);
    x[1] = cadd(E1, O1);
    x[5] = csub(E1, O1);
    x[2] = cadd(E2, O2);
    x[6] = csub(E2, O2);
    x[3] = cadd(E3, O3);
    x[7] = csub(E3, O3);
}
__device__ __forceinline__ float2 shfl2(float2 v, int src) {
    return make_float2(__shfl_sync(0xFFFFFFFFu, v.x, src), __shfl_sync(0xFFFFFFFFu, v.y, src));
}
__device__ __forceinline__ int bitrev2(int x) { return ((x & 1) << 1) | ((x >> 1) & 1); }
// two int16 PCM samples (low half first) -> (s0, s1) / 32768, exactly: flipping each sign
// bit maps s to s + 32768 in [0, 65535]; PRMT places it under 0x4B00'0000 (the float
// 2^23 + s + 32768); one paired FFMA removes the offset and scales by 2^-15
__device__ __forceinline__ float2 pcm_pair(uint32_t w) {
    w ^= 0x80008000u;
    const float2 m = make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7410u)),
                                 __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7432u)));
    constexpr float k = 1.0f / 32768.0f, off = -(8388608.0f + 32768.0f) / 32768.0f;
    return __ffma2_rn(m, make_float2(k, k), make_float2(off, off));
}

// Frames are dealt to warps round-robin over the launch's flattened frame space
// (L.tile_start holds per-utterance frame prefix sums for this kernel), so every SM
// works until the last few frames: no CTA-granular tail.  A frame's 320 taps are read
// straight from the waveform (L1 / L2: neighbouring frames, on neighbouring warps of
// the same CTA, share half of them); only the first frame of an utterance and the last
// ones need the reflect padding.
#ifndef LFG_FFT_REG_TW
#define LFG_FFT_REG_TW 0   // (build-time A/B) lane twiddles held in registers, 2 CTAs / SM
#endif
template <bool kPcm>   // int16 PCM waveforms (else f32): one instantiation each, no per-tap selects
__global__ void __launch_bounds__(32 * kFftWarps, LFG_FFT_REG_TW ? 2 : 3)
speech_fft_kernel(const __grid_constant__ SpLaunch L, const FftTables* __restrict__ g) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int ts[kMaxSp + 1];                      // the launch's frame prefix sums
    FftTables* tb = reinterpret_cast<FftTables*>(smem);
    float2* tr_all = reinterpret_cast<float2*>(smem + sizeof(FftTables));
    float* pw_all = reinterpret_cast<float*>(tr_all + kFftWarps * 8 * kTrPitch);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const float4* src = reinterpret_cast<const float4*>(g);
        float4* dst = reinterpret_cast<float4*>(tb);
#pragma unroll 4
        for (int q = tid; q < (int)(sizeof(FftTables) / 16); q += blockDim.x) dst[q] = __ldg(src + q);
        for (int q = tid; q <= L.n; q += blockDim.x) ts[q] = L.tile_start[q];
    }
    __syncthreads();
    float2* tr = tr_all + warp * 8 * kTrPitch;
    float* pw = pw_all + warp * kPwPitch;
    const int qk1 = lane >> 2, qb = lane & 3;          // (k1, b) after the transpose
    const int qd = bitrev2(qb);
#if LFG_FFT_REG_TW
    float2 rtw256[8], rtw32[8];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        rtw256[k] = tb->tw256[k * 32 + lane];
        rtw32[k] = tb->tw32[k * 4 + qb];
    }
#define TW256(k1) rtw256[k1]
#define TW32(c) rtw32[c]
#else
#define TW256(k1) tb->tw256[(k1) * 32 + lane]
#define TW32(c) tb->tw32[(c) * 4 + qb]
#endif
    const int total = L.tile_start[L.n];
    const int stride = gridDim.x * kFftWarps;
    // the raw taps x[(f - 1) * 160 + 2 n .. + 1], n = 32 n1 + lane (n1 < 5), of frame gf,
    // loaded one frame ahead so their latency hides behind the current frame's FFT
    auto load_taps = [&](int gfx, int& ux, float2 xv[5]) {
        // the utterance holding frame gfx: warp-uniform and monotone; the lanes test 32
        // utterances per step (a warp's next frame is ~stride / 600 utterances further on)
        for (;;) {
            const int idx = ux + 1 + lane;
            const unsigned past = __ballot_sync(0xFFFFFFFFu, idx > L.n ? true : ts[idx] > gfx);
            if (past != 0u) {
                ux += __ffs(past) - 1;
                break;
            }
            ux += 32;
        }
        const SpDesc& dx = L.d[ux];
        const int f = gfx - ts[ux];
        const int base = (f - 1) * kHop, Lw = dx.L;
        if (f >= dx.T) return;                          // splice padding: no taps
        // taps come in pairs (2 n, 2 n + 1): one 8-B load of f32, or one 4-B load of int16
        // PCM kept as the raw word in .x until the frame's stage 1 (pcm_pair) -- converting
        // here would wait on the load one frame early; reflect padding at the utterance ends
        const int esh = kPcm ? 1 : 2;                     // log2 bytes per sample
        const bool interior = base >= 0 && base + kTaps <= Lw &&
                              ((reinterpret_cast<uintptr_t>(dx.wav) & ((2u << esh) - 1)) == 0);
        const float* wf = static_cast<const float*>(dx.wav);
        const unsigned short* ws = static_cast<const unsigned short*>(dx.wav);
#pragma unroll
        for (int n1 = 0; n1 < 5; ++n1) {
            const int j = 2 * (32 * n1 + lane);
            if (interior) {
                if constexpr (kPcm) xv[n1] = make_float2(__uint_as_float(__ldg(reinterpret_cast<const unsigned int*>(ws + base + j))), 0.f);
                else xv[n1] = __ldg(reinterpret_cast<const float2*>(wf + base + j));
            } else {
                int i0 = base + j, i1 = base + j + 1;
                i0 = i0 < 0 ? -i0 : (i0 >= Lw ? 2 * (Lw - 1) - i0 : i0);
                i1 = i1 < 0 ? -i1 : (i1 >= Lw ? 2 * (Lw - 1) - i1 : i1);
                if constexpr (kPcm) xv[n1] = make_float2(__uint_as_float((uint32_t)__ldg(ws + i0) | ((uint32_t)__ldg(ws + i1) << 16)), 0.f);
                else xv[n1] = make_float2(__ldg(wf + i0), __ldg(wf + i1));
            }
        }
    };
    // Frame deal: round robin -- warp w of CTA b takes frames b * 8 + w + k * stride, so
    // neighbouring frames, which share half their taps, sit on neighbouring warps of one
    // CTA.  With L.work (A/B switch LFG_SPEECH_DEAL=tail) the last kFftDynRounds rounds come
    // from the launch's counter instead, so no SM of a lone launch idles while others
    // finish (masked and padding frames are cheap: ncu showed sm__cycles_active min 57 k /
    // avg 69 k / max 82 k of 86 k); lane 0's atomic runs one take ahead.  A warp's frames
    // increase either way (load_taps' utterance search relies on it).
    const bool dyn = L.work != nullptr;
    const int n_rr = dyn ? max(0, total / stride - kFftDynRounds) : (total + stride - 1) / stride;
    const int rr_end = n_rr * stride;
    uint32_t pend = 0;
    int k_rr = 0;
    auto take = [&]() -> int {
        if (k_rr < n_rr) return blockIdx.x * kFftWarps + warp + (k_rr++) * stride;
        if (!dyn) return total;
        const int g = rr_end + __shfl_sync(0xFFFFFFFFu, (int)pend, 0);
        if (lane == 0) pend = atomicAdd(L.work, 1u);
        return g;
    };
    if (dyn && lane == 0) pend = atomicAdd(L.work, 1u);
    int u = 0, un = 0;
    float2 cur[5], nxt[5];
    int gf = take(), gn = take();
    if (gf < total) load_taps(gf, un, cur);
    for (; gf < total; gf = gn, gn = take()) {
        u = un;
        if (gn < total) load_taps(gn, un, nxt);
        const SpDesc& d = L.d[u];
        const int f = gf - ts[u];
        const int T = d.T;
        float* out = d.out + (int64_t)f * kMels;
        bool tmask = f >= T;                            // splice padding frames are zero
        {   // time masks: lane q tests mask q
            const int qm = lane < 10 ? lane : 9;
            tmask |= __any_sync(0xFFFFFFFFu, lane < L.n_tmask && (unsigned)(f - d.t_lo[qm]) < (unsigned)d.t_w[qm]);
        }
        if (tmask) {
            for (int m = lane; m < kMels; m += 32) out[m] = 0.0f;
        } else {
            // stage 1: z[32 n1 + l] = a(2n) + i a(2n + 1), windowed taps
            float2 v[8];
#pragma unroll
            for (int n1 = 0; n1 < 8; ++n1) {
                if (n1 < 5) {
                    const int j = 2 * (32 * n1 + lane);
                    const float2 ww = *reinterpret_cast<const float2*>(tb->win + j);
                    float2 x = cur[n1];
                    if constexpr (kPcm) x = pcm_pair(__float_as_uint(cur[n1].x));
                    v[n1] = make_float2(x.x * ww.x, x.y * ww.y);
                } else {
                    v[n1] = make_float2(0.f, 0.f);
                }
            }
            dft8(v);
#pragma unroll
            for (int k1 = 1; k1 < 8; ++k1) v[k1] = cmul(v[k1], TW256(k1));
#pragma unroll
            for (int k1 = 0; k1 < 8; ++k1) tr[k1 * kTrPitch + lane] = v[k1];
            __syncwarp();
            // stage 2: lane (k1, b) takes the values of lanes 4a + b; 8-point DFT over a
#pragma unroll
            for (int a = 0; a < 8; ++a) v[a] = tr[qk1 * kTrPitch + 4 * a + qb];
            dft8(v);
#pragma unroll
            for (int c = 1; c < 8; ++c) v[c] = cmul(v[c], TW32(c));
            // stage 3: 4-point DFT across the lane quad (decimation in frequency); the
            // butterflies' p -/+ v as fmaf(-/+1, v, p): exact, one FFMA per component
            const float s2 = (qb & 2) ? -1.0f : 1.0f, s1 = (qb & 1) ? -1.0f : 1.0f;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float2 p2 = shfl2(v[c], lane ^ 2);
                v[c] = make_float2(fmaf(s2, v[c].x, p2.x), fmaf(s2, v[c].y, p2.y));
                if (qb == 3) v[c] = mul_mi(v[c]);                  // W4^1 on the upper half, j = 1
                const float2 p1 = shfl2(v[c], lane ^ 1);
                v[c] = make_float2(fmaf(s1, v[c].x, p1.x), fmaf(s1, v[c].y, p1.y));
            }
            // lane (k1, b') holds Z[k1 + 8 c + 64 d], d = bitrev2(b').  Real-FFT split:
            // Z[256 - k] lives at lane 4 (8 - k1) + 3 - b', element 7 - c (k1 >= 1), or in
            // the k1 = 0 quad: lane 3 - b', element 8 - c (c >= 1) / lane bitrev2(4 - d), element 0
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float2 give = qk1 >= 1 ? v[7 - c] : v[(8 - c) & 7];
                int src;
                if (qk1 >= 1) src = 4 * (8 - qk1) + 3 - qb;
                else if (c >= 1) src = 3 - qb;
                else src = bitrev2((4 - qd) & 3);
                const float2 zp = shfl2(give, src);
                const int k = qk1 + 8 * c + 64 * qd;
                const float2 zk = v[c];
                // 2 X_k = A + (-i W512^k) B with A = zk + conj zp (= 2 E_k), B = zk - conj zp
                // (= 2i O_k): the table holds -i W512^k and the mel weights carry the 1/4 of
                // |X_k|^2 = |2 X_k|^2 / 4
                const float2 A = make_float2(zk.x + zp.x, zk.y - zp.y);
                const float2 Bv = make_float2(zk.x - zp.x, zk.y + zp.y);
                const float2 t = tb->tw512[c * 32 + lane];
                const float yx = fmaf(t.x, Bv.x, fmaf(-t.y, Bv.y, A.x));
                const float yy = fmaf(t.x, Bv.y, fmaf(t.y, Bv.x, A.y));
                const float p = fmaf(yx, yx, yy * yy);
                pw[pw_at(k)] = p;
                if (c < kPwGap / 8 && qd != 0) pw[pw_at(k) - kPwGap] = p;   // the previous block's gap
                if (k == 0) {
                    const float ny = A.x - Bv.y;             // 2 X_256 = 2 E_0 - 2 O_0 (both real)
                    pw[pw_at(kBins) - kPwGap] = ny * ny;
                }
            }
            __syncwarp();
            // mel filters m = lane, lane + 32, lane + 64, log, frequency masks, store
            const int fl0 = d.f_lo[0], fw0 = L.n_fmask > 0 ? d.f_w[0] : 0;
            const int fl1 = d.f_lo[1], fw1 = L.n_fmask > 1 ? d.f_w[1] : 0;
            // Each filter's W-tap window starts s_m bins before its first bin (zero weights there;
            // s_m within the filter's slack W - span, chosen on the host so that a warp's
            // power-row loads of one tap step fall in distinct banks -- unshifted, the filters'
            // first bins collide 2-4 ways).
            auto mel_out = [&](auto W, int m) {
                const int a0 = tb->mel_b0[m];
                float acc = 0.0f;
#pragma unroll
                for (int q = 0; q < decltype(W)::value; ++q) acc = fmaf(tb->mel_wd[q * kMels + m], pw[a0 + q], acc);
                const bool masked = (unsigned)(m - fl0) < (unsigned)fw0 || (unsigned)(m - fl1) < (unsigned)fw1;
                out[m] = masked ? 0.0f : __logf(acc + 5.9604644775390625e-8f);   // + 2^-24
            };
            mel_out(std::integral_constant<int, kMelW0>{}, lane);
            mel_out(std::integral_constant<int, kMelW1>{}, lane + 32);
            {   // filters 64..79 (the widest): two lanes per filter, 9 taps each
                const int m = 64 + (lane & 15), h = lane >> 4;
                const int a0 = tb->mel_b2[lane];
                float acc = 0.0f;
#pragma unroll
                for (int q = 0; q < kMelW2 / 2; ++q)
                    acc = fmaf(tb->mel_wd[((kMelW2 / 2) * h + q) * kMels + m], pw[a0 + q], acc);
                acc += __shfl_xor_sync(0xFFFFFFFFu, acc, 16);
                const bool masked = (unsigned)(m - fl0) < (unsigned)fw0 || (unsigned)(m - fl1) < (unsigned)fw1;
                if (h == 0) out[m] = masked ? 0.0f : __logf(acc + 5.9604644775390625e-8f);
            }
        }
        __syncwarp();   // (tr / pw are reused by the next frame; the frame's stores precede the count)
        if (L.st.cnt != nullptr && lane == 0)
            sample_part_done(L.st.cnt + d.slot, L.st.stamp + d.slot, (uint32_t)(ts[u + 1] - ts[u]));
#pragma unroll
        for (int n1 = 0; n1 < 5; ++n1) cur[n1] = nxt[n1];
    }
    if (dyn) {
        // Hand the counter back zeroed: every warp's last grab must have landed (reading
        // pend waits for the atomic's return), then each CTA counts itself out and the
        // last one zeroes both words for the next launch on this pair.
        if (lane == 0 && pend == 0xFFFFFFFFu) __trap();   // (never: a counter value; waits on pend)
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (atomicAdd(L.work + 1, 1u) == gridDim.x - 1) {
                L.work[0] = 0u;
                L.work[1] = 0u;
            }
        }
    }
}
constexpr int kFftSmem = (int)sizeof(FftTables) + kFftWarps * 8 * kTrPitch * 8 + kFftWarps * kPwPitch * 4;

// K11: PermuteAudio + Pad: per-sample [T'_i, W] slots -> batch [T'_max, n, W], zero-padded.
// Grid (t_max, ceil(n / 4)): a CTA moves one time row of 4 samples, 64 threads per
// sample row (16-B loads / stores), so a batch is ~t_max * n / 4 small CTAs rather
// than t_max CTAs looping over every sample (2.5x fewer bytes in flight per SM).
__global__ void __launch_bounds__(256) speech_collate_kernel(const __grid_constant__ SpCollate C) {
    const int t = blockIdx.x;
    const int b = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (b >= C.n) return;
    const int w4 = C.width / 4;
    const bool live = t < C.rows[b];
    const float4* src = reinterpret_cast<const float4*>(C.src[b] + (int64_t)t * C.width);
    float4* dst = reinterpret_cast<float4*>(C.dst + ((int64_t)t * C.n + b) * C.width);
    for (int q = threadIdx.x & 63; q < w4; q += 64)
        dst[q] = live ? __ldcs(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// ------------------------------------------------------------------ host tables
uint32_t h_tf32_rna(float x) {   // cvt.rna.tf32.f32: round to nearest, ties away, 10-bit mantissa
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return u & 0xFFFFE000u;
    u += 0x1000u;
    return u & 0xFFFFE000u;
}
float as_f(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

}  // namespace

// FFT-kernel tail counters: one {next frame, CTAs done} pair per launch, taken
// round-robin; the last CTA of a launch zeroes its pair, so a pair is free again once
// that launch has finished -- far fewer than kWorkSlots launches are in flight at once.
constexpr int kWorkSlots = 4096;

struct SpeechTables {
    char* basis = nullptr;   // kChunks x 64 KB, the per-stage smem image of B (tensor-core kernel)
    FftTables* fft = nullptr;   // window, twiddles and mel (bin, weight) lists (FFT kernel)
    uint32_t* work = nullptr;   // kWorkSlots x {next frame, CTAs done}
    mutable std::atomic<uint32_t> seq{0};   // next pair (launches take pairs through a const table)
};

namespace {
// LFG_SPEECH_KERNEL=tc: the tcgen05 DFT-GEMM kernel (A/B); default: the FFT kernel
bool speech_use_tc() {
    static const bool tc = getenv("LFG_SPEECH_KERNEL") && std::strcmp(getenv("LFG_SPEECH_KERNEL"), "tc") == 0;
    return tc;
}
}  // namespace

cudaError_t speech_tables_create(SpeechTables** out) {
    // B: column col of N half h is bin 128 h + (col mod 128), cos (col < 128) or
    // -sin; row j is window tap j (frame position j + 96).  Computed in fp64.
    std::vector<double> win(kTaps);
    for (int j = 0; j < kTaps; ++j) win[j] = 0.5 - 0.5 * std::cos(2.0 * M_PI * j / kTaps);
    std::vector<char> img((size_t)kChunks * kBStageBytes, 0);
    for (int it = 0; it < kChunks; ++it)
        for (int q = 0; q < kKChunk / 8; ++q)
            for (int h = 0; h < 2; ++h)
                for (int col = 0; col < 256; ++col) {
                    const int k = 128 * h + (col & 127);
                    for (int jj = 0; jj < 8; ++jj) {
                        const int j = it * kKChunk + q * 8 + jj;
                        const int n = j + kWinOff;
                        const double ang = 2.0 * M_PI * (double)((int64_t)k * n % kNfft) / kNfft;
                        const double v = win[j] * (col < 128 ? std::cos(ang) : -std::sin(ang));
                        const uint32_t vh = h_tf32_rna((float)v);
                        const uint32_t vl = h_tf32_rna((float)(v - (double)as_f(vh)));
                        const int c = jj >> 2, e = jj & 3;
                        const size_t blk = (size_t)it * kBStageBytes + (size_t)((q * 2 + h) * 2) * kBBlock;
                        const size_t off = (size_t)sw32_off(col, c) + e * 4;
                        std::memcpy(&img[blk + off], &vh, 4);
                        std::memcpy(&img[blk + kBBlock + off], &vl, 4);
                    }
                }
    // Nyquist coefficients w[j] * (-1)^(j + 96)
    float nyq[kTaps];
    for (int j = 0; j < kTaps; ++j) nyq[j] = (float)(win[j] * (((j + kWinOff) & 1) ? -1.0 : 1.0));
    // slaney mel bank (torchaudio melscale_fbanks norm='slaney', mel_scale='slaney'), fp64
    auto hz2mel = [](double f) {
        const double fsp = 200.0 / 3.0, lo_hz = 1000.0, lo_mel = lo_hz / fsp, step = std::log(6.4) / 27.0;
        return f >= lo_hz ? lo_mel + std::log(f / lo_hz) / step : f / fsp;
    };
    auto mel2hz = [](double m) {
        const double fsp = 200.0 / 3.0, lo_hz = 1000.0, lo_mel = lo_hz / fsp, step = std::log(6.4) / 27.0;
        return m >= lo_mel ? lo_hz * std::exp(step * (m - lo_mel)) : fsp * m;
    };
    const int nf = kBins + 1;
    std::vector<double> pts(kMels + 2);
    const double m0 = hz2mel(0.0), m1 = hz2mel(8000.0);
    for (int i = 0; i < kMels + 2; ++i) pts[i] = mel2hz(m0 + (m1 - m0) * i / (kMels + 1));
    std::vector<double> fb((size_t)kMels * nf, 0.0);
    for (int m = 0; m < kMels; ++m)
        for (int k = 0; k < nf; ++k) {
            const double fk = 8000.0 * k / (nf - 1);
            const double down = (fk - pts[m]) / (pts[m + 1] - pts[m]);
            const double up = (pts[m + 2] - fk) / (pts[m + 2] - pts[m + 1]);
            const double v = std::max(0.0, std::min(down, up));
            fb[(size_t)m * nf + k] = v * 2.0 / (pts[m + 2] - pts[m]);
        }
    int mel_m[kBins + 1];
    float wa[kBins + 1], wb[kBins + 1];
    for (int k = 0; k < nf; ++k) {
        int first = -1;
        for (int m = 0; m < kMels; ++m)
            if (fb[(size_t)m * nf + k] != 0.0) {
                first = m;
                break;
            }
        mel_m[k] = first;
        wa[k] = first >= 0 ? (float)fb[(size_t)first * nf + k] : 0.f;
        wb[k] = (first >= 0 && first + 1 < kMels) ? (float)fb[(size_t)(first + 1) * nf + k] : 0.f;
        for (int m = first + 2; first >= 0 && m < kMels; ++m)
            if (fb[(size_t)m * nf + k] != 0.0) return cudaErrorInvalidValue;   // > 2 filters per bin
    }
    // FFT kernel tables (fp64 -> fp32)
    FftTables ft;
    std::memset(&ft, 0, sizeof(ft));
    for (int j = 0; j < kTaps; ++j) ft.win[j] = (float)win[j];
    auto tw = [](int num, int den) {   // exp(-2 pi i num / den)
        const double a = -2.0 * M_PI * (double)(num % den) / (double)den;
        return make_float2((float)std::cos(a), (float)std::sin(a));
    };
    for (int k1 = 0; k1 < 8; ++k1)
        for (int l = 0; l < 32; ++l) ft.tw256[k1 * 32 + l] = tw(l * k1, 256);
    for (int b = 0; b < 4; ++b)
        for (int c = 0; c < 8; ++c) ft.tw32[c * 4 + b] = tw(b * c, 32);
    for (int c = 0; c < 8; ++c)
        for (int l = 0; l < 32; ++l) {
            const int b = l & 3, d = ((b & 1) << 1) | ((b >> 1) & 1);
            const float2 w = tw((l >> 2) + 8 * c + 64 * d, 512);
            ft.tw512[c * 32 + l] = make_float2(w.y, -w.x);            // -i W512^k
        }
    int mel_lo[kMels];
    for (int m = 0; m < kMels; ++m) {
        int lo = -1, hi = -1;
        for (int k = 0; k < nf; ++k)
            if (fb[(size_t)m * nf + k] != 0.0) {
                if (lo < 0) lo = k;
                hi = k;
            }
        const int width = m < 32 ? kMelW0 : (m < 64 ? kMelW1 : kMelW2);
        if (lo < 0) lo = hi = 0;
        if (hi - lo + 1 > width || lo + width > nf) return cudaErrorInvalidValue;   // bank wider than the taps
        mel_lo[m] = lo;
    }
    int mel_hi[kMels];
    for (int m = 0; m < kMels; ++m) {
        mel_hi[m] = mel_lo[m];
        for (int k = mel_lo[m]; k < nf; ++k)
            if (fb[(size_t)m * nf + k] != 0.0) mel_hi[m] = k;
    }
    // Window shifts: filter m's W-tap window starts s_m bins before its first bin, 0 <= s_m <=
    // min(W - span_m, lo_m) (the extra taps carry zero weights).  The 32 lanes of a group read
    // pw_at(lo - s) + q at tap step q; s is chosen by coordinate descent to minimise the summed
    // shared-memory wavefronts of the W steps (distinct addresses per bank; the row's bank is
    // its word offset mod 32: the per-warp pitch is 13 x 32 words).  For the slaney bank:
    // 30 -> 10 wavefronts for the 10-tap group (one per step), 6 for the 3-tap group (no
    // slack); the 18-tap group below.
    // LFG_MEL_SHIFT=0 keeps every s = 0 (A/B switch).
    static const bool shift_on = !(getenv("LFG_MEL_SHIFT") && std::strcmp(getenv("LFG_MEL_SHIFT"), "0") == 0);
    // group of 32 lanes, lane l = filter m0 + l, W taps each
    auto shifts = [&](int W, int m0, int sh[32]) {
        auto cost = [&]() {
            int total = 0;
            for (int q = 0; q < W; ++q) {
                int addr[32];
                for (int l = 0; l < 32; ++l) addr[l] = pw_at(mel_lo[m0 + l] - sh[l]) + q;
                int worst = 0, sq = 0;
                for (int b = 0; b < 32; ++b) {
                    int seen[32], ns = 0;
                    for (int l = 0; l < 32; ++l) {
                        if ((addr[l] & 31) != b) continue;
                        bool dup = false;
                        for (int i = 0; i < ns; ++i) dup |= seen[i] == addr[l];
                        if (!dup) seen[ns++] = addr[l];
                    }
                    worst = std::max(worst, ns);
                    sq += ns * ns;
                }
                total += 1000 * worst + sq;   // wavefronts; the squares break the descent's ties
            }
            return total;
        };
        for (int l = 0; l < 32; ++l) sh[l] = 0;
        if (!shift_on) return;
        for (int pass = 0; pass < 8; ++pass)
            for (int f = 0; f < 32; ++f) {
                const int m = m0 + f;
                const int slack = std::min(W - (mel_hi[m] - mel_lo[m] + 1), mel_lo[m]);
                int best = sh[f], best_c = cost();
                for (int r = 0; r <= slack; ++r) {
                    sh[f] = r;
                    const int c = cost();
                    if (c < best_c) best = r, best_c = c;
                }
                sh[f] = best;
            }
    };
    auto wgt = [&](int m, int k) { return (float)fb[(size_t)m * nf + k] * 0.25f; };
    for (int g = 0; g < 2; ++g) {   // filters 0..31 (3 taps), 32..63 (10 taps): lane l = filter 32 g + l
        const int W = g == 0 ? kMelW0 : kMelW1;
        int sh[32];
        shifts(W, 32 * g, sh);
        for (int l = 0; l < 32; ++l) {
            const int m = 32 * g + l, k0 = mel_lo[m] - sh[l];
            ft.mel_b0[m] = pw_at(k0);
            for (int q = 0; q < W; ++q) ft.mel_wd[q * kMels + m] = wgt(m, k0 + q);
        }
    }
    {   // filters 64..79 (18 taps): lane l = filter 64 + (l & 15), half h = l >> 4.  Half 0
        // reads bins k0 .. k0 + 8 (k0 = lo - s), half 1 bins k0 + 9 - t .. k0 + 17 - t; bins both
        // halves read carry their weight in half 0 only.  Coverage of [lo, hi] needs
        // s + t <= 18 - span.  (s, t) per filter by a fixed-seed annealing (coordinate descent
        // stalls here; model: 27 -> 9 wavefronts per frame), computed once per process.
        constexpr int W = kMelW2 / 2;
        struct G2 {
            int s[16], t[16];
        };
        static const G2 g2 = [&] {
            G2 g{};
            if (!shift_on) return g;
            int span[16];
            for (int f = 0; f < 16; ++f) span[f] = mel_hi[64 + f] - mel_lo[64 + f] + 1;
            auto cost = [&](const G2& x) {
                int total = 0;
                for (int q = 0; q < W; ++q) {
                    int addr[32];
                    for (int l = 0; l < 32; ++l) {
                        const int f = l & 15;
                        addr[l] = pw_at(mel_lo[64 + f] - x.s[f]) + (l >> 4) * (W - x.t[f]) + q;
                    }
                    int worst = 0, sq = 0;
                    for (int b = 0; b < 32; ++b) {
                        int seen[32], ns = 0;
                        for (int l = 0; l < 32; ++l) {
                            if ((addr[l] & 31) != b) continue;
                            bool dup = false;
                            for (int i = 0; i < ns; ++i) dup |= seen[i] == addr[l];
                            if (!dup) seen[ns++] = addr[l];
                        }
                        worst = std::max(worst, ns);
                        sq += ns * ns;
                    }
                    total += 1000 * worst + sq;
                }
                return total;
            };
            uint64_t rng = 0x9E3779B97F4A7C15ull;
            auto next = [&](int n) {   // uniform in [0, n)
                rng = rng * 6364136223846793005ull + 1442695040888963407ull;
                return static_cast<int>((rng >> 33) % static_cast<uint64_t>(n));
            };
            G2 cur = g, best = g;
            int c_cur = cost(cur), c_best = c_cur;
            double T = 200.0;
            for (int it = 0; it < 30000; ++it) {
                const int f = next(16);
                const int smax = std::min(kMelW2 - span[f], mel_lo[64 + f]);
                G2 cand = cur;
                cand.s[f] = next(smax + 1);
                cand.t[f] = next(kMelW2 - span[f] - cand.s[f] + 1);
                const int c = cost(cand);
                const double u = static_cast<double>(next(1 << 30)) / static_cast<double>(1 << 30);
                if (c <= c_cur || u < std::exp((c_cur - c) / T)) cur = cand, c_cur = c;
                if (c_cur < c_best) best = cur, c_best = c_cur;
                T = std::max(0.5, T * 0.9997);
            }
            return best;
        }();
        for (int f = 0; f < 16; ++f) {
            const int m = 64 + f, k0 = mel_lo[m] - g2.s[f], k1 = k0 + W - g2.t[f];
            ft.mel_b0[m] = pw_at(k0);
            for (int q = 0; q < W; ++q) {
                ft.mel_wd[q * kMels + m] = wgt(m, k0 + q);
                ft.mel_wd[(W + q) * kMels + m] = k1 + q < k0 + W ? 0.0f : wgt(m, k1 + q);
            }
            ft.mel_b2[f] = pw_at(k0);
            ft.mel_b2[16 + f] = pw_at(k0) + W - g2.t[f];
        }
    }
    cudaError_t e;
    if ((e = cudaMemcpyToSymbol(c_win_nyq, nyq, sizeof(nyq))) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_mel_m, mel_m, sizeof(mel_m))) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_mel_wa, wa, sizeof(wa))) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_mel_wb, wb, sizeof(wb))) != cudaSuccess) return e;
    auto* t = new SpeechTables;
    if ((e = cudaMalloc(&t->basis, img.size())) != cudaSuccess) {
        delete t;
        return e;
    }
    if ((e = cudaMemcpy(t->basis, img.data(), img.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
        cudaFree(t->basis);
        delete t;
        return e;
    }
    if ((e = cudaFuncSetAttribute(speech_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBytes)) != cudaSuccess)
        return e;
    if ((e = cudaMalloc(&t->fft, sizeof(FftTables))) != cudaSuccess ||
        (e = cudaMemcpy(t->fft, &ft, sizeof(FftTables), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(speech_fft_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFftSmem)) !=
            cudaSuccess ||
        (e = cudaFuncSetAttribute(speech_fft_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFftSmem)) !=
            cudaSuccess ||
        (e = cudaMalloc(&t->work, sizeof(uint32_t) * 2 * kWorkSlots)) != cudaSuccess ||
        (e = cudaMemset(t->work, 0, sizeof(uint32_t) * 2 * kWorkSlots)) != cudaSuccess) {
        speech_tables_destroy(t);
        return e;
    }
    *out = t;
    return cudaSuccess;
}

void speech_tables_destroy(SpeechTables* t) {
    if (!t) return;
    cudaFree(t->basis);
    cudaFree(t->fft);
    cudaFree(t->work);
    delete t;
}

int speech_frames_per_cta() { return speech_use_tc() ? kFramesPerCta : kFftFrames; }   // (stack must divide it)

cudaError_t launch_speech(const SpLaunch& L0, const SpeechTables* t, cudaStream_t s) {
    if (L0.n <= 0) return cudaSuccess;
    static const int dbg = getenv("LFG_SPEECH_DEBUG") ? atoi(getenv("LFG_SPEECH_DEBUG")) : 0;
    SpLaunch L = L0;
    L.debug = dbg;
    L.tile_start[0] = 0;
    if (speech_use_tc()) {   // CTA tiles of kFramesPerCta frames
        if (L.pcm16) return cudaErrorNotSupported;   // (the A/B tensor-core kernel reads f32 only)
        for (int i = 0; i < L.n; ++i)
            L.tile_start[i + 1] = L.tile_start[i] + (L.d[i].T + kFramesPerCta - 1) / kFramesPerCta;
        speech_kernel<<<L.tile_start[L.n], kThreads, kSmemBytes, s>>>(L, t->basis);
        return cudaGetLastError();
    }
    // FFT kernel: frame prefix sums (splice-padded frame counts); 3 CTAs per SM
    for (int i = 0; i < L.n; ++i)
        L.tile_start[i + 1] = L.tile_start[i] + (L.d[i].T + L.stack - 1) / L.stack * L.stack;
    static int sms = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    const int need = (L.tile_start[L.n] + kFftWarps - 1) / kFftWarps;
    const int grid = need < 3 * sms ? need : 3 * sms;
    // LFG_SPEECH_DEAL=tail: the last rounds of the frame deal from the launch's counter (A/B
    // switch).  It evens out one launch alone (46.5 -> 45.2 us per 64 utterances), but in
    // the shard, where launch groups overlap on their streams, it keeps every CTA of a
    // launch alive to its end instead of retiring CTAs as their frames run out, so the
    // next launch's CTAs start later: C4 1.67 M -> 1.50 M utterances/s.  Default: the
    // pure round-robin deal.
    static const bool tail = getenv("LFG_SPEECH_DEAL") && std::strcmp(getenv("LFG_SPEECH_DEAL"), "tail") == 0;
    L.work = tail ? t->work + 2 * (t->seq.fetch_add(1, std::memory_order_relaxed) & (kWorkSlots - 1)) : nullptr;
    if (L.pcm16) speech_fft_kernel<true><<<grid > 0 ? grid : 1, 32 * kFftWarps, kFftSmem, s>>>(L, t->fft);
    else speech_fft_kernel<false><<<grid > 0 ? grid : 1, 32 * kFftWarps, kFftSmem, s>>>(L, t->fft);
    return cudaGetLastError();
}

cudaError_t launch_speech_collate(const SpCollate& C, cudaStream_t s) {
    if (C.n <= 0 || C.t_max <= 0) return cudaSuccess;
    speech_collate_kernel<<<dim3(C.t_max, (C.n + 3) / 4), 256, 0, s>>>(C);
    return cudaGetLastError();
}

cudaError_t warm_speech() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, speech_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, speech_fft_kernel<false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, speech_fft_kernel<true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, speech_collate_kernel);
    return e;
}

}  // namespace lfg
