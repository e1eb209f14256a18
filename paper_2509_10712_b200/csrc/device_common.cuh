// device_common.cuh -- counter-based RNG and small helpers shared by the kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lfg {

// Philox4x32-10 (Salmon et al. SC'11), Random123 constants.  The CPU oracle
// restates the same function (oracle/lf_oracle.c) and pins it to the
// Random123 known-answer vectors.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// -2 ln(u), u = (x + 0.5) * 2^-32, accurate at both ends of (0, 1): the upper
// half goes through log1p of the exact complement so values of u near 1 keep
// their relative precision (the oracle computes this in fp64).
__device__ __forceinline__ float neg2ln_u(uint32_t x) {
    const float two_m32 = 2.3283064365386963e-10f;  // 2^-32
    float l;
    if (x < 0x80000000u) {
        l = logf(fmaf((float)x, two_m32, 0.5f * two_m32));
    } else {
        const uint32_t m = 0xFFFFFFFFu - x;          // exact: 1 - u = (m + 0.5) * 2^-32
        l = log1pf(-fmaf((float)m, two_m32, 0.5f * two_m32));
    }
    return -2.0f * l;
}

// Box-Muller on one pair of 32-bit uniforms (same pairing as lfo_normals4).
__device__ __forceinline__ float2 box_muller(uint32_t xa, uint32_t xb) {
    const float two_m31 = 4.656612873077393e-10f;    // 2 * 2^-32
    const float r = sqrtf(neg2ln_u(xa));
    float s, c;
    sincospif(fmaf((float)xb, two_m31, two_m31 * 0.5f), &s, &c);  // angle = 2*pi*u2
    return make_float2(r * c, r * s);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ mbarrier / bulk-copy PTX
// Per-sample completion stamps (the shard classifies samples, not launch groups).
// Each sample of a group's last stage has a slot: a device counter cnt[slot] and
// a host-mapped stamp[slot] the host polls.  Every part of the sample's work (a
// CTA, or a warp's tile) calls this once, from one thread, after its output
// stores are ordered before it (__syncthreads / __syncwarp): the acq_rel count
// publishes them device-wide; the part that completes the count resets it (for
// the slot's next use) and writes %globaltimer | 1 to the host with release
// semantics at system scope.
__device__ __forceinline__ void sample_part_done(uint32_t* cnt, uint64_t* stamp, uint32_t parts) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    if (old + 1 == parts) {
        *cnt = 0u;
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(stamp), "l"(t | 1ull) : "memory");
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// TMA tiled load of a 3-D box at element coordinates (x, y, z); out-of-bounds
// elements are zero-filled by the copy engine.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace lfg
