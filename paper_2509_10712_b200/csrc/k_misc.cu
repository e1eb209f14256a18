// k_misc.cu -- K12 collate gather, K13/K14 device-clock spins, synthetic inputs.
#include "device_common.cuh"
#include "kernels.h"

namespace lfg {

namespace {

// K14: per-sample synthetic cost (LightStep / HeavyStep, workloads.cpp:109-110,
// and the per-step `step_costs` of synthetic chains).  One single-warp CTA per
// group member spins on %globaltimer; __nanosleep keeps the warp off the issue
// ports so the spin models latency, not SM occupancy.
__global__ void spin_kernel(const __grid_constant__ SpinLaunch L) {
    const int64_t ns = L.ns[blockIdx.x];
    if (threadIdx.x != 0) return;
    const uint64_t t0 = globaltimer_ns();
    while (ns > 0 && (int64_t)(globaltimer_ns() - t0) < ns) __nanosleep(1000);
    if (L.st.cnt != nullptr) {
        const int sl = L.slot[blockIdx.x];
        sample_part_done(L.st.cnt + sl, L.st.stamp + sl, 1u);
    }
}

// K13: synthetic trainer step (trainer.cpp:50-51): `ctas` CTAs spin for ns.
__global__ void trainer_spin_kernel(int64_t ns) {
    if (threadIdx.x != 0) return;
    const uint64_t t0 = globaltimer_ns();
    while ((int64_t)(globaltimer_ns() - t0) < ns) __nanosleep(2000);
}

// K12: collate per-sample output slots into one contiguous planar batch.
// blockIdx.y = sample, grid-stride over 16-byte words of each plane.
__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ GatherLaunch L) {
    const int i = blockIdx.y;
    for (int p = 0; p < L.nplanes; ++p) {
        const int64_t words = L.plane_bytes[p] >> 4;
        const int4* src =
            reinterpret_cast<const int4*>(L.src[i] + (p ? L.src_plane_stride[i] : 0));
        int4* dst = reinterpret_cast<int4*>(L.dst + p * L.dst_plane_stride +
                                            (int64_t)i * L.plane_bytes[p]);
        for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
             w += (int64_t)gridDim.x * blockDim.x) {
            dst[w] = __ldcs(src + w);
        }
    }
}

// ---- synthetic inputs: Philox(seed, id) streams --------------------------------
__device__ __forceinline__ uint4 synth_rand(uint64_t seed, uint64_t id, uint64_t ctr,
                                            uint32_t stream) {
    const uint64_t k = seed * 0x9E3779B97F4A7C15ull ^ (id + 1) * 0xC2B2AE3D27D4EB4Full;
    return philox4x32_10(make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), stream, 0x5EEDu),
                         (uint32_t)k, (uint32_t)(k >> 32));
}

// KiTS19-shaped volume: img ~ N(0,1); label 1 inside an ellipsoid ("kidney"),
// 2 inside a smaller off-centre one ("tumour"), else 0.
__global__ void synth_volume_kernel(uint64_t seed, uint64_t id, int64_t D, int64_t H, int64_t W,
                                    float* img, uint8_t* lbl) {
    const int64_t n = D * H * W;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 4 < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = synth_rand(seed, id, (uint64_t)q, 1u);
        const float2 a = box_muller(r.x, r.y), b = box_muller(r.z, r.w);
        const float zz[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t v = q * 4 + j;
            if (v >= n) break;
            img[v] = zz[j];
            const int64_t x = v % W, y = (v / W) % H, z = v / (W * H);
            const float dz = (z - 0.5f * D) / (0.25f * D), dy = (y - 0.5f * H) / (0.25f * H),
                        dx = (x - 0.5f * W) / (0.25f * W);
            const float e = dz * dz + dy * dy + dx * dx;
            const float tz = (z - 0.55f * D) / (0.08f * D), ty = (y - 0.45f * H) / (0.08f * H),
                        tx = (x - 0.5f * W) / (0.08f * W);
            const float t = tz * tz + ty * ty + tx * tx;
            lbl[v] = t <= 1.0f ? 2 : (e <= 1.0f ? 1 : 0);
        }
    }
}

// ImageNet-shaped u8 HWC image: bytes straight from Philox.
__global__ void synth_image_kernel(uint64_t seed, uint64_t id, int64_t n, uint8_t* out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 16 < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = synth_rand(seed, id, (uint64_t)q, 2u);
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int64_t v = q * 16 + j;
            if (v < n) out[v] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
        }
    }
}

// 16 kHz utterance: three sines (per-id frequencies) + N(0, 0.01) noise.
__global__ void synth_waveform_kernel(uint64_t seed, uint64_t id, int64_t L, float* wav) {
    const uint4 f = synth_rand(seed, id, 0xFFFFFFFFull, 3u);
    const float f1 = 100.0f + (f.x % 700u), f2 = 300.0f + (f.y % 1500u), f3 = 1000.0f + (f.z % 5000u);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 4 < L;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = synth_rand(seed, id, (uint64_t)q, 4u);
        const float2 a = box_muller(r.x, r.y), b = box_muller(r.z, r.w);
        const float zz[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t v = q * 4 + j;
            if (v >= L) break;
            const float t = (float)v / 16000.0f;
            wav[v] = 0.5f * sinpif(2.0f * f1 * t) + 0.3f * sinpif(2.0f * f2 * t) +
                     0.2f * sinpif(2.0f * f3 * t) + 0.01f * zz[j];
        }
    }
}

int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace

cudaError_t launch_spin(const SpinLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    spin_kernel<<<L.n, 32, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_trainer_spin(int64_t ns, int ctas, cudaStream_t s) {
    trainer_spin_kernel<<<ctas > 0 ? ctas : 1, 32, 0, s>>>(ns);
    return cudaGetLastError();
}

cudaError_t launch_gather(const GatherLaunch& L, cudaStream_t s) {
    if (L.n <= 0) return cudaSuccess;
    // planes are copied in 16-B words: slot strides are 16-B multiples (chain_create)
    for (int p = 0; p < L.nplanes; ++p)
        if (L.plane_bytes[p] & 15) return cudaErrorInvalidValue;
    int64_t words = L.plane_bytes[0] >> 4;
    int gx = (int)((words + 256 * 8 - 1) / (256 * 8));
    if (gx < 1) gx = 1;
    if (gx > 1024) gx = 1024;
    gather_kernel<<<dim3(gx, L.n), 256, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_synth_volume(uint64_t seed, uint64_t id, int64_t D, int64_t H, int64_t W,
                                float* img, uint8_t* lbl, cudaStream_t s) {
    synth_volume_kernel<<<grid_for((D * H * W + 3) / 4, 256), 256, 0, s>>>(seed, id, D, H, W,
                                                                            img, lbl);
    return cudaGetLastError();
}

cudaError_t launch_synth_image(uint64_t seed, uint64_t id, int64_t H, int64_t W, uint8_t* hwc,
                               cudaStream_t s) {
    const int64_t n = H * W * 3;
    synth_image_kernel<<<grid_for((n + 15) / 16, 256), 256, 0, s>>>(seed, id, n, hwc);
    return cudaGetLastError();
}

cudaError_t launch_synth_waveform(uint64_t seed, uint64_t id, int64_t L, float* wav,
                                  cudaStream_t s) {
    synth_waveform_kernel<<<grid_for((L + 3) / 4, 256), 256, 0, s>>>(seed, id, L, wav);
    return cudaGetLastError();
}

}  // namespace lfg

namespace lfg {
cudaError_t warm_misc() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, spin_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, trainer_spin_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gather_kernel);
    return e;
}
}  // namespace lfg
