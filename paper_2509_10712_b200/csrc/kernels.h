// kernels.h -- launch-parameter structs and host launchers for the sm_100a
// transform kernels.  Each fused kernel takes a whole launch group (up to
// kMax* samples) as one __grid_constant__ parameter block, so a group costs
// one launch and no descriptor upload.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace lfg {

constexpr int kMax3D = 16;   // img_seg samples per launch group
constexpr int kMax2D = 256;  // obj_det samples per launch group
constexpr int kMaxSp = 64;   // speech utterances per launch group
constexpr int kMaxSpin = 256;   // >= the largest launch group
constexpr int kMaxGather = 256;
constexpr int kTapsDft = 320;   // speech: non-zero window taps per frame (the DFT GEMM's K)

// Row addressing shared by K1/K3: a source row (z, y) starts at
//   base + z*pitch_z + y*pitch_y + ((skew0 + z*skew_z + y*skew_y) & mask)
// For HBM-resident payloads the skews are 0.  For payloads staged from pinned
// host memory by K0 the skews re-create the source's 16-byte alignment phase,
// which lets K0 move every row with aligned 16-byte loads and stores.

// ---- per-sample completion stamps (device_common.cuh sample_part_done): the
// launch of a group's LAST stage carries them; sample i of the launch owns slot
// d[i].slot (stamp_cnt: device counters, stamp: host-mapped pinned words).
// Null: no stamps (the group's completion event alone).
struct StampRef {
    uint32_t* cnt;
    uint64_t* stamp;
};

// ---- K0: strided-box gather from pinned host memory (PCIe) into HBM staging
struct StageDesc {
    const char* src;         // first byte of the box in host memory (UVA pointer)
    char* dst;               // 16-B aligned staging base
    int64_t src_py, src_pz;  // host row / plane pitch (bytes)
    int64_t dst_py, dst_pz;  // staging row / plane pitch (bytes, multiples of 16)
    int32_t row_bytes, ny, nz;
    int32_t pad;
};
constexpr int kMaxStage = 256;   // boxes per K0 launch (>= kMax2D, 2 * kMax3D)
struct StageLaunch {
    int32_t n;
    StageDesc d[kMaxStage];
};
static_assert(kMaxStage >= 2 * 16 && kMaxStage >= 256, "K0 must hold a whole launch group");

// ---- K0w: the crop windows of foreground-oversampled samples from pinned host
// memory.  Their origin is resolved on the device (K2 over the staged label
// volume), so the window cannot be a host-described K0 box: this kernel reads the
// origin from offs[i], pulls the image window rows over PCIe (16-B aligned reads,
// realigned by warp shuffles) and the label window rows from the staged label
// volume in HBM, into compact windows (skew 0, zero outside the volume).
struct WindowDesc {
    const float* img_host;   // UVA pointer of the pinned D x H x W f32 image volume
    const uint8_t* lbl;      // the staged label volume (K0 layout: pitches + skews)
    int64_t lbl_py, lbl_pz;
    int32_t lbl_sk0, lbl_sky, lbl_skz;
    int32_t dims[3];         // D, H, W of the source volume
    int32_t win[3];          // window edge (crop, or the RandomZoom3D window)
    int32_t img_pitch;       // floats per compact window row (multiple of 4)
    int32_t lbl_pitch;       // bytes per compact label row (multiple of 16)
    float* dst_img;          // [win0][win1][img_pitch]
    uint8_t* dst_lbl;        // [win0][win1][lbl_pitch]
};
struct WindowLaunch {
    int32_t n;
    const int4* offs;        // K2's window origins (d, h, w), one per sample
    WindowDesc d[16];
};

// ---- K1: RandomCrop + RandomFlip + RandomBrightness + GaussianNoise + Cast
struct Img3dDesc {
    const float* img;        // source: full volume (HBM) or staged crop window
    const uint8_t* lbl;
    float* out_img;          // [cd, ch, cw] f32
    uint8_t* out_lbl;        // [cd, ch, cw] u8
    int64_t img_py, img_pz;  // row / plane pitch in elements
    int64_t lbl_py, lbl_pz;  // row / plane pitch in bytes
    int32_t img_sk0, img_sky, img_skz;  // skew in floats (mask 3)
    int32_t lbl_sk0, lbl_sky, lbl_skz;  // skew in bytes (mask 15)
    int32_t sdim[3];         // valid extents of the source (d, h, w)
    int32_t off[3];          // crop origin inside the source
    int32_t flip;            // bit a = flip axis a
    float scale;             // brightness multiplier
    float sigma;             // noise std (0 = no noise)
    uint32_t key0, key1;     // Philox key
    int32_t win[3];          // source window edge (RandomZoom3D; = crop otherwise)
    float contrast;          // RandomContrast factor (1 = not applied)
    const double* csum;      // contrast: sum of the (resampled) crop, written by K5 (null: none)
    double zscale[3];        // RandomZoom3D source-index scale win / crop (IEEE division, host)
    int32_t slot;            // completion stamp slot
    int32_t contrast_on;     // (host) RandomContrast drawn: K5 sums the crop first
};
// Contrast folded into one affine per sample: out = A * v + B (+ noise), with
// A = scale * c and B = scale * (1 - c) * mean, mean = csum / crop voxels.
__device__ __forceinline__ void img3d_affine(const Img3dDesc& d, int64_t crop_vox, float& A, float& B) {
    if (d.csum == nullptr) {
        A = d.scale;
        B = 0.0f;
        return;
    }
    const double mean = *d.csum / (double)crop_vox;
    A = (float)((double)d.scale * (double)d.contrast);
    B = (float)((double)d.scale * (1.0 - (double)d.contrast) * mean);
}
struct Img3dLaunch {
    int32_t crop[3];
    int32_t n;
    // RandomCrop foreground oversampling: window origins resolved on the device by K2
    // (offs[i].w = 1: use offs[i].xyz = (d, h, w) instead of d[i].off); null: none
    const int4* offs;
    int32_t tma;             // 1: every sample has tm_img/tm_lbl (TMA tile path)
    int32_t debug;           // profiling switch (LFG_IMG3D_DEBUG): 1 no stores, 2 no loads
    StampRef st;             // per-sample completion stamps (null cnt: none)
    Img3dDesc d[kMax3D];
    // TMA path: 3-D tiled maps over the whole source volume (dims W, H, D),
    // box (cw + 16, kImg3dTileRows, 1); out-of-bounds boxes fill zeros, which is
    // exactly RandomCrop's zero padding.
    CUtensorMap tm_img[kMax3D];
    CUtensorMap tm_lbl[kMax3D];
};
__device__ __forceinline__ void img3d_offsets(const Img3dLaunch& L, int i, int off[3]) {
    const Img3dDesc& d = L.d[i];
    off[0] = d.off[0];
    off[1] = d.off[1];
    off[2] = d.off[2];
    if (L.offs != nullptr) {
        const int4 o = L.offs[i];
        if (o.w) {
            off[0] = o.x;
            off[1] = o.y;
            off[2] = o.z;
        }
    }
}
#ifndef LFG_IMG3D_TILE_ROWS
#define LFG_IMG3D_TILE_ROWS 8   // (build-time A/B switch)
#endif
constexpr int kImg3dTileRows = LFG_IMG3D_TILE_ROWS;
// TMA path preconditions on the sample / crop geometry (else the row kernel runs)
inline bool img3d_tma_ok(const void* img, const void* lbl, const int64_t dims[3], const int crop[3]) {
    return (reinterpret_cast<uintptr_t>(img) & 15) == 0 && (reinterpret_cast<uintptr_t>(lbl) & 15) == 0 &&
           dims[2] % 16 == 0 && crop[2] % 16 == 0 && crop[2] <= 240 && dims[0] < (int64_t(1) << 31) &&
           dims[1] < (int64_t(1) << 31) && dims[2] < (int64_t(1) << 31);
}

// ---- K3: RandomResizedCrop (bilinear) + RandomHorizontalFlip + ToTensor + Normalize
// 16 B per image, packed: the launch passes up to 256 of these as kernel
// parameters, and the launch call's host cost grows with the parameter block
// (8 KB of 32-B descriptors: ~12 us per call; 4 KB: ~8 us).  h / oh and w / ow
// are divided on the device, IEEE-rounded like the host / oracle.
//   a: bits  0-47 src (crop-box origin, row 0 column 0, of an HWC u8 image; UVA)
//           48-51 sk0, 52-55 sky (row skew, see above), 56-63 output buffer (low 8 bits)
//   b: bits  0-17 pitch (bytes per source row), 18-33 h, 34-49 w (crop box),
//           50 flip, 51-59 position in the output buffer, 60-63 output buffer (high 4 bits)
// The output of image i is out_tab[buffer] + position * out_stride floats; the
// buffer index is the context's slot-buffer index (out_tab: device table).
struct RrcDesc {
    uint64_t a, b;
};
static_assert(sizeof(RrcDesc) == 16, "RrcDesc layout");
__host__ __device__ inline const uint8_t* rrc_src(const RrcDesc& d) {
    return reinterpret_cast<const uint8_t*>(d.a & 0xFFFFFFFFFFFFull);
}
__host__ __device__ inline int rrc_sk0(const RrcDesc& d) { return (int)((d.a >> 48) & 15); }
__host__ __device__ inline int rrc_sky(const RrcDesc& d) { return (int)((d.a >> 52) & 15); }
__host__ __device__ inline int rrc_pitch(const RrcDesc& d) { return (int)(d.b & 0x3FFFF); }
__host__ __device__ inline int rrc_h(const RrcDesc& d) { return (int)((d.b >> 18) & 0xFFFF); }
__host__ __device__ inline int rrc_w(const RrcDesc& d) { return (int)((d.b >> 34) & 0xFFFF); }
__host__ __device__ inline int rrc_flip(const RrcDesc& d) { return (int)((d.b >> 50) & 1); }
__host__ __device__ inline int rrc_pos(const RrcDesc& d) { return (int)((d.b >> 51) & 0x1FF); }
__host__ __device__ inline int rrc_buf(const RrcDesc& d) { return (int)(((d.a >> 56) & 0xFF) | (((d.b >> 60) & 0xF) << 8)); }
// false if a field does not fit (src >= 2^48, pitch >= 2^18, position >= 512, buffer >= 4096)
inline bool rrc_pack(RrcDesc& d, const void* src, int sk0, int sky, int pitch, int h, int w, int flip, int pos,
                     int buf) {
    const uint64_t p = reinterpret_cast<uint64_t>(src);
    if ((p >> 48) || pitch < 0 || pitch >= (1 << 18) || h < 1 || h > 0xFFFF || w < 1 || w > 0xFFFF || pos < 0 ||
        pos >= 512 || buf < 0 || buf >= 4096)
        return false;
    d.a = p | (uint64_t(sk0 & 15) << 48) | (uint64_t(sky & 15) << 52) | (uint64_t(buf & 0xFF) << 56);
    d.b = uint64_t(pitch) | (uint64_t(h) << 18) | (uint64_t(w) << 34) | (uint64_t(flip & 1) << 50) |
          (uint64_t(pos) << 51) | (uint64_t(buf >> 8) << 60);
    return true;
}
constexpr int kMaxRrcBufs = 4096;
struct RrcLaunch {
    int32_t oh, ow;
    float a[3], b[3];        // out = v * a_c + b_c  (= (v/255 - mean_c) / std_c)
    int32_t n;
    int32_t slot_base;       // completion stamp slot of image i: slot_base + i
    StampRef st;
    float* const* out_tab;   // device table: slot-buffer index -> base
    int64_t out_stride;      // floats per output slot
    RrcDesc d[kMax2D];
};

// ---- K8-K11 (speech): STFT power -> mel -> log -> SpecAugment -> FrameSplicing
struct SpDesc {
    const void* wav;         // f32 samples, or int16 PCM (SpLaunch.pcm16)
    float* out;              // spliced log-mel [T', stack*n_mels]  (time-major)
    int32_t L;
    int32_t T;               // frames
    int32_t f_lo[2], f_w[2];
    int32_t t_lo[10], t_w[10];
    int32_t slot;            // completion stamp slot
    int32_t pad_;
};
struct SpLaunch {
    int32_t n;
    int32_t n_fmask, n_tmask;
    int32_t stack;
    int32_t debug;            // profiling switch: 1 builders skip loads, 2 skip MMAs
    int32_t pcm16;            // waveforms are int16 PCM (x = s / 32768), else f32
    uint32_t* work;           // FFT kernel: this launch's {next tail frame, CTAs done} (null: no tail deal)
    StampRef st;
    int32_t tile_start[kMaxSp + 1];   // CTA prefix sums (flattened grid), filled by the launcher
    SpDesc d[kMaxSp];
};

// ---- K11 (speech seal): PermuteAudio + Pad, per-sample [T'_i, width] -> [t_max, n, width]
struct SpCollate {
    int32_t n;
    int32_t width;
    int32_t t_max;
    int32_t rows[kMaxGather];
    const float* src[kMaxGather];
    float* dst;
};

// ---- K14: synthetic per-sample cost (LightStep / HeavyStep / step_costs)
struct SpinLaunch {
    int32_t n;
    StampRef st;
    int64_t ns[kMaxSpin];
    int32_t slot[kMaxSpin];
};

// ---- K12: batch collation gather (planar: plane p of sample i -> dst + p*plane_stride + i*plane_bytes[p])
struct GatherLaunch {
    int32_t n;
    int32_t nplanes;
    int64_t plane_bytes[2];
    int64_t src_plane_stride[kMaxGather];   // per source slot: distance from plane 0 to plane 1
    const char* src[kMaxGather];
    char* dst;
    int64_t dst_plane_stride;
};

cudaError_t launch_stage(const StageLaunch& L, cudaStream_t s);
cudaError_t launch_stage_window(const WindowLaunch& L, cudaStream_t s);
cudaError_t launch_img3d(const Img3dLaunch& L, cudaStream_t s);
// K4: RandomZoom3D chains (trilinear image / nearest label resample of the window)
cudaError_t launch_img3d_zoom(const Img3dLaunch& L, cudaStream_t s);
// K5: per-sample sum of the (resampled) crop for RandomContrast; L.d[i].csum
// must point at zeroed doubles
cudaError_t launch_img3d_mean(const Img3dLaunch& L, cudaStream_t s);
// K2: RandomCrop foreground oversampling.  fg_scan: per-class (labels 1..7)
// bounding boxes of the samples that drew it into box: mins [kMax3D][8][3] then
// maxs [kMax3D][8][3] (mins preset to 0x7f7f7f7f, maxs to -1); fg_offsets: the
// window origins of every sample into offs (w = 0 where the random offsets hold).
struct FgDraw {
    int32_t fg;              // foreground crop drawn (its label volume is scanned)
    int32_t pad;
    double u_cls, u_adj[3];
};
struct FgLaunch {
    FgDraw d[kMax3D];        // per sample of the Img3dLaunch
    // (filled by launch_fg_scan) the scanned samples' planes as one flat grid: CTA x
    // scans plane x - scan_start[k] of sample scan_i[k]; no CTA for unscanned samples
    int32_t n_scan;
    int32_t scan_i[kMax3D];
    int32_t scan_start[kMax3D + 1];
};
cudaError_t launch_fg_scan(const Img3dLaunch& L, const FgLaunch& F, int32_t* box, cudaStream_t s);
cudaError_t launch_fg_offsets(const Img3dLaunch& L, const FgLaunch& F, const int32_t* box, int4* offs,
                              cudaStream_t s);
// encodes L.tm_img[i] / L.tm_lbl[i] for a D,H,W f32 volume + u8 label (see img3d_tma_ok)
cudaError_t img3d_encode_maps(Img3dLaunch& L, int i, const void* img, const void* lbl,
                              const int64_t dims[3]);
cudaError_t launch_rrc2d(const RrcLaunch& L, cudaStream_t s);
cudaError_t launch_spin(const SpinLaunch& L, cudaStream_t s);
cudaError_t launch_gather(const GatherLaunch& L, cudaStream_t s);
cudaError_t launch_trainer_spin(int64_t ns, int ctas, cudaStream_t s);
int rrc2d_smem_bytes(const RrcLaunch& L);

// Force module loading at context creation: with lazy loading the first launch
// of a kernel loads its module, which can stall the shard loop mid-run.
cudaError_t warm_stage();
cudaError_t warm_img3d();
cudaError_t warm_img3d_zoom();
cudaError_t warm_rrc2d();
cudaError_t warm_misc();

// speech: constant tables (window, DFT basis, mel filterbank) live in device memory
struct SpeechTables;
cudaError_t speech_tables_create(SpeechTables** out);
void speech_tables_destroy(SpeechTables* t);
cudaError_t launch_speech(const SpLaunch& L, const SpeechTables* t, cudaStream_t s);
cudaError_t launch_speech_collate(const SpCollate& C, cudaStream_t s);
int speech_frames_per_cta();
cudaError_t warm_speech();

// synthetic data (Philox(seed, id)); device kernels
cudaError_t launch_synth_volume(uint64_t seed, uint64_t id, int64_t D, int64_t H, int64_t W,
                                float* img, uint8_t* lbl, cudaStream_t s);
cudaError_t launch_synth_image(uint64_t seed, uint64_t id, int64_t H, int64_t W, uint8_t* hwc,
                               cudaStream_t s);
cudaError_t launch_synth_waveform(uint64_t seed, uint64_t id, int64_t L, float* wav,
                                  cudaStream_t s);

}  // namespace lfg
