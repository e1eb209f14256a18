/*
 * lf_oracle.h -- CPU restatement (test infrastructure ONLY) of the MinatoLoader
 * per-sample transform chains that the B200 path implements as CUDA kernels.
 *
 * THIS IS A CHECKER, NOT A PRODUCT PATH.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Provenance / parity status
 * --------------------------
 * The reference (/root/reference/proj) names the transforms and their size
 * factors but contains no transform arithmetic:
 *   img_seg chain  RandomCrop .0735, RandomFlip, RandomBrightness,
 *                  GaussianNoise, Cast            (proj/src/workloads.cpp:142-148)
 *   obj_det chain  Resize 1.2, RandomHorizontalFlip, ToTensor 8.0, Normalize
 *                                                 (proj/src/workloads.cpp:151-156)
 *   speech chain   Pad 1.12, SpecAugment, FilterBank, FrameSplicing .9,
 *                  PermuteAudio, LightStep, HeavyStep (proj/src/workloads.cpp:103-111)
 * The real-function extension point is Transform::apply over an fp64
 * Payload (proj/include/loadflow/sample.hpp:23,35), so this oracle computes in
 * fp64.  The per-sample generator is the reference's Rng = std::mt19937_64
 * (sample.hpp:25) seeded per sample id with the mixing constant of
 * proj/src/experiment.cpp:163:  seed ^ (0x9e3779b97f4a7c15 * (id + 1)).
 *
 * Pixel/voxel/audio values are therefore "parity unpinned" with respect to the
 * reference itself (it has no golden vectors for them).  The formulas below
 * restate the public algorithms the paper's pipelines use (MLPerf 3D-UNet
 * transforms, torchvision RandomResizedCrop / bilinear resize, torchaudio
 * spectrogram + slaney mel) and are cross-checked against torch / torchvision /
 * torchaudio CPU in tests/test_oracle.py.  The generators (mt19937_64,
 * Philox4x32-10) are pinned by known-answer vectors.
 *
 * Exact semantics (the contract the CUDA kernels must meet) are documented at
 * each function below and in DESIGN.md section 3.
 */
#ifndef LF_ORACLE_H
#define LF_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------- generators ---------------- */

typedef struct {
    uint64_t mt[312];
    int idx;
} lfo_mt64;

void lfo_mt64_seed(lfo_mt64* g, uint64_t seed);
uint64_t lfo_mt64_next(lfo_mt64* g);

/* per-sample generator: mt19937_64(seed ^ (0x9e3779b97f4a7c15 * (id + 1))) */
void lfo_sample_rng(lfo_mt64* g, uint64_t seed, uint64_t id);

/* draw primitives on raw 64-bit outputs (portable, builder-defined) */
double lfo_unif01(lfo_mt64* g);                        /* (u >> 11) * 2^-53 */
int64_t lfo_randint(lfo_mt64* g, int64_t lo, int64_t hi); /* lo + floor(unif01*(hi-lo+1)) */
double lfo_uniform(lfo_mt64* g, double a, double b);   /* a + (b-a)*unif01 */

/* Philox4x32-10 (Salmon et al., SC'11; Random123 reference constants) */
void lfo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Box-Muller normals for Philox counter group g (4 normals per group). */
void lfo_normals4(uint64_t group, uint32_t k0, uint32_t k1, double z[4]);

/* ---------------- img_seg (3D) chain ---------------- */

typedef struct {
    int64_t crop[3];        /* crop edge per axis (d, h, w); default 128 */
    double p_flip;          /* per-axis flip probability, default 1/3 (MLPerf RandFlip) */
    double p_bright;        /* default 0.1 (MLPerf RandomBrightnessAugmentation) */
    double bright_lo, bright_hi; /* default 0.7, 1.3 */
    double p_noise;         /* default 0.1 (MLPerf GaussianNoise) */
    double noise_std_max;   /* default 0.1 */
    /* optional ops (north_star "trilinear resize", "brightness/contrast"; not in
     * the reference's img_seg chain, so off by default and their draws are
     * skipped: the default chain's draw sequence is unchanged) */
    int32_t has_zoom;       /* RandomZoom3D after RandomCrop */
    double p_zoom;          /* default 0.5 */
    double zoom_lo, zoom_hi;/* default 0.8, 1.2 (window edge = round(crop * f)) */
    int32_t has_contrast;   /* RandomContrast after RandomBrightness */
    double p_contrast;      /* default 0.15 (nnU-Net ContrastAugmentation) */
    double contrast_lo, contrast_hi; /* default 0.75, 1.25 */
    /* RandomCrop's foreground oversampling (MLPerf 3D-UNet RandBalancedCrop): with
     * probability p_fg the window is placed around a random foreground class
     * (labels 1..7) -- see lfo_fg_offsets */
    int32_t has_fg;
    double p_fg;            /* default 0.4 (MLPerf oversampling) */
} lfo_cfg3d;

typedef struct {
    int64_t off[3];         /* window origin per axis (0 when dim < window: zero pad) */
    int32_t flip[3];        /* flip flags per axis */
    double scale;           /* brightness multiplier (1.0 when not applied) */
    double sigma;           /* noise std (0.0 when not applied) */
    uint32_t key[2];        /* Philox key */
    int64_t win[3];         /* source window edge per axis (= crop unless zoomed) */
    double contrast;        /* contrast factor (1.0 when not applied) */
    int32_t fg;             /* foreground-biased crop drawn for this sample */
    double u_cls, u_adj[3]; /* its uniforms: class choice, per-axis placement */
} lfo_params3d;

void lfo_cfg3d_default(lfo_cfg3d* c);
void lfo_draw3d(const lfo_cfg3d* c, uint64_t seed, uint64_t id, const int64_t dims[3],
                lfo_params3d* p);
/* img f32 [D,H,W], lbl u8 [D,H,W] -> out_img f64 [cd,ch,cw], out_lbl u8.
 * Zoomed windows (win != crop) are resampled to the crop: image trilinear
 * (PyTorch upsample_trilinear3d, align_corners=False, source index in fp64),
 * label nearest with the integer index min(dst * win / crop, win - 1). */
void lfo_apply3d(const lfo_cfg3d* c, const lfo_params3d* p, const float* img,
                 const uint8_t* lbl, const int64_t dims[3], double* out_img,
                 uint8_t* out_lbl);
/* Window origin of a foreground-biased crop (MLPerf RandBalancedCrop, with the
 * bounding box of ALL voxels of the chosen class instead of its two largest
 * connected components): classes present = labels 1..7 found in the volume,
 * ascending; cl = present[floor(u_cls * n)]; per axis with the class box [lo, hi):
 *   diff = win - (hi - lo), sign = diff < 0 ? -1 : 1, diff = |diff|,
 *   ladj = floor(u_adj * diff), hadj = diff - ladj,
 *   low = max(0, lo - sign*ladj), high = min(dim, hi + sign*hadj),
 *   d2 = win - (high - low); if d2 > 0: (low == 0 ? high += d2 : low -= d2),
 *   off = clamp(low, 0, max(dim - win, 0)).
 * Returns 0 (off[] written) or -1 (not drawn / no foreground: the random offsets hold). */
int lfo_fg_offsets(const lfo_params3d* p, const uint8_t* lbl, const int64_t dims[3], int64_t off[3]);

/* ---------------- obj_det / ImageNet (2D) chain ---------------- */

typedef struct {
    int32_t out_h, out_w;   /* default 224 x 224 */
    double scale_lo, scale_hi; /* default 0.08, 1.0 */
    double ratio_lo, ratio_hi; /* default 3/4, 4/3 */
    double p_hflip;         /* default 0.5 */
    double mean[3], std[3]; /* ImageNet */
} lfo_cfg2d;

typedef struct {
    int64_t top, left, h, w; /* crop box in the source */
    int32_t flip;
} lfo_params2d;

void lfo_cfg2d_default(lfo_cfg2d* c);
void lfo_draw2d(const lfo_cfg2d* c, uint64_t seed, uint64_t id, int64_t H, int64_t W,
                lfo_params2d* p);
/* src u8 HWC [H,W,3] -> out f64 CHW [3,out_h,out_w] */
void lfo_apply2d(const lfo_cfg2d* c, const lfo_params2d* p, const uint8_t* src, int64_t H,
                 int64_t W, double* out);
/* bilinear only (no normalize / flip): float CHW crop -> f64 CHW; for torch cross-check */
void lfo_bilinear_chw(const float* src, int64_t C, int64_t H, int64_t W, int64_t oh,
                      int64_t ow, double* out);

/* ---------------- speech chain ---------------- */

typedef struct {
    int32_t n_fft;          /* 512 */
    int32_t win_length;     /* 320 (20 ms at 16 kHz) */
    int32_t hop;            /* 160 */
    int32_t n_mels;         /* 80 */
    double sample_rate;     /* 16000 */
    double f_min, f_max;    /* 0, 8000 */
    double log_eps;         /* 2^-24 */
    int32_t freq_masks;     /* 2 */
    int32_t freq_mask_max;  /* 27 */
    int32_t time_masks;     /* 10 */
    double time_mask_frac;  /* 0.05 */
} lfo_cfgsp;

typedef struct {
    int32_t n_frames;
    int32_t f_lo[8], f_w[8];   /* freq masks [f_lo, f_lo+f_w) */
    int32_t t_lo[32], t_w[32]; /* time masks */
    int32_t n_fmask, n_tmask;
} lfo_paramssp;

void lfo_cfgsp_default(lfo_cfgsp* c);
int32_t lfo_sp_frames(const lfo_cfgsp* c, int64_t L);
void lfo_drawsp(const lfo_cfgsp* c, uint64_t seed, uint64_t id, int64_t L, lfo_paramssp* p);
/* slaney mel filterbank [n_mels, n_fft/2+1] row-major, f64 */
void lfo_mel_fbank(const lfo_cfgsp* c, double* fb);
/* waveform f32 [L], L > n_fft/2 (reflect padding) -> log-mel f64 [n_mels, T] (masked),
 * also power f64 [n_fft/2+1, T] if non-null */
void lfo_applysp(const lfo_cfgsp* c, const lfo_paramssp* p, const float* wav, int64_t L,
                 double* logmel, double* power);

#ifdef __cplusplus
}
#endif

#endif
