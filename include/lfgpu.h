/*
 * lfgpu.h -- C ABI of the B200-native MinatoLoader preprocessing hot path.
 *
 * One context per GPU.  Plain pointers, sizes and int error codes; no C++
 * types and no exceptions cross this boundary.  Every entry point returns
 * LFG_OK (0) or a negative LFG_ERR_*; lfg_last_error() gives a thread-local
 * message for the last failure on the calling thread.
 *
 * The reference (/root/reference/proj) has no C ABI or FFI; its boundary is
 * the C++ API in proj/include/loadflow.  Each entry point below names the
 * reference function/type whose role it takes over on the GPU path, and the
 * C++ adapter in include/loadflow/ (our signature-compatible headers) calls
 * these entry points underneath the reference-shaped API.
 * shows the binding a maintainer would add on the reference side.
 *
 * Error codes map onto the reference's exceptions:
 *   LFG_ERR_INVALID  std::invalid_argument  (sample.cpp:27-33, balancer.cpp:83-89, batcher.cpp:43)
 *   LFG_ERR_STATE    std::logic_error       (balancer.cpp:16)
 *   LFG_ERR_CLOSED   QueueClosedError       (queue.hpp:29-33)
 *   LFG_ERR_AGAIN    a bounded resource is full (BoundedQueue::put would block, queue.hpp:57-59)
 *   LFG_ERR_CUDA     CUDA runtime failure (no reference analogue; realtime "partial", experiment.cpp:331-340)
 */
#ifndef LFGPU_H
#define LFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFG_ABI_VERSION 5   /* 2: run config percentile / scheduler fields, report scheduler fields, lfg_run_shard_source;
                               3: run config prefetch_factor;
                               4: run config output capture (capture_pos / capture_buf / ...);
                               5: streaming shard runs (lfg_shard_start / lfg_shard_next_batch / lfg_shard_finish),
                                  lfg_config.coalesce_us (was reserved0) */

#define LFG_OK 0
#define LFG_ERR_INVALID -1
#define LFG_ERR_STATE -2
#define LFG_ERR_CLOSED -3
#define LFG_ERR_AGAIN -4
#define LFG_ERR_CUDA -5
#define LFG_ERR_NOMEM -6
#define LFG_ERR_UNSUPPORTED -7

/* ---- transform op kinds: 1:1 with the reference Transform::name values ---- */
enum {
    /* img_seg chain, proj/src/workloads.cpp:142-148 */
    LFG_OP_RANDOM_CROP = 1,       /* param: crop_d, crop_h, crop_w, p_fg (foreground oversampling,
                                     MLPerf RandBalancedCrop; 0 = plain random crop) */
    LFG_OP_RANDOM_FLIP = 2,       /* param: p_flip                          */
    LFG_OP_RANDOM_BRIGHTNESS = 3, /* param: p, lo, hi                       */
    LFG_OP_GAUSSIAN_NOISE = 4,    /* param: p, std_max                      */
    LFG_OP_CAST = 5,              /* no params: img f32, label u8           */
    /* optional img_seg ops (north_star "trilinear resize", "brightness/contrast";
     * not in the reference chain): chain order Crop, Zoom3D, Flip, Brightness,
     * Contrast, Noise, Cast */
    LFG_OP_RANDOM_ZOOM3D = 6,     /* param: p, lo, hi: window = round(crop*f), trilinear back to crop */
    LFG_OP_RANDOM_CONTRAST = 7,   /* param: p, lo, hi: (v - mean) * f + mean over the crop */
    /* obj_det chain, proj/src/workloads.cpp:151-156 */
    LFG_OP_RESIZE = 10,           /* RandomResizedCrop; param: out_h, out_w, scale_lo, scale_hi, ratio_lo, ratio_hi */
    LFG_OP_RANDOM_HFLIP = 11,     /* param: p                               */
    LFG_OP_TO_TENSOR = 12,        /* no params                              */
    LFG_OP_NORMALIZE = 13,        /* param: mean[3], std[3]                 */
    /* speech chain, proj/src/workloads.cpp:103-111 */
    LFG_OP_PAD = 20,
    LFG_OP_SPEC_AUGMENT = 21,     /* param: n_freq, freq_max, n_time, time_frac */
    LFG_OP_FILTER_BANK = 22,      /* param: n_fft, win, hop, n_mels, max_len, input type (LFG_DT_F32 /
                                     0, or LFG_DT_I16: 16-bit PCM read as s / 32768) */
    LFG_OP_FRAME_SPLICING = 23,   /* param: stack (=subsample)              */
    LFG_OP_PERMUTE_AUDIO = 24,
    /* synthetic cost steps (LightStep/HeavyStep, workloads.cpp:109-110; and the
     * per-sample step_costs of synthetic chains): a %globaltimer spin whose
     * length is the sample's cost for this op (lfg_sample_desc.spin_us[k]) */
    LFG_OP_SPIN = 30
};

/* Transform, proj/include/loadflow/sample.hpp:30-38 (name, size_factor, barrier).
 * `param` carries the op's configuration (see the enum comments); unused = 0. */
typedef struct {
    int32_t kind;
    int32_t barrier;
    double size_factor;
    double param[8];
    char name[32];
} lfg_op;

enum { LFG_DT_U8 = 1, LFG_DT_I16 = 2, LFG_DT_F32 = 3 };

/* Where a sample's raw bytes live when it is submitted. */
enum {
    LFG_SRC_DEVICE = 0,      /* already resident in HBM (caller-owned device memory) */
    LFG_SRC_HOST_PINNED = 1  /* pinned host staging (lfg_host_alloc); H2D happens on the
                                sample's stream, only the bytes the chain reads are copied */
};

/* Per-sample input description (the fields of reference Sample that the
 * device path needs: id and the raw payload; sample.hpp:40-55). */
typedef struct {
    uint64_t id;
    int32_t src_kind;        /* LFG_SRC_* */
    int32_t ndim;            /* 3 (volume D,H,W), 3 (image H,W,C=3) or 1 (waveform L) */
    int64_t dims[4];
    const void* data;        /* primary payload: img f32 / image u8 HWC / waveform f32 */
    const void* aux;         /* secondary payload: u8 label volume for img_seg; else NULL */
    int64_t spin_us[4];      /* synthetic cost (microseconds) of the chain's LFG_OP_SPIN ops, in op order */
} lfg_sample_desc;

/* Context configuration.  n_workers is the reference PoolConfig::max_workers
 * analogue (worker_pool.hpp:12-15): the number of concurrently in-flight,
 * not-yet-slow launch groups, each on its own stream. */
typedef struct {
    int32_t device;
    int32_t n_workers;          /* in-flight launch groups (streams), default 12 */
    int32_t max_group;          /* samples per launch group (multi-sample launch), default 1 */
    int32_t batch_size;         /* slot-buffer capacity = batch size */
    int32_t max_slot_buffers;   /* bound on live output batch buffers (HBM budget) */
    int32_t coalesce_us;        /* ABI 5: > 0 = lfg_flush launches an open launch group only once
                                   it is full (max_group) or its first sample has waited this
                                   long; lfg_progress launches a due group, lfg_wait at once.
                                   Per-sample submitters (process_sample workers) then share
                                   launches instead of one launch per sample.  0 = flush launches */
    uint64_t seed;              /* per-sample Rng: mt19937_64(seed ^ 0x9e3779b97f4a7c15*(id+1)) */
    int64_t max_raw_bytes;      /* bound on one group's raw staging (0 = auto) */
} lfg_config;

typedef struct lfg_ctx lfg_ctx;
typedef struct lfg_chain lfg_chain;
typedef int64_t lfg_ticket;     /* >= 0; one per submitted sample */
typedef int64_t lfg_batch;      /* >= 0; one per sealed batch */

/* ---- context ---- */
const char* lfg_last_error(void);
int lfg_abi_version(void);
int lfg_device_count(int* n);
void lfg_config_default(lfg_config* cfg);
int lfg_open(const lfg_config* cfg, lfg_ctx** out);
int lfg_close(lfg_ctx* ctx);
int lfg_synchronize(lfg_ctx* ctx);

/* ---- memory helpers (caller-owned buffers) ---- */
int lfg_host_alloc(lfg_ctx* ctx, size_t bytes, void** out);     /* pinned */
int lfg_host_free(lfg_ctx* ctx, void* p);
int lfg_device_alloc(lfg_ctx* ctx, size_t bytes, void** out);
int lfg_device_free(lfg_ctx* ctx, void* p);
int lfg_memcpy_h2d(lfg_ctx* ctx, void* dst, const void* src, size_t bytes);
int lfg_memcpy_d2h(lfg_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ---- chains: TransformChain (sample.hpp:57-77) ----
 * Validates the op list and compiles it into fused launch stages (one CUDA
 * kernel per stage).  out_bytes = bytes of one sample's output slot. */
int lfg_chain_create(lfg_ctx* ctx, const lfg_op* ops, int n_ops, lfg_chain** out);
int lfg_chain_destroy(lfg_ctx* ctx, lfg_chain* chain);
int lfg_chain_info(lfg_chain* chain, int* n_stages, int64_t* out_bytes, int* family);
/* stage s covers ops [stage_first[s], stage_last[s]) */
int lfg_chain_stage(lfg_chain* chain, int s, int* first_op, int* last_op);

/* ---- per-sample parameters (host draws, product side) ----
 * Writes the sample's drawn parameters as doubles (layout per family, see
 * DESIGN.md section 3) -- used by the parity tests to check the host draws
 * bit-exactly against the oracle. */
int lfg_draw_params(lfg_chain* chain, uint64_t seed, const lfg_sample_desc* s, double* out,
                    int cap, int* n_out);

/* The per-sample generator itself (host only, no GPU needed): the first n outputs
 * of std::mt19937_64(seed ^ 0x9e3779b97f4a7c15*(id+1)) as the product draws them
 * (a lazily seeded, bit-exact evaluation; checked against libstdc++ in the tests). */
int lfg_rng_outputs(uint64_t seed, uint64_t id, int n, uint64_t* out);

/* ---- submit / progress: replaces process_sample's transform loop
 * (balancer.cpp:42-77) and the worker slot (worker_pool.cpp:63-98).
 * lfg_submit draws the sample's parameters, assigns its output slot and adds
 * it to the chain's open launch group; lfg_flush launches open groups (a
 * group also launches when it reaches max_group).  Asynchronous. */
int lfg_submit(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* s, lfg_ticket* out);
int lfg_flush(lfg_ctx* ctx);

/* Non-blocking.  ops_done is the reference RouteResult::timeout_index analogue
 * (the index of the first transform not yet finished, at fused-stage
 * granularity); complete is 1 once the whole chain finished.  elapsed_us is
 * host wall time since the sample's group was launched. */
int lfg_progress(lfg_ctx* ctx, lfg_ticket t, int* ops_done, int* complete, int64_t* elapsed_us);
/* Blocks until the ticket's chain completes (resume_slow's wait, balancer.cpp:96-113). */
int lfg_wait(lfg_ctx* ctx, lfg_ticket t);
/* Waits up to timeout_us for the ticket's sample to finish, without holding the
 * context lock: *complete = 1 when it did.  A coalescing group still open is launched
 * once due; with coalesce_us > 0 launched groups wake their waiters by a completion
 * notice (host function after the group's last stage), so per-sample workers block
 * instead of polling (ABI 5).  The process_sample budget check: balancer.cpp:55. */
int lfg_wait_for(lfg_ctx* ctx, lfg_ticket t, int64_t timeout_us, int* complete);
/* Device-timed per-op costs in microseconds (one per op; ops fused into one
 * stage share the stage's time, attributed to the stage's last op). */
int lfg_exec_costs(lfg_ctx* ctx, lfg_ticket t, double* costs_us, int cap, int* n_out);
/* Copy a completed sample's output slot to host memory (tests). */
int lfg_ticket_output(lfg_ctx* ctx, lfg_ticket t, void* host_dst, size_t bytes);
/* Ends the caller's use of t.  A released handle is dead: once every ticket of the
 * context is released, the next lfg_run_shard reuses the ticket numbers. */
int lfg_ticket_release(lfg_ctx* ctx, lfg_ticket t);

/* ---- batches: build_batches seal (batcher.cpp:50-58) ----
 * Seals the given completed tickets, in order, into one device-resident
 * batch.  If the tickets are exactly the samples of one output slot buffer,
 * the batch is that buffer (zero copy); otherwise one gather kernel collates
 * them into a fresh batch buffer.  The tickets are consumed. */
int lfg_seal_batch(lfg_ctx* ctx, const lfg_ticket* tickets, int n, lfg_batch* out);
/* Device pointer of the batch tensor, its byte size, sample count, ids in
 * batch order (ids may be NULL), and whether the seal was zero-copy. */
int lfg_batch_info(lfg_ctx* ctx, lfg_batch b, void** dev_ptr, int64_t* bytes, int* n,
                   uint64_t* ids, int* in_place);
/* Makes `stream` (a cudaStream_t, may be NULL = legacy) wait until the batch is resident. */
int lfg_batch_wait_stream(lfg_ctx* ctx, lfg_batch b, void* stream);
int lfg_batch_copy_to_host(lfg_ctx* ctx, lfg_batch b, void* host_dst, size_t bytes);
/* Speech batches (PermuteAudio + Pad, proj/src/workloads.cpp:107-108) are
 * time-major [t_max, n, stack*80] f32, zero-padded: lengths[i] = T'_i. */
int lfg_batch_lengths(lfg_ctx* ctx, lfg_batch b, int32_t* lengths, int32_t* t_max);
/* Returns the batch buffer to the pool once work already queued on `stream`
 * (the consumer) has finished with it. */
int lfg_batch_release(lfg_ctx* ctx, lfg_batch b, void* stream);

/* ---- synthetic trainer step (trainer.cpp:50-51 consumer compute): a
 * device-clock spin of `us` microseconds on `stream` after the batch is resident. */
int lfg_trainer_step(lfg_ctx* ctx, lfg_batch b, void* stream, int64_t us);

/* ---- synthetic input generators (bench / tests data source; Philox(seed, id)) ---- */
int lfg_synth_volume(lfg_ctx* ctx, uint64_t seed, uint64_t id, int64_t D, int64_t H, int64_t W,
                     void* img_f32, void* lbl_u8, int on_device);
int lfg_synth_image(lfg_ctx* ctx, uint64_t seed, uint64_t id, int64_t H, int64_t W, void* hwc_u8,
                    int on_device);
int lfg_synth_waveform(lfg_ctx* ctx, uint64_t seed, uint64_t id, int64_t L, void* wav_f32,
                       int on_device);

/* ---- counters for the end-of-run reduce (the only NCCL use) ---- */
typedef struct {
    int64_t submitted, completed, fast, slow;
    int64_t batches, short_batches, inplace_batches, gathered_batches;
    int64_t launches;           /* CUDA kernels launched by this context */
    int64_t h2d_bytes, d2h_bytes;
    int64_t kernel_bytes;       /* algorithmic HBM bytes of the transform kernels */
    int64_t reserved[4];
} lfg_counters;
int lfg_get_counters(lfg_ctx* ctx, lfg_counters* out);

/* Serial mode: every launch group runs on one stream, so per-stage CUDA
 * events time each kernel in isolation (used for the roofline measurement). */
int lfg_set_serial(lfg_ctx* ctx, int serial);

/* Roofline timing: submits the samples with launches deferred, then issues all
 * launch groups back to back on one stream; mean_ms = mean device time of one
 * transform-stage launch (CUDA events), bytes / flops = algorithmic totals. */
int lfg_time_kernels(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* samples, int n,
                     double* mean_ms, int64_t* launches, int64_t* bytes, int64_t* flops);

/* ---- event-driven shard runner: the whole Algorithm-1 loop for one GPU
 * (run_minato_pipeline, experiment.cpp:129-276, with workers -> streams,
 * resume -> completion events, batcher -> seal, consumer -> trainer stream). */
typedef struct {
    int32_t batch_size;
    int32_t policy;             /* 0 fixed t_out, 1 profiler (p75 -> p90 escalation),
                                   2 profiler at a fixed percentile (see `percentile`),
                                   3 synchronous baseline (start_sync_loader, baselines.cpp:12-151):
                                     batch k = the k-th B samples, sealed when all are done,
                                     in order -- head-of-line blocking, no timeouts */
    int64_t t_out_us;           /* fixed budget (policy 0) or initial budget (policy 1); <=0 = none */
    int64_t warmup_us;          /* profiler warm-up before the first percentile (profiler.hpp:41) */
    int64_t update_interval_us; /* profiler refresh period */
    int32_t window;             /* profiler window (profiler.hpp:40) */
    int32_t n_workers;          /* 0 = context default */
    int64_t trainer_us;         /* consumer compute per batch (trainer.hpp:15), 0 = drain only */
    int32_t trainer_priority;   /* 1 = high-priority trainer stream */
    int32_t warmup_batches;     /* batches excluded from the timed window */
    int32_t record_trace;       /* keep per-sample / per-batch records */
    int32_t d2h_probe;          /* read 16 bytes of every delivered batch back to the host
                                   on the trainer stream (end-to-end result check) */
    int32_t percentile;         /* policy 2: nearest-rank percentile of the window (1..100);
                                   the C5 timeout sweep (p50 / p75 / p90) */
    int32_t scheduler;          /* 1: adaptive in-flight group count (MinatoLoader Eq. 1-2,
                                   scheduler.cpp:16-58 via loadflow/sched_rule.h): n_workers is
                                   the initial count, grown / shrunk every sched_tick_us */
    int32_t max_workers;        /* scheduler upper bound (0 = 2 x n_workers, <= 28 streams) */
    int64_t sched_tick_us;      /* scheduler period (0 = 500 us) */
    int32_t prefetch_factor;    /* policy 3: at most prefetch_factor x n_workers batches fed ahead of
                                   the oldest unsealed batch (SyncLoaderConfig::prefetch_factor,
                                   baselines.cpp:115-151, pipeline.prefetch_factor); 0 = unbounded */
    /* Output capture (verification of delivered samples; ABI 4).  When a delivered
     * batch holds the sample fed at position capture_pos[k] of `samples`, that
     * sample's output -- exactly as it sits in the delivered batch tensor -- is
     * copied on the trainer stream to capture_buf + k * capture_stride (pinned host
     * memory, lfg_host_alloc): img_seg = f32 image then u8 label (the plane bytes
     * of lfg_chain_info's out_bytes), obj_det = f32 [3, oh, ow], speech = its T'_i
     * rows of the time-major batch, row-packed ([T'_i, stack * 80] f32).
     * capture_done[k] (may be NULL) is set to the sample's batch index + 1. */
    int32_t n_capture;
    int32_t sample_stamps;      /* 1: the transform kernels stamp each sample's completion, so the shard
                                   classifies and hands on per sample inside a launch group (costs a
                                   release fence per kernel part); 0: per sample only where the group's
                                   last kernel is a synthetic cost (always) or per sub-launch */
    const int64_t* capture_pos;
    void* capture_buf;
    int64_t capture_stride;
    int32_t* capture_done;
} lfg_run_config;

typedef struct {
    int64_t samples, batches, short_batches, fast, slow, inplace_batches;
    double elapsed_ms;          /* device time (trainer-stream events) of the timed window */
    double timed_samples;       /* samples consumed inside the timed window */
    double samples_per_s;
    double consumer_busy_ms, consumer_span_ms, consumer_idle_frac; /* ConsumerStats, trainer.hpp:30-47 */
    double final_t_out_us;
    int32_t final_percentile;
    int32_t exactly_once;       /* consumed ids == submitted ids, no duplicates */
    int64_t duplicates;
    double kernel_ms;           /* summed device time of transform stages in the timed window */
    int64_t h2d_bytes, d2h_bytes;
    int64_t launches;
    int32_t final_workers;      /* in-flight group limit at the end (scheduler) */
    int32_t sched_ticks;        /* scheduler decisions taken */
    double mean_workers;        /* time-average of the in-flight group limit */
    int32_t pct_up, pct_down;   /* profiler p75 -> p90 escalations / p90 -> p75 de-escalations (ABI 4) */
    int64_t profiled;           /* per-sample totals recorded into the profiler window (ABI 4) */
} lfg_run_report;

/* samples[i] are fed in order (the feeder, experiment.cpp:221-228).
 * consumed_ids (may be NULL, capacity n) receives ids in consumption order;
 * batch_sizes (may be NULL, capacity n) the size of each consumed batch;
 * sample_class (may be NULL, capacity n, indexed by position in `samples`)
 * receives 1 = fast, 2 = slow. */
int lfg_run_shard(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* samples, int64_t n,
                  const lfg_run_config* cfg, lfg_run_report* report, uint64_t* consumed_ids,
                  int32_t* batch_sizes, int32_t* sample_class);

/* ---- streaming input (raw reads from storage, the feeder of
 * experiment.cpp:221-228): the shard pulls samples in order from `next` as it has
 * free workers, and hands each sample back through `release` once the device no
 * longer reads its payload (its launch group completed), so a bounded pool of
 * pinned buffers can be refilled by reader threads while earlier samples run. */
typedef struct {
    void* user;
    /* fill *out with the next sample: returns 1 (a sample), 2 (not ready yet: the
     * shard keeps polling and sealing, and asks again), 0 (end) or < 0 (error) */
    int (*next)(void* user, lfg_sample_desc* out);
    void (*release)(void* user, uint64_t id);   /* may be NULL */
} lfg_source;

int lfg_run_shard_source(lfg_ctx* ctx, lfg_chain* chain, const lfg_source* src, int64_t n,
                         const lfg_run_config* cfg, lfg_run_report* report, uint64_t* consumed_ids,
                         int32_t* batch_sizes, int32_t* sample_class);

/* ---- streaming consumer (ABI 5): the shard loop runs on a library thread and each
 * sealed batch is handed to the caller, who is the trainer -- build_batches' output
 * queue and run_consumer's next_batch (batcher.cpp:50-58, trainer.cpp:7-18).  The
 * context lock is not held across the run: between loop passes the consumer's
 * lfg_batch_info / lfg_batch_wait_stream / lfg_batch_copy_to_host / lfg_batch_lengths
 * / lfg_batch_release calls interleave with sealing.  A batch stays the consumer's
 * until lfg_batch_release; the loop waits for a free batch buffer when all of
 * max_slot_buffers are held (back-pressure, BoundedQueue::put, queue.hpp:57-59).
 * While a run is active, lfg_submit / lfg_seal_batch / lfg_run_shard* /
 * lfg_time_kernels / lfg_chain_destroy / lfg_close on the context fail with
 * LFG_ERR_STATE.  cfg->trainer_us is ignored (the caller is the trainer);
 * captures and the d2h probe still run, ordered before the batch's ready event. */
typedef struct lfg_shard lfg_shard;
/* samples are copied; the payloads they point at must stay valid until finish */
int lfg_shard_start(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* samples, int64_t n,
                    const lfg_run_config* cfg, lfg_shard** out);
/* The next sealed batch in delivery order.  timeout_us < 0 waits indefinitely.
 * LFG_OK: *out (and *n, may be NULL) set; LFG_ERR_AGAIN: none within the timeout;
 * LFG_ERR_CLOSED: end of stream (every sample delivered; QueueClosedError,
 * queue.hpp:29-33); another code: the run failed (lfg_last_error). */
int lfg_shard_next_batch(lfg_shard* sh, int64_t timeout_us, lfg_batch* out, int* n);
/* Waits for the run to end, releasing batches the consumer did not take (release every
 * batch you took first: batches you hold keep their buffers, and a loop waiting for a
 * buffer cannot end), fills
 * the report (consumer_busy/span/idle from the caller's time blocked in
 * lfg_shard_next_batch, as ConsumerStats, trainer.hpp:30-47) and the optional
 * arrays as lfg_run_shard does, and frees the handle (also on error). */
int lfg_shard_finish(lfg_shard* sh, lfg_run_report* report, uint64_t* consumed_ids, int32_t* batch_sizes,
                     int32_t* sample_class);

#ifdef __cplusplus
}
#endif

#endif /* LFGPU_H */
