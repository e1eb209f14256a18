// engine.h -- internal C++ engine behind the lfgpu C ABI.
//
// Objects (all owned by one Context = one GPU):
//   Chain      compiled transform chain (reference TransformChain) -> fused stages
//   Group      a launch group: 1..max_group samples sharing one stream and one
//              kernel launch per stage, with a CUDA event after every stage
//   Ticket     one submitted sample: drawn params, output slot, group
//   SlotBuf    a device buffer of batch_size output slots (planar); samples are
//              written straight into it and a batch sealed from exactly its
//              samples is handed over in place (zero copy)
//   BatchRec   a sealed batch: slot buffer + ids + ready event
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <thread>
#include <deque>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/lfgpu.h"
#include "kernels.h"

namespace lfg {

enum Family { FAM_NONE = 0, FAM_IMG3D = 1, FAM_RRC2D = 2, FAM_SPEECH = 3 };
enum StageKind { ST_SPIN = 1, ST_IMG3D = 2, ST_RRC2D = 3, ST_SPEECH = 4 };

struct Error {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);

int64_t host_now_us();

// Chain-keyed map for the submit path: a context holds a handful of chains,
// so a linear scan of a small vector beats hashing (submit runs per sample).
struct Chain;
template <class V>
struct SmallMap {
    using Item = std::pair<const Chain*, V>;
    std::vector<Item> v;
    using iterator = typename std::vector<Item>::iterator;
    iterator begin() { return v.begin(); }
    iterator end() { return v.end(); }
    iterator find(const Chain* k) {
        for (auto it = v.begin(); it != v.end(); ++it)
            if (it->first == k) return it;
        return v.end();
    }
    V& operator[](const Chain* k) {
        auto it = find(k);
        if (it != v.end()) return it->second;
        v.emplace_back(k, V{});
        return v.back().second;
    }
    void erase(iterator it) { v.erase(it); }
    void erase(const Chain* k) {
        auto it = find(k);
        if (it != v.end()) v.erase(it);
    }
    size_t size() const { return v.size(); }
    void clear() { v.clear(); }
};

struct Stage {
    int kind;
    int first_op, last_op;   // ops [first, last) covered by this stage
    std::vector<int> spin_ops;  // spin slot indices launched in this stage (in order)
};

struct Chain {
    std::vector<lfg_op> ops;
    int64_t est_group_us = 0;   // shard runs: the group-time estimate of the query throttle, kept across runs
    Family fam = FAM_NONE;
    std::vector<Stage> stages;
    int n_spin = 0;
    // img3d
    int crop[3] = {128, 128, 128};
    double p_flip = 0, p_bright = 0, b_lo = 1, b_hi = 1, p_noise = 0, noise_max = 0;
    bool has_zoom = false, has_contrast = false;     // optional RandomZoom3D / RandomContrast
    bool has_fg = false;                              // RandomCrop foreground oversampling (K2)
    double p_fg = 0;
    double p_zoom = 0, z_lo = 1, z_hi = 1, p_contrast = 0, c_lo = 1, c_hi = 1;
    // rrc2d
    int oh = 224, ow = 224;
    double scale_lo = 0.08, scale_hi = 1.0, ratio_lo = 0.75, ratio_hi = 4.0 / 3.0, p_hflip = 0;
    double mean[3] = {0, 0, 0}, std[3] = {1, 1, 1};
    bool to_tensor = false;
    // speech
    int n_fft = 512, win = 320, hop = 160, n_mels = 80, stack = 3;
    int n_fmask = 0, fmask_max = 0, n_tmask = 0;
    double tmask_frac = 0;
    int64_t max_L = 170000;
    int wav_bytes = 4;             // waveform element: 4 = f32, 2 = int16 PCM (full scale 32768)
    // output slot layout (planar)
    bool spin_last = false;        // the last stage ends in a synthetic-cost spin (stamps)
    int nplanes = 1;
    int64_t plane_bytes[2] = {0, 0};
    int64_t out_bytes = 0;
    int64_t algo_bytes_per_sample(const lfg_sample_desc& s) const;
};

// Per-sample drawn parameters (host, std::mt19937_64 keyed by sample id).
struct Params3D {
    int64_t off[3];
    int flip[3];
    double scale, sigma;
    uint32_t key[2];
    int64_t win[3];       // source window edge (RandomZoom3D; = crop otherwise)
    double contrast;      // RandomContrast factor (1 = not applied)
    int fg;               // foreground-biased crop drawn: the window origin comes from K2
    double u_cls, u_adj[3];
};
struct Params2D { int64_t top, left, h, w; int flip; int64_t rows_touched; };
struct ParamsSp { int T; int f_lo[2], f_w[2]; int t_lo[10], t_w[10]; };

void draw_3d(const Chain& c, uint64_t seed, uint64_t id, const int64_t dims[3], Params3D& p);
void draw_2d(const Chain& c, uint64_t seed, uint64_t id, int64_t H, int64_t W, Params2D& p);
void draw_sp(const Chain& c, uint64_t seed, uint64_t id, int64_t L, ParamsSp& p);

// One sample's drawn parameters (whichever family applies); pure function of
// (chain, seed, sample id, dims), so the shard runner draws them ahead of time
// on a host thread pool.
// One sample's drawn parameters (the chain's family only).  Deliberately not
// zero-initialised: a run allocates n of these up front and the draw threads
// write (and first-touch) each one, so the submitting thread never pays for
// clearing or faulting in the table.
struct PreDraw {
    union {
        Params3D p3;
        Params2D p2;
        ParamsSp ps;
    };
    PreDraw() {}
};
void draw_params(const Chain& c, uint64_t seed, const lfg_sample_desc& s, PreDraw& out);
// the first n outputs of sample `id`'s generator (lfg_rng_outputs)
void rng_outputs(uint64_t seed, uint64_t id, int n, uint64_t* out);
int64_t rrc_algo_bytes(const Chain& c, const Params2D& p);

struct SlotBuf {
    char* base = nullptr;
    int cap = 0;
    int assigned = 0;        // slots handed to tickets
    int live = 0;            // assigned tickets whose bytes are still needed here
    bool open = false;       // still accepting slot assignments
    bool in_batch = false;   // owned by a sealed batch
    std::vector<cudaEvent_t> pending;  // readers that must finish before reuse
    const Chain* chain = nullptr;
    int64_t bytes = 0;
    bool gather_role = false;  // created as a collation target (not a sample slot buffer)
};

struct RawBuf {
    char* ptr = nullptr;
    int64_t cap = 0;
};

struct Group {
    int64_t id = 0;
    Chain* chain = nullptr;
    int src_kind = LFG_SRC_DEVICE;
    std::vector<int64_t> tickets;
    int stream_idx = -1;
    cudaStream_t stream = nullptr;
    std::vector<cudaEvent_t> ev;   // ev[0] start, ev[s+1] end of stage s
    bool launched = false;
    bool complete = false;
    int stages_done = 0;
    int64_t t_launch_us = 0;
    int64_t t_open_us = 0;       // first submit (coalescing deadline, lfg_config.coalesce_us)
    int64_t t_query_us = 0;      // last event query from lfg_progress (poll throttle)
    int64_t serial = 0;          // launch serial (> 0 once launched; the completion ring's key)
    int64_t raw_idx = -1;
    int refs = 0;
    bool timed = true;             // stage events carry timing (Context::time_groups at launch)
    std::vector<float> stage_ms;   // filled once complete (zeros when untimed)
    // per-sample completion: the group's last kernel writes one stamp per sample
    // (Context::sample_stamp); the shard delivers samples as their stamps land
    bool stamped = false;
    int n_got = 0;                 // samples handed on by the shard
    int scan_from = 0;             // first sample not yet handed on (in order)
    std::vector<uint8_t> got;      // per sample: handed on
    // a sub-launch that completes some samples early (the plain samples of a group
    // split around foreground-crop label scans): its event and the samples it covers
    cudaEvent_t part_ev = nullptr;
    std::vector<int> part_idx;
    bool part_done = false;        // the part event completed
    bool part_handed = false;      // (shard) the part's samples were handed on
    float part_ms = 0.0f;          // device time from the group's start to the part event
    bool part_ready() {
        if (!part_done && part_ev != nullptr) part_done = cudaEventQuery(part_ev) == cudaSuccess;
        return part_done;
    }
};

struct Ticket {
    uint64_t id = 0;
    int64_t group = -1;
    // the sample's descriptor and drawn parameters: the shard runner's run arrays
    // (alive until the run's tickets are released) or context-owned copies (lfg_submit);
    // a ticket is one cache line, so the per-sample submit writes ~48 B
    const lfg_sample_desc* dp = nullptr;
    const PreDraw* pp = nullptr;
    int idx = 0;
    int buf = -1, pos = -1;
    bool released = false;
    bool consumed = false;   // sealed into a batch
    bool in_seal = false;    // scratch mark for seal's duplicate check
    const lfg_sample_desc& desc() const { return *dp; }
    const Params3D& p3() const { return pp->p3; }
    const Params2D& p2() const { return pp->p2; }
    const ParamsSp& ps() const { return pp->ps; }
};

struct BatchRec {
    int buf = -1;
    bool in_place = false;
    std::vector<uint64_t> ids;
    cudaEvent_t ready = nullptr;
    const Chain* chain = nullptr;
    int n = 0;
    bool released = false;
    int t_max = 0;               // speech: padded time length of the batch tensor
    std::vector<int> rows;       // speech: per-sample spliced lengths T'_i
};

// Host worker threads owned by a context (created once at lfg_open): the shard
// runner hands them the per-sample parameter draws of each run, so no run pays
// for spawning threads.  run(f) starts f on every worker; wait() returns once all
// of them have finished it.
class WorkerThreads {
public:
    explicit WorkerThreads(int n);
    ~WorkerThreads();
    int size() const { return static_cast<int>(th_.size()); }
    void run(std::function<void(int)> f);
    void wait();

private:
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, idle_;
    std::function<void(int)> job_;
    uint64_t gen_ = 0;
    int busy_ = 0;
    bool quit_ = false;
};

// Streaming delivery (lfg_shard_start / lfg_shard_next_batch): the shard loop holds
// `lock` (the context lock) except between passes, so the consumer's batch calls
// (info / wait / release) interleave with it, and each sealed batch goes to
// deliver() instead of the internal trainer -- the consumer releases it.
struct ShardStream {
    std::mutex* lock = nullptr;
    void (*deliver)(void* user, int64_t batch, int n) = nullptr;
    void* user = nullptr;
};

class Context {
public:
    explicit Context(const lfg_config& cfg);
    ~Context();

    lfg_config cfg;
    int sm_count = 148;

    Chain* chain_create(const lfg_op* ops, int n);
    void chain_destroy(Chain* c);

    int64_t submit(Chain* c, const lfg_sample_desc& s, const PreDraw* pre = nullptr);
    void flush();
    // lfg_flush: with coalesce_us > 0 only groups open that long (or full) launch
    void flush_due();
    void progress(int64_t t, int* ops_done, int* complete, int64_t* elapsed_us);
    void wait(int64_t t);                 // blocking; callers must not hold `mu` (see lfg_wait)
    bool launch_if_pending(int64_t t);    // launches t's open group if needed; true if complete
    int exec_costs(int64_t t, double* out, int cap);
    void ticket_output(int64_t t, void* dst, size_t bytes);
    void ticket_release(int64_t t);

    int64_t seal(const int64_t* tickets, int n);
    BatchRec& batch(int64_t b);
    void batch_wait_stream(int64_t b, cudaStream_t s);
    void batch_release(int64_t b, cudaStream_t s, bool readers = true);
    void trainer_step(int64_t b, cudaStream_t s, int64_t us);
    // Copies the sample at batch position `pos` out of the delivered batch tensor
    // into pinned host memory on `s` (after the batch is resident there); returns
    // the bytes copied (lfg_run_config capture layout).
    int64_t capture_sample(int64_t b, int pos, char* dst, int64_t cap_bytes, cudaStream_t s);
    // samples assigned to slot buffer bi once it stopped accepting new ones; -1 otherwise
    int buf_closed_count(int bi) const {
        const SlotBuf& b = bufs_[bi];
        return (b.open || b.in_batch) ? -1 : b.assigned;
    }
    void batch_ptr(const BatchRec& br, void** p, int64_t* bytes) const {
        *p = bufs_[br.buf].base;
        *bytes = bufs_[br.buf].bytes;
    }

    // group-level queries used by the shard runner
    Group& group_of(int64_t t);
    // Per-sample completion stamps: %globaltimer (| 1) written to host-mapped memory
    // by the group's last kernel when the sample's outputs are complete, else 0.
    static constexpr int64_t kStampSlots = int64_t(1) << 20;   // ring, indexed by ticket
    uint64_t sample_stamp(int64_t t) const {
        return *static_cast<volatile const uint64_t*>(stamp_host_ + (t & (kStampSlots - 1)));
    }
    // the sample's outputs are complete (its stamp landed, or its whole group finished)
    bool sample_ready(int64_t t) {
        Group& g = groups[tickets[t].group];
        if (g.complete || (g.stamped && sample_stamp(t) != 0)) return true;
        if (!g.part_idx.empty() && g.part_ready() &&
            std::find(g.part_idx.begin(), g.part_idx.end(), tickets[t].idx) != g.part_idx.end())
            return true;
        return poll_group(g);
    }
    cudaEvent_t make_ready_event() { return get_event(); }
    void forget_pinned() { pinned_pages_.clear(); }   // (a pinned buffer was freed)
    // Completion notices for per-sample waiters (lfg_wait_for; enabled with coalesce_us > 0):
    // each launched group enqueues a host function after its last stage that records the
    // group's launch serial in a ring and wakes the waiters, so process_sample workers
    // block until their group finishes instead of polling events.
    static constexpr int kDoneSlots = 1 << 16;
    std::unique_ptr<std::atomic<int64_t>[]> done_ring_;
    // waiters of a group sleep on one of kDoneWaits condition variables (by launch serial),
    // so a group's completion wakes its own waiters, not every blocked worker
    static constexpr int kDoneWaits = 64;
    std::mutex done_mu_[kDoneWaits];
    std::condition_variable done_cv_[kDoneWaits];
    int64_t launch_serial_ = 0;
    bool group_done_notified(int64_t serial) const {
        return serial > 0 && done_ring_[serial & (kDoneSlots - 1)].load(std::memory_order_acquire) >= serial;
    }   // a batch's pooled ready event
    bool poll_group(Group& g);          // updates stages_done/complete; true if complete
    void finalize_group_timing(Group& g);
    int64_t open_group_count() const;
    // Drop every ticket and group if none is still referenced (all tickets released,
    // all groups complete, nothing open or deferred), keeping the tables' storage:
    // the next run reuses memory that is already faulted in.  Returns whether it did.
    bool recycle_tables();

    // Launch-group streams: one per hardware work queue the process configured
    // (CUDA_DEVICE_MAX_CONNECTIONS, read at context creation; see Context()).
    static constexpr int kMaxStreamPool = 28;
    int stream_pool = kMaxStreamPool;
    int free_stream_count() const { return static_cast<int>(free_streams_.size()); }
    lfg_counters counters{};
    double prof_group_ns = 0, prof_launch_ns = 0;   // host time in launch_group / kernel launch calls
    double prof_views_ns = 0, prof_desc_ns = 0;     // launch_group: payload views / descriptor fill (LFG_SHARD_PROF)
    bool prof_on = false;
    double prof_query_ns = 0, prof_final_ns = 0;    // event queries / completed-group timing reads
    int64_t prof_queries = 0;
    bool serial = false;
    bool defer_launch = false;
    // Per-sample completion stamps.  A group whose last kernel is a synthetic cost
    // (K14 spin: LightStep / HeavyStep, workloads.cpp:109-110) always stamps its
    // samples (one CTA per sample, nothing to fence).  The transform kernels stamp
    // only when this is set (lfg_run_config.sample_stamps): there every kernel part
    // pays a release fence (its output stores acknowledged before the count),
    // ~30% of K1 / K3 time, so by default a transform-last group completes as a
    // whole -- or per sub-launch, as the foreground-crop split does (see launch_group).
    bool stamp_transforms = false;
    // Launch groups carry timed stage events (device-timed stage / sample costs:
    // the profiler, device-timed timeout classification, lfg_exec_costs, the
    // roofline).  A query + elapsed-time read of timed events costs the submitting
    // thread ~8 us per group, so shard runs without a profiler or timeout use
    // untimed events (run_shard sets this).
    bool time_groups = true;
    void time_kernels(Chain* c, const lfg_sample_desc* s, int n, double* mean_ms, int64_t* launches,
                      int64_t* bytes, int64_t* flops);
    std::mutex mu;   // one lock per context (C ABI calls serialise on it)
    // a streaming shard run (lfg_shard_start) is active: its loop takes `mu` per pass;
    // calls that submit or run another shard are refused until it ends
    bool streaming = false;
    std::unique_ptr<WorkerThreads> workers;   // parameter draws of shard runs

    cudaStream_t seal_stream = nullptr;
    cudaStream_t aux_stream = nullptr;

    std::vector<Ticket> tickets;
    std::deque<std::pair<lfg_sample_desc, PreDraw>> owned_;   // samples submitted through the ABI
    std::vector<PreDraw> pre_store;   // the shard runner's per-sample draws (reused between runs)
    std::vector<Group> groups;
    std::vector<BatchRec> batches;

private:
    std::vector<std::unique_ptr<Chain>> chains_;
    SpeechTables* speech_ = nullptr;   // DFT basis + mel tables, created with the first speech chain
    uint64_t* stamp_host_ = nullptr;   // [kStampSlots] host-mapped pinned completion stamps
    uint64_t* stamp_dev_ = nullptr;    // the same words' device address
    uint32_t* stamp_cnt_ = nullptr;    // [kStampSlots] device part counters (self-resetting)
    bool img3d_tma_ = true;            // LFG_IMG3D_TMA=0 forces the row kernel (A/B checks)
    static constexpr int kCsumSlots = 4096;   // RandomContrast crop sums (a ring; stream-ordered)
    double* csum_ = nullptr;
    int csum_next_ = 0;
    static constexpr int kFgSlots = 256;   // K2 scratch rings (launch groups; stream-ordered)
    int32_t* fg_box_ = nullptr;            // [kFgSlots][kMax3D][8 classes][6]
    int4* fg_offs_ = nullptr;              // [kFgSlots][kMax3D]
    int fg_next_ = 0;
    std::vector<cudaStream_t> streams_;
    std::vector<cudaStream_t> side_streams_;   // forked work of a group (the K2 label scans)
    int64_t side_next_ = 0;
    std::vector<int> free_streams_;
    std::vector<cudaEvent_t> free_events_, free_tevents_;   // untimed / timed
    std::vector<SlotBuf> bufs_;
    float** out_tab_ = nullptr;         // device copy of the slot-buffer bases (K3 descriptors index it)
    void sync_out_tab();
    size_t alloc_cursor_[2] = {0, 0};   // [for_batch] last buffer handed out
    std::vector<RawBuf> raws_;
    cudaMemPool_t raw_pool_ = nullptr;   // the context's stream-ordered pool for the staging buffers
    std::unordered_set<uintptr_t> pinned_pages_;   // 4 KB pages of validated pinned payloads
    std::vector<int64_t> free_raws_;
    SmallMap<int> open_buf_;                 // chain -> open slot buffer
    std::vector<int64_t> deferred_;          // full groups awaiting launch (timing mode)
    SmallMap<int64_t> open_group_[2];        // [src_kind] chain -> group

    // events: untimed (cudaEventDisableTiming: ordering and completion only; cheap to
    // record and query) unless `timed` (stage timing of a launch group)
    cudaEvent_t get_event(bool timed = false);
    void put_event(cudaEvent_t e, bool timed = false);
    int get_stream();
    int alloc_buf(const Chain* c, bool for_batch);
    void reserve_bufs(const Chain* c);
    bool chain_alive(const Chain* c) const;
    bool buf_reusable(SlotBuf& b);
    void assign_slot(Ticket& t, const Chain* c);
    int64_t get_raw(int64_t bytes, cudaStream_t st);
    void launch_group(Group& g);
    char* slot_ptr(const Ticket& t, int plane) const;
    int64_t stage_raw_bytes(const Chain& c, const Ticket& t) const;
};

}  // namespace lfg
