// loadflow/api.hpp -- reference-shaped C++ API of the B200 MinatoLoader hot path.
//
// Every declaration here keeps the signature of the reference C++ API in
// /root/reference/proj/include/loadflow (cited per block), so a user of the
// reference can recompile against these headers unchanged; the per-file
// headers (balancer.hpp, batcher.hpp, ...) forward here.  Extensions are
// additive only: trailing struct fields with defaults and new functions.
//
// The GPU path enters through two extension fields:
//   Transform::device  -- the lfg_op this transform maps to (include/lfgpu.h)
//   Sample::device     -- where the raw payload lives and which GPU shard runs it
// When a chain's transforms carry device ops, process_sample submits the
// sample to the CUDA library (liblfgpu.so, C ABI) instead of running the host
// body, polls its per-stage CUDA events against t_out on the Runtime clock,
// and resume_slow waits on the completion event (see lf_gpu.cpp).
#pragma once

#include <atomic>
#include <cassert>
#include <cstdint>
#include <deque>
#include <functional>
#include <iosfwd>
#include <limits>
#include <memory>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../lfgpu.h"

namespace loadflow {

// ---------------------------------------------------------------- time (time.hpp:11-16)
// Integer run time.  Reference runtimes tick in milliseconds; the GPU
// realtime runtime (make_realtime_runtime_ticks) ticks in microseconds so
// per-sample device budgets are representable.
using TimeMs = std::int64_t;
using DurationMs = std::int64_t;
inline constexpr DurationMs kNoTimeout = std::numeric_limits<std::int64_t>::max() / 4;

// ---------------------------------------------------------------- runtime (runtime.hpp:15-72)
class Mutex {
public:
    virtual ~Mutex() = default;
    virtual void lock() = 0;
    virtual void unlock() = 0;
};

class Cond {
public:
    virtual ~Cond() = default;
    virtual void wait(Mutex& m) = 0;   // caller holds m; may wake spuriously
    virtual void notify_one() = 0;
    virtual void notify_all() = 0;
};

class LockGuard {
public:
    explicit LockGuard(Mutex& m) : m_(m) { m_.lock(); }
    ~LockGuard() { m_.unlock(); }
    LockGuard(const LockGuard&) = delete;
    LockGuard& operator=(const LockGuard&) = delete;

private:
    Mutex& m_;
};

// The only source of time and concurrency: loops run as actors and block only
// through sleep() or Cond::wait().
class Runtime {
public:
    virtual ~Runtime() = default;
    virtual TimeMs now() = 0;
    virtual void sleep(DurationMs d) = 0;
    virtual void spawn(std::string name, std::function<void()> body) = 0;
    virtual void run() = 0;
    virtual std::unique_ptr<Mutex> make_mutex() = 0;
    virtual std::unique_ptr<Cond> make_cond() = 0;
    virtual bool is_virtual() const = 0;
    // Extension: length of one clock tick in nanoseconds (1 ms for the
    // reference runtimes), used to express device-measured costs in ticks.
    virtual std::int64_t tick_ns() const { return 1'000'000; }
};

std::unique_ptr<Runtime> make_realtime_runtime();
std::unique_ptr<Runtime> make_virtual_runtime();
// Extension: realtime runtime whose tick is `tick_ns` nanoseconds (1000 = the
// microsecond clock the GPU balancer uses); sleep(d) sleeps d ticks.
std::unique_ptr<Runtime> make_realtime_runtime_ticks(std::int64_t tick_ns);

// ---------------------------------------------------------------- channels (queue.hpp:15-126)
enum class QueueRole : std::uint8_t { fast, slow, temp, batch, input };

inline const char* to_string(QueueRole r) {
    static const char* const names[] = {"fast", "slow", "temp", "batch", "input"};
    const auto i = static_cast<std::size_t>(r);
    return i < 5 ? names[i] : "?";
}

class QueueClosedError : public std::runtime_error {
public:
    explicit QueueClosedError(const std::string& name) : std::runtime_error("queue closed: " + name) {}
};

// Bounded blocking FIFO; close() rejects further puts, get() drains then
// reports end of stream.  All blocking goes through Runtime primitives.
template <typename T>
class BoundedQueue {
public:
    BoundedQueue(Runtime& rt, std::size_t capacity = 100, QueueRole role = QueueRole::input,
                 std::string name = "")
        : cap_(capacity), role_(role), name_(name.empty() ? std::string(to_string(role)) : name),
          lock_(rt.make_mutex()), has_items_(rt.make_cond()), has_room_(rt.make_cond()) {
        if (cap_ == 0) throw std::invalid_argument("queue capacity must be > 0");
    }

    void put(T item) {
        LockGuard hold(*lock_);
        for (;;) {
            if (closed_) throw QueueClosedError(name_);
            if (buf_.size() < cap_) break;
            has_room_->wait(*lock_);
        }
        buf_.push_back(std::move(item));
        has_items_->notify_one();
    }

    std::optional<T> get() {
        LockGuard hold(*lock_);
        while (buf_.empty()) {
            if (closed_) return std::nullopt;
            has_items_->wait(*lock_);
        }
        return pop_locked();
    }

    std::optional<T> try_get() {
        LockGuard hold(*lock_);
        if (buf_.empty()) return std::nullopt;
        return pop_locked();
    }

    void close() {
        LockGuard hold(*lock_);
        closed_ = true;
        has_items_->notify_all();
        has_room_->notify_all();
    }

    bool closed() const { LockGuard hold(*lock_); return closed_; }
    bool drained() const { LockGuard hold(*lock_); return closed_ && buf_.empty(); }
    bool empty() const { LockGuard hold(*lock_); return buf_.empty(); }
    std::size_t size() const { LockGuard hold(*lock_); return buf_.size(); }
    std::size_t capacity() const { return cap_; }
    QueueRole role() const { return role_; }
    const std::string& name() const { return name_; }

private:
    std::optional<T> pop_locked() {
        std::optional<T> out(std::move(buf_.front()));
        buf_.pop_front();
        has_room_->notify_one();
        return out;
    }

    const std::size_t cap_;
    const QueueRole role_;
    const std::string name_;
    mutable std::unique_ptr<Mutex> lock_;
    std::unique_ptr<Cond> has_items_;
    std::unique_ptr<Cond> has_room_;
    std::deque<T> buf_;
    bool closed_ = false;
};

// ---------------------------------------------------------------- samples (sample.hpp:16-98)
class TransformChain;
struct Sample;

enum class SampleClass : std::uint8_t { unclassified, fast, slow };
using Payload = std::vector<double>;
using Rng = std::mt19937_64;

// Extension: the device op a transform maps to (kind 0 = host-only transform).
struct DeviceOp {
    lfg_op op{};
    bool on_device() const { return op.kind != 0; }
};

struct Transform {
    std::string name;
    double size_factor = 1.0;
    bool barrier = false;
    std::function<DurationMs(const Sample&, Rng&)> cost;   // synthetic mode
    std::function<Payload(Payload)> apply;                 // real-function mode
    DeviceOp device{};                                     // GPU mode (extension)

    bool synthetic() const { return static_cast<bool>(cost); }
};

// Extension: a sample's raw payload for the GPU path, plus the ticket of its
// in-flight device work (-1 before submission).
struct DeviceRef {
    lfg_sample_desc desc{};
    std::int64_t ticket = -1;
    int shard = 0;
};

struct Sample {
    std::uint64_t id = 0;
    double bytes_in = 0;
    double size_bytes = 0;
    double bytes_out = 0;
    const TransformChain* chain = nullptr;
    std::size_t next_index = 0;
    SampleClass classification = SampleClass::unclassified;
    TimeMs t_enqueue = -1;
    TimeMs t_ready = -1;
    std::vector<DurationMs> step_costs;
    Payload payload;
    DeviceRef device{};                                    // GPU mode (extension)
};

class TransformChain {
public:
    TransformChain() = default;
    explicit TransformChain(std::vector<Transform> transforms) : steps_(std::move(transforms)) {}

    const std::vector<Transform>& transforms() const { return steps_; }
    std::vector<Transform>& transforms() { return steps_; }
    std::size_t size() const { return steps_.size(); }
    bool empty() const { return steps_.empty(); }
    const Transform& at(std::size_t i) const { return steps_.at(i); }
    std::vector<std::pair<std::size_t, std::size_t>> sections() const;
    double size_factor_product() const;
    bool on_device() const;   // extension: every transform carries a device op

private:
    std::vector<Transform> steps_;
};

struct Batch {
    std::vector<Sample> samples;
    TimeMs sealed_at = -1;
    std::int64_t device_batch = -1;   // extension: lfg_batch handle when sealed on the GPU

    double bytes_out() const {
        double total = 0;
        for (const auto& s : samples) total += s.bytes_out;
        return total;
    }
};

void apply_transform(Sample& sample, std::size_t index, Runtime& rt, Rng& rng);
void apply_all_transforms(Sample& sample, Runtime& rt, Rng& rng);

// ---------------------------------------------------------------- balancer (balancer.hpp:15-72)
struct TimeoutPolicy {
    enum class Source : std::uint8_t { configured, p75, p90 };
    std::atomic<DurationMs> t_out{kNoTimeout};
    std::atomic<Source> source{Source::configured};
    DurationMs timeout() const { return t_out.load(std::memory_order_relaxed); }
    void set(DurationMs v, Source s) {
        t_out.store(v, std::memory_order_relaxed);
        source.store(s, std::memory_order_relaxed);
    }
};

struct TempItem {
    Sample sample;
    std::size_t resume_index = 0;
    std::vector<DurationMs> fg_costs;
};

using SampleQueue = BoundedQueue<Sample>;
using TempQueue = BoundedQueue<TempItem>;
using BatchQueue = BoundedQueue<Batch>;

enum class Route : std::uint8_t { fast, temp };

struct RouteResult {
    Route route = Route::fast;
    DurationMs foreground_ms = 0;
    std::size_t timeout_index = 0;
    std::vector<DurationMs> exec_costs;
};

RouteResult process_sample(Sample sample, DurationMs t_out, SampleQueue& fast_q,
                           TempQueue& temp_q, Runtime& rt, Rng& rng);

using ResumeHook =
    std::function<void(const Sample&, const std::vector<DurationMs>&, DurationMs)>;
void resume_slow(TempQueue& temp_q, SampleQueue& slow_q, Runtime& rt, Rng& rng,
                 const ResumeHook& on_complete = nullptr);

// ---------------------------------------------------------------- batcher (batcher.hpp:12-39)
struct BatcherConfig {
    std::size_t batch_size = 1;
    DurationMs sleep_ms = 10;
};

struct SlotDecision {
    TimeMs t = 0;
    QueueRole source = QueueRole::fast;
    std::uint64_t sample_id = 0;
    bool fast_available = false;
    bool slow_available = false;
};

struct BatcherTrace {
    std::vector<SlotDecision> slots;
    std::vector<std::pair<TimeMs, std::size_t>> batch_queue_occupancy;
};

void build_batches(std::span<SampleQueue* const> fast_qs, std::span<SampleQueue* const> slow_qs,
                   BatchQueue& batch_q, const BatcherConfig& cfg, Runtime& rt,
                   BatcherTrace* trace = nullptr);

// ---------------------------------------------------------------- consumer (trainer.hpp:14-59)
struct ConsumerConfig {
    DurationMs compute_per_batch = 200;
    DurationMs transfer_per_batch = 0;
    DurationMs poll_sleep = 10;
    bool prefetch = true;
    std::optional<std::int64_t> max_batches;
    std::optional<DurationMs> horizon_ms;
};

struct BatchEvent {
    TimeMs compute_end = 0;
    TimeMs sealed_at = 0;
    std::int64_t n_samples = 0;
    double bytes = 0;
};

struct ConsumerStats {
    TimeMs start = 0;
    TimeMs end = 0;
    DurationMs busy = 0;
    DurationMs idle_accounted = 0;
    std::int64_t batches = 0;
    std::int64_t samples = 0;
    double bytes = 0;
    std::vector<BatchEvent> events;
    std::vector<std::uint64_t> consumed_ids;

    TimeMs span() const { return end - start; }
    DurationMs idle() const { return span() - busy; }
    double busy_fraction() const {
        return span() > 0 ? static_cast<double>(busy) / static_cast<double>(span()) : 0.0;
    }
    double idle_fraction() const { return span() > 0 ? 1.0 - busy_fraction() : 0.0; }
};

std::optional<Batch> next_batch(BatchQueue& q, const ConsumerConfig& cfg, Runtime& rt,
                                ConsumerStats& stats);
ConsumerStats run_consumer(const ConsumerConfig& cfg, BatchQueue& q, Runtime& rt);

// ---------------------------------------------------------------- worker pool (worker_pool.hpp:12-68)
struct PoolConfig {
    int initial_workers = 12;
    int max_workers = 12;
};

class WorkerPool {
public:
    using Handler = std::function<void(int slot, Sample&&)>;
    using SlotExitHook = std::function<void(int slot)>;

    WorkerPool(Runtime& rt, PoolConfig cfg, BoundedQueue<Sample>& input, Handler handler,
               SlotExitHook on_slot_exit);
    void start();
    void resize(int target);
    int target_active() const;
    int spawned() const;
    bool stopped() const;
    void note_busy_start(int slot);
    void note_busy_end(int slot, DurationMs fg_ms);
    DurationMs effective_busy() const;

private:
    struct Slot {
        bool active = false;
        bool spawned = false;
        DurationMs busy = 0;
        TimeMs busy_since = -1;
    };
    void launch(int slot);
    void slot_main(int slot);

    Runtime& rt_;
    PoolConfig cfg_;
    BoundedQueue<Sample>& input_;
    Handler handler_;
    SlotExitHook on_exit_;
    mutable std::unique_ptr<Mutex> mu_;
    std::unique_ptr<Cond> wake_;
    std::vector<Slot> slots_;
    int target_ = 0;
    int n_spawned_ = 0;
    int n_exited_ = 0;
    bool input_done_ = false;
    bool started_ = false;
};

// ---------------------------------------------------------------- adaptive scheduler (scheduler.hpp:13-52)
// SURVEY 8(f) row 1.  Host pool: the reference's control loop over WorkerPool.
// GPU shard: the same rule (sched_rule.h) resizes the number of in-flight
// launch groups (lfg_run_config.scheduler), with c_usage = the stream pool's
// busy fraction from CUDA events and q = delivered batches the trainer has not
// consumed yet.
struct SchedulerConfig {
    double alpha = 2.0;   // queue-sensitivity scale
    double beta = 2.0;    // CPU-sensitivity scale
    double theta_c = 0.7; // utilization threshold
    double q_max = 100;   // batch queue capacity
    int delta_clip = 2;
    int initial_workers = 12;
    int max_workers = static_cast<int>(std::thread::hardware_concurrency());
    DurationMs tick = 500;
    double ema_alpha = 0.3; // smoothing for the queue-size moving average
};

struct SchedulerObservation {
    double q_size_avg = 0; // moving average of batch-queue length, in [0, q_max]
    double c_usage = 0;    // worker-pool busy fraction, in [0, 1]
};

struct SchedulerTraceRow {
    TimeMs t = 0;
    int workers = 0;
    double q_avg = 0;
    double c_usage = 0;
    int delta = 0;
};

int compute_delta(const SchedulerObservation& obs, const SchedulerConfig& cfg);
int update_workers(int current, int delta, const SchedulerConfig& cfg);
void scheduler_loop(WorkerPool& pool, std::span<BatchQueue* const> batch_queues,
                    const SchedulerConfig& cfg, Runtime& rt,
                    std::vector<SchedulerTraceRow>* trace = nullptr);

// ---------------------------------------------------------------- baselines (baselines.hpp:12-47)
// the synchronous (PyTorch-DataLoader-like) loader with
// head-of-line blocking, Pecan AutoOrder and the size heuristic.
struct SyncLoaderConfig {
    std::size_t batch_size = 1;
    int n_workers = 1;
    int prefetch_factor = 2; // batches loaded in advance per worker
};

struct SyncBatchRecord {
    std::size_t batch_index = 0;
    TimeMs published_at = 0;          // seal time
    TimeMs max_member_completion = 0; // completion time of the slowest member
};

void start_sync_loader(Runtime& rt, std::vector<Sample> samples, const SyncLoaderConfig& cfg,
                       BatchQueue& batch_q, std::vector<SyncBatchRecord>* records = nullptr);
TransformChain autoorder(const TransformChain& chain);
SampleClass size_heuristic_classify(const Sample& sample, double size_cutoff_bytes);

// ---------------------------------------------------------------- profiler (profiler.hpp:17-85)
class InsufficientProfileData : public std::runtime_error {
public:
    InsufficientProfileData() : std::runtime_error("no profiling data recorded yet") {}
};

DurationMs percentile(std::vector<DurationMs> durations, double p);

struct SampleStats {
    std::uint64_t sample_id = 0;
    double size_bytes = 0;
    std::vector<DurationMs> per_transform;
    DurationMs total = 0;
    int transform_count = 0;
    bool slow = false;

    static SampleStats from_costs(std::uint64_t id, double size_bytes,
                                  std::vector<DurationMs> costs, bool slow);
};

struct ProfilerConfig {
    std::size_t window = 1024;
    DurationMs warmup = 10'000;
    DurationMs update_interval = 1'000;
    double escalate_threshold = 0.35;
    double deescalate_threshold = 0.15;
    DurationMs initial_timeout = kNoTimeout;
};

class Profiler {
public:
    Profiler(Runtime& rt, ProfilerConfig cfg);
    void record(SampleStats stats);
    DurationMs update_timeout(TimeoutPolicy& policy);
    int current_percentile() const;
    double slow_rate() const;
    std::size_t recorded_total() const;
    std::size_t window_size() const;
    void dump_csv(std::ostream& out) const;
    const ProfilerConfig& config() const { return cfg_; }

private:
    ProfilerConfig cfg_;
    mutable std::unique_ptr<Mutex> mu_;
    std::deque<SampleStats> recent_;
    std::size_t n_recorded_ = 0;
    int pct_ = 75;
};

void profiler_loop(Profiler& prof, TimeoutPolicy& policy, Runtime& rt,
                   const std::function<bool()>& stop);

// ---------------------------------------------------------------- workloads (workloads.hpp:13-63)
enum class WorkloadKind : std::uint8_t { img_seg, obj_det, speech_3s, speech_10s };
const char* workload_name(WorkloadKind k);
WorkloadKind workload_from_name(const std::string& name);

struct TargetStats {
    double avg = 0, med = 0, p75 = 0, p90 = 0, min = 0, max = 0;
};

struct WorkloadSpec {
    WorkloadKind kind = WorkloadKind::speech_3s;
    std::int64_t n_samples = 1000;
    std::uint64_t seed = 1;
    TargetStats target;
    DurationMs load_latency = 0;
    void validate() const;
};

WorkloadSpec default_spec(WorkloadKind kind, std::int64_t n_samples, std::uint64_t seed);

struct Stream {
    std::shared_ptr<TransformChain> chain;
    std::vector<Sample> samples;
};

Stream gen_speech(bool ten_seconds, std::int64_t n, std::uint64_t seed);
Stream gen_empirical(const WorkloadSpec& spec);
Stream generate(const WorkloadSpec& spec);
void export_stream_csv(const Stream& stream, std::ostream& out);

// ---------------------------------------------------------------- GPU binding (extension)
namespace gpu {

// Binds the calling process's chains to a GPU shard: the lfg context that
// device-mode process_sample / resume_slow / seal use.  One binding per
// device; `shard` indexes it from Sample::device.shard.
int bind_shard(lfg_ctx* ctx);
lfg_ctx* shard_context(int shard);
void unbind_all();

// Builds the reference chains with device ops attached (names and size
// factors from proj/src/workloads.cpp:103-156).
TransformChain img_seg_chain(int crop = 128);
TransformChain obj_det_chain(int out = 224);

// Compiles a device chain for a shard ahead of the run (allocates its output
// pools); otherwise the first process_sample compiles it on the clock.
void prepare_chain(const TransformChain& chain, int shard);

// Seals a batch of completed device samples into a device-resident batch
// (lfg_seal_batch); fills Batch::device_batch.
void seal_device_batch(Batch& batch);

// The high-throughput path under the reference's consumer: runs `samples` (device
// payloads, one bound shard) through the event-driven shard loop (lfg_shard_start: launch
// groups, timeouts, fast-first eager device seals) and publishes every sealed batch into
// `out` as it is sealed -- Batch::device_batch set, samples carrying ids and accounting
// -- so run_consumer (trainer.cpp:20-66) consumes and releases them unchanged.  Closes
// `out` at the end; blocks while `out` is full (back-pressure).  Run it as an actor
// (rt.spawn).  cfg.trainer_us is ignored: the consumer is the trainer.
lfg_run_report feed_shard(const TransformChain& chain, std::vector<Sample> samples, BatchQueue& out, Runtime& rt,
                          const lfg_run_config& cfg);

}  // namespace gpu

}  // namespace loadflow
