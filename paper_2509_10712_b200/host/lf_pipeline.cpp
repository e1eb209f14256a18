// lf_pipeline.cpp -- the pipeline stages of include/loadflow/api.hpp:
// transform application, the balancer (process_sample / resume_slow), the
// eager batcher, the consumer, the worker pool and the timeout profiler.
//
// Host-side semantics follow the reference exactly (cited per function) so
// the reference's own doctest suites pass against this library; the device
// branch of process_sample / resume_slow lives in lf_gpu.cpp.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <ostream>

#include "loadflow/api.hpp"

namespace loadflow {

namespace detail {
// lf_gpu.cpp
RouteResult process_on_device(Sample s, DurationMs t_out, SampleQueue& fast_q, TempQueue& temp_q,
                              Runtime& rt);
void finish_on_device(Sample& s, std::vector<DurationMs>& costs, Runtime& rt);
void release_device_batch(Batch& b);
}  // namespace detail

// ------------------------------------------------------------ chain (sample.cpp:7-48)
std::vector<std::pair<std::size_t, std::size_t>> TransformChain::sections() const {
    std::vector<std::pair<std::size_t, std::size_t>> runs;
    std::size_t open = 0;
    for (std::size_t i = 0; i <= steps_.size(); ++i) {
        const bool end = i == steps_.size();
        if (!end && !steps_[i].barrier) continue;
        if (i > open) runs.emplace_back(open, i);          // reorderable run before the barrier
        if (!end) runs.emplace_back(i, i + 1);             // the pinned barrier itself
        open = i + 1;
    }
    return runs;
}

double TransformChain::size_factor_product() const {
    return std::accumulate(steps_.begin(), steps_.end(), 1.0,
                           [](double acc, const Transform& t) { return acc * t.size_factor; });
}

bool TransformChain::on_device() const {
    if (steps_.empty()) return false;
    for (const auto& t : steps_)
        if (!t.device.on_device()) return false;
    return true;
}

void apply_transform(Sample& sample, std::size_t index, Runtime& rt, Rng& rng) {
    if (sample.chain == nullptr) throw std::invalid_argument("sample has no chain");
    const TransformChain& chain = *sample.chain;
    if (index >= chain.size() || index != sample.next_index) {
        throw std::invalid_argument("apply_transform: index " + std::to_string(index) +
                                    " is out of range or not next_index " +
                                    std::to_string(sample.next_index));
    }
    const Transform& step = chain.at(index);
    if (step.synthetic()) rt.sleep(step.cost(sample, rng));
    else if (step.apply) sample.payload = step.apply(std::move(sample.payload));
    sample.size_bytes *= step.size_factor;
    sample.next_index = index + 1;
}

void apply_all_transforms(Sample& sample, Runtime& rt, Rng& rng) {
    while (sample.chain != nullptr && sample.next_index < sample.chain->size())
        apply_transform(sample, sample.next_index, rt, rng);
}

// ------------------------------------------------------------ balancer (balancer.cpp:9-113)
namespace {

RouteResult to_temp(Sample&& s, std::size_t i, DurationMs charged, RouteResult res,
                    TempQueue& temp_q) {
    s.classification = SampleClass::slow;
    res.route = Route::temp;
    res.foreground_ms = charged;
    res.timeout_index = i;
    temp_q.put(TempItem{std::move(s), i, res.exec_costs});
    return res;
}

RouteResult to_fast(Sample&& s, DurationMs charged, RouteResult res, SampleQueue& fast_q,
                    Runtime& rt) {
    s.classification = SampleClass::fast;
    s.t_ready = rt.now();
    res.route = Route::fast;
    res.foreground_ms = charged;
    fast_q.put(std::move(s));
    return res;
}

// Synthetic chains: the budget is checked before each step; a step that would
// overrun it is interrupted at exactly t_out (the inclusive boundary means a
// chain costing exactly t_out is fast).
RouteResult run_synthetic(Sample s, DurationMs t_out, SampleQueue& fast_q, TempQueue& temp_q,
                          Runtime& rt, Rng& rng) {
    const TransformChain& chain = *s.chain;
    RouteResult res;
    DurationMs spent = 0;
    for (std::size_t i = 0; i < chain.size(); ++i) {
        const Transform& step = chain.at(i);
        const DurationMs c = step.cost(s, rng);
        if (c < 0) throw std::logic_error("negative transform cost");
        if (spent + c > t_out) {
            rt.sleep(t_out - spent);
            return to_temp(std::move(s), i, t_out, std::move(res), temp_q);
        }
        rt.sleep(c);
        spent += c;
        s.size_bytes *= step.size_factor;
        s.next_index = i + 1;
        res.exec_costs.push_back(c);
    }
    return to_fast(std::move(s), spent, std::move(res), fast_q, rt);
}

// Real-function chains: cooperative check after each step; the step that
// overran is rolled back (its input is kept aside) and re-executed later.
RouteResult run_real(Sample s, DurationMs t_out, SampleQueue& fast_q, TempQueue& temp_q,
                     Runtime& rt) {
    const TransformChain& chain = *s.chain;
    RouteResult res;
    const TimeMs t0 = rt.now();
    for (std::size_t i = 0; i < chain.size(); ++i) {
        const Transform& step = chain.at(i);
        Payload before = s.payload;
        const double size_before = s.size_bytes;
        const TimeMs step_t0 = rt.now();
        if (step.apply) s.payload = step.apply(std::move(s.payload));
        const DurationMs step_ms = rt.now() - step_t0;
        if (rt.now() - t0 > t_out) {
            s.payload = std::move(before);
            s.size_bytes = size_before;
            return to_temp(std::move(s), i, rt.now() - t0, std::move(res), temp_q);
        }
        s.size_bytes *= step.size_factor;
        s.next_index = i + 1;
        res.exec_costs.push_back(step_ms);
    }
    return to_fast(std::move(s), rt.now() - t0, std::move(res), fast_q, rt);
}

}  // namespace

RouteResult process_sample(Sample sample, DurationMs t_out, SampleQueue& fast_q,
                           TempQueue& temp_q, Runtime& rt, Rng& rng) {
    if (sample.chain == nullptr || sample.chain->empty())
        throw std::invalid_argument("process_sample: sample has no chain");
    if (sample.next_index != 0 || sample.classification != SampleClass::unclassified)
        throw std::invalid_argument("process_sample: sample already started");
    if (t_out <= 0) throw std::invalid_argument("process_sample: t_out must be > 0");
    if (sample.chain->at(0).synthetic())
        return run_synthetic(std::move(sample), t_out, fast_q, temp_q, rt, rng);
    if (sample.chain->on_device())
        return detail::process_on_device(std::move(sample), t_out, fast_q, temp_q, rt);
    return run_real(std::move(sample), t_out, fast_q, temp_q, rt);
}

void resume_slow(TempQueue& temp_q, SampleQueue& slow_q, Runtime& rt, Rng& rng,
                 const ResumeHook& on_complete) {
    for (;;) {
        std::optional<TempItem> item = temp_q.get();
        if (!item) return;
        Sample s = std::move(item->sample);
        std::vector<DurationMs> costs = std::move(item->fg_costs);
        const TimeMs bg_t0 = rt.now();
        if (s.chain->on_device()) {
            // the device work was never interrupted: wait for its completion event
            detail::finish_on_device(s, costs, rt);
        } else {
            for (std::size_t i = item->resume_index; i < s.chain->size(); ++i) {
                const TimeMs step_t0 = rt.now();
                apply_transform(s, i, rt, rng);
                costs.push_back(rt.now() - step_t0);
            }
        }
        s.t_ready = rt.now();
        const DurationMs bg = rt.now() - bg_t0;
        if (on_complete) on_complete(s, costs, bg);
        slow_q.put(std::move(s));
    }
}

// ------------------------------------------------------------ batcher (batcher.cpp:12-91)
namespace {

struct RoundRobin {
    std::span<SampleQueue* const> qs;
    std::size_t next = 0;

    std::optional<Sample> take() {
        const std::size_t n = qs.size();
        for (std::size_t k = 0; k < n; ++k) {
            const std::size_t i = (next + k) % n;
            if (auto s = qs[i]->try_get()) {
                next = (i + 1) % n;
                return s;
            }
        }
        return std::nullopt;
    }
    bool any_ready() const {
        return std::any_of(qs.begin(), qs.end(), [](SampleQueue* q) { return !q->empty(); });
    }
    bool exhausted() const {
        return std::all_of(qs.begin(), qs.end(), [](SampleQueue* q) { return q->drained(); });
    }
};

}  // namespace

void build_batches(std::span<SampleQueue* const> fast_qs, std::span<SampleQueue* const> slow_qs,
                   BatchQueue& batch_q, const BatcherConfig& cfg, Runtime& rt,
                   BatcherTrace* trace) {
    if (cfg.batch_size < 1) throw std::invalid_argument("batch_size must be >= 1");
    RoundRobin fast{fast_qs}, slow{slow_qs};
    Batch open;
    open.samples.reserve(cfg.batch_size);

    auto publish = [&] {
        open.sealed_at = rt.now();
        gpu::seal_device_batch(open);   // no-op for host samples
        batch_q.put(std::move(open));
        if (trace) trace->batch_queue_occupancy.emplace_back(rt.now(), batch_q.size());
        open = Batch{};
        open.samples.reserve(cfg.batch_size);
    };

    for (;;) {
        const bool fast_ready = trace ? fast.any_ready() : false;
        const bool slow_ready = trace ? slow.any_ready() : false;
        QueueRole from = QueueRole::fast;
        std::optional<Sample> s = fast.take();
        if (!s) {
            s = slow.take();
            from = QueueRole::slow;
        }
        if (!s) {
            if (fast.exhausted() && slow.exhausted()) {
                if (!open.samples.empty()) publish();          // end-of-epoch partial batch
                batch_q.close();
                return;
            }
            rt.sleep(cfg.sleep_ms);
            continue;
        }
        if (trace) trace->slots.push_back(SlotDecision{rt.now(), from, s->id, fast_ready, slow_ready});
        open.samples.push_back(std::move(*s));
        if (open.samples.size() == cfg.batch_size) publish();
    }
}

// ------------------------------------------------------------ consumer (trainer.cpp:7-66)
std::optional<Batch> next_batch(BatchQueue& q, const ConsumerConfig& cfg, Runtime& rt,
                                ConsumerStats& stats) {
    for (;;) {
        if (auto b = q.try_get()) return b;
        if (q.drained()) return std::nullopt;
        if (cfg.horizon_ms && rt.now() - stats.start >= *cfg.horizon_ms) return std::nullopt;
        rt.sleep(cfg.poll_sleep);
        stats.idle_accounted += cfg.poll_sleep;
    }
}

ConsumerStats run_consumer(const ConsumerConfig& cfg, BatchQueue& q, Runtime& rt) {
    ConsumerStats st;
    st.start = st.end = rt.now();
    TimeMs link_free = st.start;   // the transfer engine, shared by consecutive batches
    while (!cfg.max_batches || st.batches < *cfg.max_batches) {
        std::optional<Batch> b = next_batch(q, cfg, rt, st);
        if (!b) break;
        DurationMs stall = 0;
        if (cfg.prefetch) {
            const TimeMs resident = std::max(b->sealed_at, link_free) + cfg.transfer_per_batch;
            link_free = resident;
            stall = std::max<DurationMs>(0, resident - rt.now());
        } else {
            stall = cfg.transfer_per_batch;
        }
        if (stall > 0 || !cfg.prefetch) {
            rt.sleep(stall);
            st.idle_accounted += stall;
        }
        rt.sleep(cfg.compute_per_batch);
        st.busy += cfg.compute_per_batch;
        const double bytes = b->bytes_out();
        ++st.batches;
        st.samples += static_cast<std::int64_t>(b->samples.size());
        st.bytes += bytes;
        for (const auto& s : b->samples) st.consumed_ids.push_back(s.id);
        st.events.push_back(
            BatchEvent{rt.now(), b->sealed_at, static_cast<std::int64_t>(b->samples.size()), bytes});
        detail::release_device_batch(*b);
        st.end = rt.now();
    }
    st.end = rt.now();
    return st;
}

// ------------------------------------------------------------ worker pool (worker_pool.cpp:9-135)
WorkerPool::WorkerPool(Runtime& rt, PoolConfig cfg, BoundedQueue<Sample>& input, Handler handler,
                       SlotExitHook on_slot_exit)
    : rt_(rt), cfg_(cfg), input_(input), handler_(std::move(handler)),
      on_exit_(std::move(on_slot_exit)), mu_(rt.make_mutex()), wake_(rt.make_cond()) {
    if (cfg_.max_workers < 1) throw std::invalid_argument("max_workers must be >= 1");
    if (cfg_.initial_workers < 1 || cfg_.initial_workers > cfg_.max_workers)
        throw std::invalid_argument("initial_workers out of [1, max_workers]");
    slots_.resize(static_cast<std::size_t>(cfg_.max_workers));
}

void WorkerPool::launch(int slot) {   // caller holds mu_
    slots_[slot].spawned = true;
    ++n_spawned_;
    rt_.spawn("worker." + std::to_string(slot), [this, slot] { slot_main(slot); });
}

void WorkerPool::start() {
    LockGuard g(*mu_);
    if (started_) throw std::logic_error("pool already started");
    started_ = true;
    target_ = cfg_.initial_workers;
    for (int i = 0; i < target_; ++i) {
        slots_[i].active = true;
        launch(i);
    }
}

void WorkerPool::resize(int target) {
    target = std::clamp(target, 1, cfg_.max_workers);
    LockGuard g(*mu_);
    if (!started_ || input_done_) return;
    target_ = target;
    for (int i = 0; i < cfg_.max_workers; ++i) {
        Slot& s = slots_[i];
        if (i < target && !s.active) {
            s.active = true;
            if (!s.spawned) launch(i);
        } else if (i >= target && s.active) {
            s.active = false;   // parks after its current sample
        }
    }
    wake_->notify_all();
}

void WorkerPool::slot_main(int slot) {
    for (;;) {
        {
            LockGuard g(*mu_);
            while (!slots_[slot].active && !input_done_) wake_->wait(*mu_);
            if (input_done_) break;
        }
        std::optional<Sample> s = input_.get();
        if (!s) {
            LockGuard g(*mu_);
            input_done_ = true;
            wake_->notify_all();
            break;
        }
        handler_(slot, std::move(*s));
    }
    on_exit_(slot);
    bool last;
    {
        LockGuard g(*mu_);
        last = ++n_exited_ == n_spawned_;
    }
    if (!last) return;
    // slots that never ran still owe their downstream queues a close
    for (int i = 0; i < cfg_.max_workers; ++i) {
        bool never;
        {
            LockGuard g(*mu_);
            never = !slots_[i].spawned;
        }
        if (never) on_exit_(i);
    }
}

int WorkerPool::target_active() const { LockGuard g(*mu_); return target_; }
int WorkerPool::spawned() const { LockGuard g(*mu_); return n_spawned_; }
bool WorkerPool::stopped() const { LockGuard g(*mu_); return input_done_; }

void WorkerPool::note_busy_start(int slot) {
    LockGuard g(*mu_);
    slots_[slot].busy_since = rt_.now();
}

void WorkerPool::note_busy_end(int slot, DurationMs fg_ms) {
    LockGuard g(*mu_);
    slots_[slot].busy += fg_ms;
    slots_[slot].busy_since = -1;
}

DurationMs WorkerPool::effective_busy() const {
    LockGuard g(*mu_);
    const TimeMs t = rt_.now();
    DurationMs total = 0;
    for (const Slot& s : slots_) total += s.busy + (s.busy_since >= 0 ? t - s.busy_since : 0);
    return total;
}

// ------------------------------------------------------------ profiler (profiler.cpp:13-121)
DurationMs percentile(std::vector<DurationMs> d, double p) {
    if (d.empty()) throw InsufficientProfileData();
    if (!(p > 0.0 && p <= 100.0)) throw std::invalid_argument("percentile p out of (0,100]");
    std::sort(d.begin(), d.end());
    std::size_t rank = static_cast<std::size_t>(std::ceil(p / 100.0 * static_cast<double>(d.size())));
    return d[std::max<std::size_t>(rank, 1) - 1];   // nearest rank, 1-based
}

SampleStats SampleStats::from_costs(std::uint64_t id, double size_bytes,
                                    std::vector<DurationMs> costs, bool slow) {
    SampleStats st;
    st.sample_id = id;
    st.size_bytes = size_bytes;
    st.total = std::accumulate(costs.begin(), costs.end(), DurationMs{0});
    st.transform_count = static_cast<int>(costs.size());
    st.per_transform = std::move(costs);
    st.slow = slow;
    return st;
}

Profiler::Profiler(Runtime& rt, ProfilerConfig cfg) : cfg_(cfg), mu_(rt.make_mutex()) {
    if (cfg_.window == 0) throw std::invalid_argument("profiler window must be > 0");
}

void Profiler::record(SampleStats stats) {
    LockGuard g(*mu_);
    recent_.push_back(std::move(stats));
    while (recent_.size() > cfg_.window) recent_.pop_front();
    ++n_recorded_;
}

DurationMs Profiler::update_timeout(TimeoutPolicy& policy) {
    LockGuard g(*mu_);
    if (recent_.empty()) throw InsufficientProfileData();
    std::vector<DurationMs> totals;
    totals.reserve(recent_.size());
    std::size_t n_slow = 0;
    for (const auto& st : recent_) {
        totals.push_back(st.total);
        n_slow += st.slow ? 1 : 0;
    }
    const double rate = static_cast<double>(n_slow) / static_cast<double>(recent_.size());
    if (pct_ == 75 && rate > cfg_.escalate_threshold) {
        pct_ = 90;
    } else if (pct_ == 90 && recent_.size() == cfg_.window && rate < cfg_.deescalate_threshold) {
        pct_ = 75;   // only on a full window: hysteresis
    }
    const DurationMs t = percentile(std::move(totals), pct_);
    policy.set(t, pct_ == 75 ? TimeoutPolicy::Source::p75 : TimeoutPolicy::Source::p90);
    return t;
}

int Profiler::current_percentile() const { LockGuard g(*mu_); return pct_; }

double Profiler::slow_rate() const {
    LockGuard g(*mu_);
    if (recent_.empty()) return 0.0;
    const auto n = std::count_if(recent_.begin(), recent_.end(), [](const SampleStats& s) { return s.slow; });
    return static_cast<double>(n) / static_cast<double>(recent_.size());
}

std::size_t Profiler::recorded_total() const { LockGuard g(*mu_); return n_recorded_; }
std::size_t Profiler::window_size() const { LockGuard g(*mu_); return recent_.size(); }

void Profiler::dump_csv(std::ostream& out) const {
    LockGuard g(*mu_);
    out << "sample_id,size_bytes,total_ms,n_transforms\n";
    for (const auto& st : recent_)
        out << st.sample_id << "," << static_cast<std::int64_t>(st.size_bytes) << "," << st.total
            << "," << st.transform_count << "\n";
}

void profiler_loop(Profiler& prof, TimeoutPolicy& policy, Runtime& rt,
                   const std::function<bool()>& stop) {
    const DurationMs quantum = std::max<DurationMs>(1, prof.config().update_interval);
    const DurationMs warmup = prof.config().warmup;
    const TimeMs t0 = rt.now();
    for (DurationMs waited = 0; waited < warmup; waited = rt.now() - t0) {
        if (stop()) return;
        rt.sleep(std::min(quantum, warmup - waited));
    }
    while (!stop()) {
        if (prof.window_size() > 0) prof.update_timeout(policy);
        rt.sleep(quantum);
    }
}

}  // namespace loadflow
