// shard.cpp -- event-driven Algorithm 1 for one GPU shard.
//
// The reference wires one actor per role (run_minato_pipeline,
// proj/src/experiment.cpp:129-276): N worker threads running process_sample
// (balancer.cpp:81-94), N resume threads (balancer.cpp:96-113), a batcher
// polling in 10 ms sleeps (batcher.cpp:60-90), a consumer (trainer.cpp:20-66)
// and a profiler loop (profiler.cpp:108-121).  On the GPU the transform work
// is asynchronous, so all of those collapse into one host loop driven by CUDA
// event queries:
//   workers     -> at most n_workers in-flight launch groups, each on its own stream
//   timeout     -> host clock since launch > t_out while the group's last stage
//                  event is still pending: the group is classified slow and its
//                  stream is parked (no preemption; nothing is re-executed)
//   resume      -> the parked group's completion event -> slow list
//   batcher     -> seal B samples, fast list first (FIFO), then slow list
//   consumer    -> a (high-priority) trainer stream that waits on each batch's
//                  ready event and runs the synthetic step; idle accounting from
//                  CUDA events exactly like ConsumerStats (trainer.hpp:30-47)
//   profiler    -> sliding window of device-timed per-sample totals; nearest-rank
//                  p75 after warm-up, p90 escalation above a 0.35 slow rate,
//                  de-escalation on a full window below 0.15 (profiler.cpp:47-72)
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <deque>
#include <thread>

#include <sys/mman.h>

#include "loadflow/sched_rule.h"
#include <unordered_map>

#include "engine.h"

namespace lfg {

namespace {

constexpr int64_t kNoTimeoutUs = INT64_MAX / 4;  // time.hpp:16 analogue

struct Profile {
    // SampleStats window (profiler.hpp:27-46), totals in microseconds
    std::deque<std::pair<int64_t, bool>> window;
    size_t cap = 1024;
    int pct = 75;
    bool adaptive = true;   // false: a fixed percentile (policy 2, the C5 sweep)
    double escalate = 0.35, deescalate = 0.15;

    int up = 0, down = 0;
    int64_t recorded = 0;
    void record(int64_t total_us, bool slow) {
        window.emplace_back(total_us, slow);
        if (window.size() > cap) window.pop_front();
        ++recorded;
    }
    // Profiler::update_timeout (profiler.cpp:47-72) with nearest-rank percentile (profiler.cpp:13-21)
    int64_t update() {
        std::vector<int64_t> totals;
        size_t slow = 0;
        for (auto& w : window) {
            totals.push_back(w.first);
            slow += w.second;
        }
        const double rate = double(slow) / double(window.size());
        if (adaptive && pct == 75 && rate > escalate) {
            pct = 90;
            ++up;
        } else if (adaptive && pct == 90 && window.size() == cap && rate < deescalate) {
            pct = 75;   // only on a full window: hysteresis against flapping
            ++down;
        }
        std::sort(totals.begin(), totals.end());
        size_t rank = static_cast<size_t>(std::ceil(pct / 100.0 * double(totals.size())));
        if (rank == 0) rank = 1;
        return totals[rank - 1];
    }
};

// Host-loop phase clock (LFG_SHARD_PROF=1 prints the split to stderr): the
// resident-input rate is bounded by this loop, so its cost is kept visible.
#ifdef MADV_POPULATE_WRITE
constexpr int kMadvPopulateWrite = MADV_POPULATE_WRITE;
#else
constexpr int kMadvPopulateWrite = 23;   // Linux >= 5.14; older kernels reject it (harmless)
#endif

struct Phases {
    enum { POLL, PARKED, SUBMIT, FLUSH, SEAL, DELIVER, IDLE, DRAW, N };
    bool on = std::getenv("LFG_SHARD_PROF") != nullptr;
    double ns[N] = {};
    double setup_ns = 0;
    std::chrono::steady_clock::time_point t;
    void start() {
        if (on) t = std::chrono::steady_clock::now();
    }
    void lap(int k) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        ns[k] += std::chrono::duration<double, std::nano>(now - t).count();
        t = now;
    }
    void print(int64_t n, double group_ns, double launch_ns, int64_t groups) const {
        if (!on || n <= 0) return;
        static const char* names[N] = {"poll", "parked", "submit", "flush", "seal", "deliver", "idle",
                                       "draw_wait"};
        std::fprintf(stderr, "[lfg shard] setup=%.2f ms; ns/sample:", setup_ns / 1e6);
        for (int k = 0; k < N; ++k) std::fprintf(stderr, " %s=%.0f", names[k], ns[k] / double(n));
        std::fprintf(stderr, " | per group (%lld): launch_group=%.0f kernel_launch=%.0f ns\n",
                     static_cast<long long>(groups),
                     group_ns / double(std::max<int64_t>(groups, 1)),
                     launch_ns / double(std::max<int64_t>(groups, 1)));
    }
};

}  // namespace

int run_shard(Context& ctx, Chain* chain, const lfg_sample_desc* samples, int64_t n,
              const lfg_run_config& rc, lfg_run_report& rep, uint64_t* consumed_ids,
              int32_t* batch_sizes, int32_t* sample_class, const lfg_source* src,
              const ShardStream* ss) {
    // streaming delivery: the context lock is held except between loop passes
    std::unique_lock<std::mutex> lk;
    if (ss != nullptr) lk = std::unique_lock<std::mutex>(*ss->lock);
    if (src != nullptr && src->next == nullptr) fail(LFG_ERR_INVALID, "source without next()");
    // streaming input: descriptors arrive through src->next, in feed order
    std::vector<lfg_sample_desc> src_descs;
    if (src != nullptr) {
        src_descs.resize(static_cast<size_t>(std::max<int64_t>(n, 0)));
        samples = src_descs.data();
    }
    int64_t fetched = 0;
    auto release_group = [&](const Group& g) {
        if (src != nullptr && src->release != nullptr)
            for (int64_t t : g.tickets) src->release(src->user, ctx.tickets[t].id);
    };
    if (n < 0 || (n > 0 && samples == nullptr)) fail(LFG_ERR_INVALID, "bad sample list");
    const int B = rc.batch_size > 0 ? rc.batch_size : ctx.cfg.batch_size;
    if (B > ctx.cfg.batch_size) fail(LFG_ERR_INVALID, "run batch_size exceeds context batch_size");
    int n_workers = rc.n_workers > 0 ? rc.n_workers : ctx.cfg.n_workers;
    // adaptive scheduler (scheduler.cpp:26-58 on the GPU): workers = in-flight groups,
    // q = delivered batches the trainer has not finished, c = busy fraction of the
    // in-flight slots over the tick (time-integral of inflight / limit)
    const int max_workers = std::max(1, std::min(rc.max_workers > 0 ? rc.max_workers : 2 * n_workers,
                                                 ctx.stream_pool));
    if (rc.scheduler) n_workers = std::min(n_workers, max_workers);
    const int64_t sched_tick = rc.sched_tick_us > 0 ? rc.sched_tick_us : 500;
    const double q_max = std::max(1, ctx.cfg.max_slot_buffers);
    double sched_ema = 0.0, busy_integral = 0.0, workers_integral = 0.0;
    int64_t sched_last = 0, sched_prev_t = 0, sched_t0 = 0, sched_ticks = 0;
    std::deque<cudaEvent_t> consume_q;   // one event per delivered batch, recorded after its trainer step
    const int cap = chain->fam == FAM_IMG3D ? kMax3D : (chain->fam == FAM_RRC2D ? kMax2D : kMaxSp);
    const int group = std::max(1, std::min(ctx.cfg.max_group, cap));

    rep = lfg_run_report{};
    const lfg_counters c0 = ctx.counters;

    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    cudaStream_t trainer;
    cuda_check(cudaStreamCreateWithPriority(&trainer, cudaStreamNonBlocking,
                                            rc.trainer_priority ? hi : lo),
               "trainer stream");
    std::vector<cudaEvent_t> evs;
    auto mk = [&]() {
        cudaEvent_t e;
        cuda_check(cudaEventCreate(&e), "event");
        evs.push_back(e);
        return e;
    };
    // end-to-end probe: 16 bytes of every delivered batch are read back on the trainer
    // stream (pinned before the run's clock starts: cudaMallocHost can take milliseconds)
    char* probe = nullptr;
    if (rc.d2h_probe) cuda_check(cudaMallocHost(&probe, 16 * 1024), "probe buffer");
    int64_t probe_bytes = 0;
    // output capture (verification): feed position -> capture slot
    std::vector<int32_t> cap_slot;
    if (rc.n_capture > 0) {
        if (rc.capture_pos == nullptr || rc.capture_buf == nullptr || rc.capture_stride <= 0)
            fail(LFG_ERR_INVALID, "capture needs capture_pos, capture_buf and capture_stride");
        cap_slot.assign(static_cast<size_t>(std::max<int64_t>(n, 0)), -1);
        for (int k = 0; k < rc.n_capture; ++k) {
            const int64_t p = rc.capture_pos[k];
            if (p < 0 || p >= n) fail(LFG_ERR_INVALID, "capture position out of range");
            cap_slot[static_cast<size_t>(p)] = k;
            if (rc.capture_done) rc.capture_done[k] = 0;
        }
    }
    cudaEvent_t t_start = mk();
    cuda_check(cudaEventRecord(t_start, trainer), "record");
    const auto setup_t0 = std::chrono::steady_clock::now();
    cudaEvent_t t_timed = t_start;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> steps;   // timed-window trainer steps


    Profile prof;
    prof.cap = rc.window > 0 ? static_cast<size_t>(rc.window) : 1024;
    if (rc.policy == 2) {
        if (rc.percentile < 1 || rc.percentile > 100) fail(LFG_ERR_INVALID, "percentile must be in 1..100");
        prof.pct = rc.percentile;
        prof.adaptive = false;
    }
    // policy 3: the synchronous (PyTorch-DataLoader-like) baseline, baselines.cpp:12-151 --
    // batch k = the k-th B samples fed, sealed only when all of them are done, in
    // batch order (head-of-line blocking); no timeouts.
    const bool sync = rc.policy == 3;
    int64_t t_out = (rc.t_out_us > 0 && !sync) ? rc.t_out_us : kNoTimeoutUs;
    std::vector<char> ready_pos(sync ? static_cast<size_t>(n) : 0, 0);
    // per-sample completion stamps from the transform kernels too (sample_stamps = 1)
    struct StampMode {
        Context& c;
        bool saved;
        ~StampMode() { c.stamp_transforms = saved; }
    } stamp_mode{ctx, ctx.stamp_transforms};
    ctx.stamp_transforms = rc.sample_stamps == 1;
    // device-timed stage events only where the run uses device time (Context::time_groups)
    struct TimeMode {
        Context& c;
        bool saved;
        ~TimeMode() { c.time_groups = saved; }
    } time_mode{ctx, ctx.time_groups};
    ctx.time_groups = t_out < kNoTimeoutUs || rc.policy == 1 || rc.policy == 2 || std::getenv("LFG_SHARD_TIMED");
    int64_t sync_next = 0;   // first position of the next batch to seal
    const int64_t run_t0 = host_now_us();
    int64_t last_update = run_t0;
    // LFG_SHARD_TRACE=1: host timeline of the run (group fed / group finished / batch sealed), on stderr
    const bool trace_on = std::getenv("LFG_SHARD_TRACE") != nullptr;
    struct TraceEv {
        int64_t t_us;
        int kind;
        int64_t id;
    };
    std::vector<TraceEv> trace;

    ctx.recycle_tables();   // a previous run's finished tickets: reuse their storage
    const int64_t tbase = static_cast<int64_t>(ctx.tickets.size());
    ctx.tickets.reserve(static_cast<size_t>(tbase + n));
    ctx.groups.reserve(ctx.groups.size() + static_cast<size_t>(n));
    // The run's ticket storage is fresh memory: a helper thread has the kernel
    // populate its pages (MADV_POPULATE_WRITE leaves contents untouched, so it may
    // run while submit constructs tickets), instead of the submitting thread taking
    // one page fault per ~15 tickets.
    std::vector<int64_t> inflight, parked;
    std::deque<int64_t> fast, slow;
    // Zero-copy bookkeeping: fast_cnt[buf] = tickets of slot buffer `buf` in
    // `fast`; full_bufs = buffers whose every sample is in `fast` (candidates
    // for an in-place seal).  Maintained incrementally so the batcher never
    // rescans the fast list.
    std::vector<int> fast_cnt;
    std::deque<int> full_bufs;
    auto fast_add = [&](int64_t t, bool front) {
        const int b = ctx.tickets[t].buf;
        if (b >= static_cast<int>(fast_cnt.size())) fast_cnt.resize(static_cast<size_t>(b) + 1, 0);
        if (front) fast.push_front(t);
        else fast.push_back(t);
        if (++fast_cnt[b] == B && ctx.buf_closed_count(b) == B) full_bufs.push_back(b);
    };
    auto fast_take = [&]() {
        const int64_t t = fast.front();
        fast.pop_front();
        --fast_cnt[ctx.tickets[t].buf];
        return t;
    };
    int64_t fed = 0, consumed = 0, nbatches = 0, timed_samples = 0;
    std::vector<uint64_t> all_ids;
    all_ids.reserve(static_cast<size_t>(n));
    double kernel_ms = 0;

    auto total_us = [&](const Group& g) {
        double ms = 0;
        for (float x : g.stage_ms) ms += x;
        return static_cast<int64_t>(std::llround(ms * 1000.0));
    };
    // Per-sample classification (balancer.cpp:42-77 decides per sample): a sample is
    // handed on as soon as its completion stamp lands -- fast while its group is
    // within budget, slow once the group was parked -- so the fast members of a
    // launch group never wait for a slow one.
    std::vector<uint8_t> cls(static_cast<size_t>(std::max<int64_t>(n, 0)), 0);   // 1 fast, 2 slow
    auto hand_on = [&](Group& g, int i, bool is_slow) {
        g.got[static_cast<size_t>(i)] = is_slow ? 2 : 1;
        ++g.n_got;
        const int64_t t = g.tickets[static_cast<size_t>(i)];
        cls[static_cast<size_t>(t - tbase)] = is_slow ? 2 : 1;
        if (sample_class) sample_class[t - tbase] = is_slow ? 2 : 1;
        if (is_slow) ++rep.slow;
        else ++rep.fast;
        if (sync) ready_pos[static_cast<size_t>(t - tbase)] = 1;
        else if (is_slow) slow.push_back(t);
        else fast_add(t, false);
    };
    // stamps in sample order from scan_from; `all` also looks past the first pending one
    auto scan_stamps = [&](Group& g, bool all, bool is_slow) {
        const int sz = static_cast<int>(g.tickets.size());
        const int before = g.n_got;
        while (g.scan_from < sz &&
               (g.got[static_cast<size_t>(g.scan_from)] || ctx.sample_stamp(g.tickets[g.scan_from]) != 0)) {
            if (!g.got[static_cast<size_t>(g.scan_from)]) hand_on(g, g.scan_from, is_slow);
            ++g.scan_from;
        }
        for (int i = g.scan_from + 1; all && i < sz; ++i)
            if (!g.got[static_cast<size_t>(i)] && ctx.sample_stamp(g.tickets[i]) != 0) hand_on(g, i, is_slow);
        return g.n_got != before;
    };
    // a sub-launch that finished part of the group (the plain samples of a split
    // foreground-crop group) hands that part on
    auto check_part = [&](Group& g, bool is_slow) {
        if (g.part_idx.empty() || g.part_handed || !g.part_ready()) return false;
        for (int i : g.part_idx)
            if (!g.got[static_cast<size_t>(i)]) hand_on(g, i, is_slow);
        g.part_handed = true;
        return true;
    };
    const bool profiled = rc.policy == 1 || rc.policy == 2;
    // ~70% of the recent groups' device time, or host-observed time when the groups are
    // untimed (query throttle); starts from the chain's previous runs
    int64_t est_group_us = chain->est_group_us;
    // the group's last event completed: hand on the rest; per-sample device-timed
    // totals (the group's event-timed span less the time from the sample's stamp to
    // the group's last stamp) go to the profiler window, one record per sample as
    // profiler.cpp:40-45
    auto finish_group = [&](Group& g, bool parked_group) {
        if (trace_on) trace.push_back({host_now_us() - run_t0, 1, g.id});
        const int sz = static_cast<int>(g.tickets.size());
        const int64_t tot = total_us(g);
        const bool per = g.stamped && (profiled || t_out < kNoTimeoutUs);
        uint64_t last = 0;
        for (int i = 0; per && i < sz; ++i) last = std::max(last, ctx.sample_stamp(g.tickets[i]));
        if (!per && g.n_got == 0 && g.part_idx.empty()) {
            // the common case -- a whole group finishing together: hand it on in bulk
            const bool slow_all = parked_group || tot > t_out;   // inclusive budget, balancer.cpp:17
            const uint8_t cv = slow_all ? 2 : 1;
            std::fill(g.got.begin(), g.got.end(), cv);
            g.n_got = sz;
            for (int64_t t : g.tickets) {
                cls[static_cast<size_t>(t - tbase)] = cv;
                if (sample_class) sample_class[t - tbase] = cv;
            }
            (slow_all ? rep.slow : rep.fast) += sz;
            if (sync) {
                for (int64_t t : g.tickets) ready_pos[static_cast<size_t>(t - tbase)] = 1;
            } else if (slow_all) {
                slow.insert(slow.end(), g.tickets.begin(), g.tickets.end());
            } else {
                fast.insert(fast.end(), g.tickets.begin(), g.tickets.end());
                for (int64_t t : g.tickets) {
                    const int b = ctx.tickets[t].buf;
                    if (b >= static_cast<int>(fast_cnt.size())) fast_cnt.resize(static_cast<size_t>(b) + 1, 0);
                    if (++fast_cnt[b] == B && ctx.buf_closed_count(b) == B) full_bufs.push_back(b);
                }
            }
            for (int i = 0; profiled && i < sz; ++i) prof.record(tot, slow_all);
            if (nbatches >= rc.warmup_batches) kernel_ms += tot / 1000.0;
            est_group_us = static_cast<int64_t>(0.8 * est_group_us + 0.2 * 0.7 * (tot > 0 ? tot : host_now_us() - g.t_launch_us));
            release_group(g);
            return;
        }
        std::vector<uint8_t> in_part(static_cast<size_t>(sz), 0);
        for (int i : g.part_idx) in_part[static_cast<size_t>(i)] = 1;
        for (int i = 0; i < sz; ++i) {
            int64_t us = in_part[static_cast<size_t>(i)] ? static_cast<int64_t>(std::llround(g.part_ms * 1000.0)) : tot;
            if (per) {
                const uint64_t st = ctx.sample_stamp(g.tickets[i]);
                if (st != 0 && last >= st) us = std::max<int64_t>(0, tot - static_cast<int64_t>((last - st) / 1000));
            }
            if (!g.got[static_cast<size_t>(i)]) hand_on(g, i, parked_group || us > t_out);   // inclusive budget, balancer.cpp:17
            if (profiled) prof.record(us, g.got[static_cast<size_t>(i)] == 2);
        }
        if (nbatches >= rc.warmup_batches) kernel_ms += tot / 1000.0;
        est_group_us = static_cast<int64_t>(0.8 * est_group_us + 0.2 * 0.7 * (tot > 0 ? tot : host_now_us() - g.t_launch_us));
        release_group(g);
    };

    // Parameter prefetch: the per-sample draws (mt19937_64 keyed by id, ~0.5 us each
    // with the lazily seeded generator) are a pure function of (seed, id, dims), so
    // the context's worker threads draw them ahead of the submit loop, chunk by
    // chunk; the first chunks are small so the first launch group is ready soon.
    // One worker first has the kernel populate the run's fresh ticket storage
    // (MADV_POPULATE_WRITE leaves contents untouched, so it may run while submit
    // constructs tickets) instead of the submitting thread taking one page fault
    // per ~15 tickets.
    constexpr int64_t kChunk = 32;
    const int64_t n_chunks = (n + kChunk - 1) / kChunk;
    // (the context keeps this table between runs: its pages stay mapped and warm)
    std::vector<PreDraw>& pre = ctx.pre_store;
    if (pre.size() < static_cast<size_t>(n)) {   // grow without copying the old (scratch) entries
        std::vector<PreDraw> fresh(static_cast<size_t>(n));
        pre.swap(fresh);
    }
    std::unique_ptr<std::atomic<uint8_t>[]> ready(new std::atomic<uint8_t>[std::max<int64_t>(n_chunks, 1)]);
    for (int64_t i = 0; i < n_chunks; ++i) ready[i].store(0, std::memory_order_relaxed);
    std::atomic<int64_t> next_chunk{0};
    std::atomic<bool> stop_draw{false};
    uintptr_t pop_lo = 0, pop_hi = 0;
    if (!std::getenv("LFG_NO_POPULATE")) {   // (A/B switch)
        const uintptr_t pg = 4096;
        pop_lo = (reinterpret_cast<uintptr_t>(ctx.tickets.data() + tbase) + pg - 1) & ~(pg - 1);
        pop_hi = reinterpret_cast<uintptr_t>(ctx.tickets.data() + tbase + n) & ~(pg - 1);
        if (pop_hi <= pop_lo + (1u << 20)) pop_lo = pop_hi = 0;
    }
    const bool draw = src == nullptr && n > 0;
    if (draw || pop_hi > pop_lo) {
        ctx.workers->run([&, draw](int w) {
            if (w == ctx.workers->size() - 1 && pop_hi > pop_lo) {
                for (uintptr_t p = pop_lo; p < pop_hi && !stop_draw.load(std::memory_order_relaxed);
                     p += (1u << 20))   // in 1 MB steps, front first
                    madvise(reinterpret_cast<void*>(p), std::min<uintptr_t>(1u << 20, pop_hi - p), kMadvPopulateWrite);
            }
            if (!draw) return;
            for (;;) {
                const int64_t ck = next_chunk.fetch_add(1);
                if (ck >= n_chunks || stop_draw.load(std::memory_order_relaxed)) return;
                for (int64_t i = ck * kChunk; i < std::min(n, (ck + 1) * kChunk); ++i)
                    draw_params(*chain, ctx.cfg.seed, samples[i], pre[i]);
                ready[ck].store(1, std::memory_order_release);
            }
        });
    }
    struct Joiner {   // the workers reference this run's tables: wait for them on every exit path
        WorkerThreads& w;
        std::atomic<bool>& stop;
        bool on;
        ~Joiner() {
            if (!on) return;
            stop.store(true);
            w.wait();
        }
    } joiner{*ctx.workers, stop_draw, draw || pop_hi > pop_lo};

    Phases ph;
    ctx.prof_on = ph.on;
    const double g_ns0 = ctx.prof_group_ns, l_ns0 = ctx.prof_launch_ns;
    const double v_ns0 = ctx.prof_views_ns, d_ns0 = ctx.prof_desc_ns;
    const double q_ns0 = ctx.prof_query_ns, f_ns0 = ctx.prof_final_ns;
    const int64_t nq0 = ctx.prof_queries;
    int64_t iters = 0, idle_passes = 0;
    const size_t groups0 = ctx.groups.size();
    // Full scans (every in-flight group's event queried) every 10 us when timeouts
    // or the profiler need prompt completions.  Without them a group's samples only
    // matter once sealable, and the groups complete nearly in launch order, so the
    // oldest group is queried each pass and a full scan (~0.7 us per event query on
    // the submitting thread) runs every 500 us.
    const int64_t kScanUs = (t_out < kNoTimeoutUs || profiled) ? 10 : 500;
    int64_t last_scan_us = 0;
    ph.start();
    ph.setup_ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - setup_t0).count();
    while (consumed < n) {
        bool progressed = false;
        ++iters;
        const int64_t now = host_now_us();

        // (1) in-flight groups.  Samples whose completion stamp landed are handed on
        // (fast: the group is within budget).  A group finished in budget hands on the
        // rest; over budget, its unfinished samples are slow and the group is parked.
        // An event query costs ~0.5 us with 32 hardware queues, so groups are queried
        // in launch order up to the first unfinished one, and all of them only every
        // kScanUs (out-of-order finishers are picked up within that); a group is
        // always queried before it is parked for its timeout.  Stamps are plain reads.
        const bool full_scan = now - last_scan_us >= kScanUs;
        if (full_scan) last_scan_us = now;
        bool query = true;
        for (size_t k = 0; k < inflight.size();) {
            Group& g = ctx.groups[inflight[k]];
            const bool over = now - g.t_launch_us > t_out;
            const int sz = static_cast<int>(g.tickets.size());
            if (g.stamped && g.n_got < sz && scan_stamps(g, full_scan || over, false)) progressed = true;
            if ((query || full_scan || over) && check_part(g, false)) progressed = true;
            // a group is not queried before ~70% of the recent groups' device time has
            // passed since its launch (the query would only cost the submitting thread)
            const bool due = now - g.t_launch_us >= est_group_us;
            const bool done = ((query && due) || full_scan || over || g.n_got == sz) && ctx.poll_group(g);
            if (!done) query = false;
            bool remove = false;
            if (done) {
                finish_group(g, false);
                remove = true;
            } else if (over) {
                parked.push_back(inflight[k]);   // its unfinished samples are slow
                remove = true;
            }
            if (remove) {
                inflight.erase(inflight.begin() + static_cast<long>(k));  // keep launch order
                progressed = true;
            } else {
                ++k;
            }
        }
        ph.lap(Phases::POLL);
        // (2) parked groups finishing in the background (resume_slow, balancer.cpp:96-113):
        // their remaining samples reach the slow list as their stamps land
        for (size_t k = 0; k < parked.size();) {
            Group& g = ctx.groups[parked[k]];
            const int sz = static_cast<int>(g.tickets.size());
            if (g.stamped && g.n_got < sz && scan_stamps(g, full_scan, true)) progressed = true;
            if (full_scan && check_part(g, true)) progressed = true;
            if ((full_scan || g.n_got == sz) && ctx.poll_group(g)) {
                finish_group(g, true);
                parked.erase(parked.begin() + static_cast<long>(k));
                progressed = true;
            } else {
                ++k;
            }
        }
        ph.lap(Phases::PARKED);
        // (3) feed new samples while a worker (stream) is free
        // policy 3 feeds at most prefetch_factor x workers batches ahead of the oldest
        // unsealed one (the sync loader's claim window, baselines.cpp:115-151)
        const int64_t sync_window = sync && rc.prefetch_factor > 0
                                        ? (sync_next / B + int64_t(rc.prefetch_factor) * n_workers) * B
                                        : n;
        while (static_cast<int>(inflight.size()) < n_workers && fed < std::min(n, sync_window) &&
               (ctx.serial || ctx.free_stream_count() > 0)) {
            const int64_t take = std::min<int64_t>(group, std::min(n, sync_window) - fed);
            int64_t got = 0;
            int64_t gid = -1;
            try {
                for (; got < take; ++got) {
                    const int64_t i = fed + got;
                    if (src != nullptr) {   // streaming input: fetch and draw in feed order
                        if (i >= fetched) {
                            const int r = src->next(src->user, &src_descs[static_cast<size_t>(i)]);
                            if (r == 2) break;
                            if (r == 0) fail(LFG_ERR_STATE, "source ended before n samples");
                            if (r != 1) fail(LFG_ERR_INVALID, "source next() failed");
                            draw_params(*chain, ctx.cfg.seed, src_descs[static_cast<size_t>(i)], pre[i]);
                            fetched = i + 1;
                        }
                    } else if (!ready[i / kChunk].load(std::memory_order_acquire)) {
                        ph.lap(Phases::SUBMIT);
                        // help rather than wait: draw the next unclaimed chunk (the
                        // workers may still be waking up at the start of a run)
                        while (!ready[i / kChunk].load(std::memory_order_acquire)) {
                            const int64_t ck = next_chunk.fetch_add(1);
                            if (ck >= n_chunks) {
                                std::this_thread::yield();
                                continue;
                            }
                            for (int64_t q = ck * kChunk; q < std::min(n, (ck + 1) * kChunk); ++q)
                                draw_params(*chain, ctx.cfg.seed, samples[q], pre[q]);
                            ready[ck].store(1, std::memory_order_release);
                        }
                        ph.lap(Phases::DRAW);
                    }
                    const int64_t t = ctx.submit(chain, samples[i], &pre[i]);
                    gid = ctx.tickets[t].group;
                }
            } catch (const Error& e) {
                if (e.code != LFG_ERR_AGAIN) throw;
            }
            ph.lap(Phases::SUBMIT);
            if (got == 0) break;
            ctx.flush();
            ph.lap(Phases::FLUSH);
            fed += got;
            inflight.push_back(gid);
            if (trace_on) trace.push_back({host_now_us() - run_t0, 0, gid});
            progressed = true;
            if (got < take) break;
            // keep feeding while the oldest in-flight group is still running; once it has
            // finished, go poll and seal first, so the first batches are not held back
            // behind the whole feed (one event query, only once the group is due)
            if (inflight.size() > 1) {
                Group& og = ctx.groups[inflight.front()];
                if (host_now_us() - og.t_launch_us >= est_group_us && ctx.poll_group(og)) break;
            }
        }
        // (4) batcher: seal eagerly, fast first
        const bool tail = fed == n && inflight.empty() && parked.empty();
        auto sync_ready = [&]() {
            if (sync_next >= n) return false;
            const int64_t k = std::min<int64_t>(B, n - sync_next);
            if (sync_next + k > fed) return false;
            for (int64_t i = sync_next; i < sync_next + k; ++i)
                if (!ready_pos[static_cast<size_t>(i)]) return false;
            return true;
        };
        while (sync ? sync_ready()
                    : (static_cast<int64_t>(fast.size() + slow.size()) >= B || (tail && !fast.empty()) ||
                       (tail && !slow.empty()))) {
            const int64_t k = sync ? std::min<int64_t>(B, n - sync_next)
                                   : std::min<int64_t>(B, static_cast<int64_t>(fast.size() + slow.size()));
            std::vector<int64_t> ts;
            ts.reserve(static_cast<size_t>(k));
            if (sync)
                for (int64_t i = 0; i < k; ++i) ts.push_back(tbase + sync_next + i);
            // Zero-copy preference: if every sample of some closed slot buffer is
            // in the fast list, seal exactly those (the buffer becomes the batch).
            // Eagerness is unchanged -- a batch is sealed whenever B samples are
            // ready -- only its membership is chosen to avoid the gather copy.
            while (!full_bufs.empty() && (fast_cnt[full_bufs.front()] != B ||
                                          ctx.buf_closed_count(full_bufs.front()) != B))
                full_bufs.pop_front();   // stale candidate
            if (!sync && k == B && !full_bufs.empty()) {
                const int pick = full_bufs.front();
                full_bufs.pop_front();
                bool at_front = true;   // common case: the buffer's samples lead the fast list
                for (int64_t i = 0; i < B && at_front; ++i)
                    at_front = ctx.tickets[fast[static_cast<size_t>(i)]].buf == pick;
                if (at_front) {   // (bulk: the first B entries are exactly buffer `pick`)
                    ts.assign(fast.begin(), fast.begin() + B);
                    fast.erase(fast.begin(), fast.begin() + B);
                    fast_cnt[pick] -= static_cast<int>(B);
                } else {
                    for (auto it = fast.begin(); it != fast.end();) {
                        if (ctx.tickets[*it].buf == pick) {
                            ts.push_back(*it);
                            it = fast.erase(it);
                        } else {
                            ++it;
                        }
                    }
                    fast_cnt[pick] = 0;
                }
            }
            for (int64_t i = static_cast<int64_t>(ts.size()); i < k; ++i) {
                if (!fast.empty()) {
                    ts.push_back(fast_take());
                } else {
                    ts.push_back(slow.front());
                    slow.pop_front();
                }
            }
            int64_t b;
            try {
                b = ctx.seal(ts.data(), static_cast<int>(k));
                ph.lap(Phases::SEAL);
            } catch (const Error& e) {
                ph.lap(Phases::SEAL);
                if (e.code != LFG_ERR_AGAIN) throw;
                if (sync) break;   // the batch stays ready; retried next pass
                for (auto it = ts.rbegin(); it != ts.rend(); ++it) {
                    if (cls[static_cast<size_t>(*it - tbase)] == 2) slow.push_front(*it);
                    else fast_add(*it, true);
                }
                break;
            }
            BatchRec& br = ctx.batch(b);
            if (sync) sync_next += k;
            if (trace_on) trace.push_back({host_now_us() - run_t0, 2, nbatches});
            const bool timed = nbatches >= rc.warmup_batches;
            if (ss != nullptr) {
                // the consumer owns the batch: the trainer stream only marks its delivery
                // (the run's device-timed span) and carries the captures / probe
                ctx.batch_wait_stream(b, trainer);
            } else if (timed && rc.trainer_us > 0) {
                cudaEvent_t s0 = mk(), s1 = mk();
                ctx.batch_wait_stream(b, trainer);
                cuda_check(cudaEventRecord(s0, trainer), "record");
                ctx.trainer_step(b, trainer, rc.trainer_us);
                cuda_check(cudaEventRecord(s1, trainer), "record");
                steps.emplace_back(s0, s1);
            } else if (rc.trainer_us > 0 || probe) {
                ctx.trainer_step(b, trainer, rc.trainer_us);
            }
            bool captured = false;
            if (!cap_slot.empty()) {
                for (size_t q = 0; q < ts.size(); ++q) {
                    const int k = cap_slot[static_cast<size_t>(ts[q] - tbase)];
                    if (k < 0) continue;
                    // batch position: the slot (zero-copy seal) or the seal order (collated)
                    const int pos = br.in_place ? ctx.tickets[ts[q]].pos : static_cast<int>(q);
                    probe_bytes += ctx.capture_sample(b, pos, static_cast<char*>(rc.capture_buf) + k * rc.capture_stride,
                                                      rc.capture_stride, trainer);
                    if (rc.capture_done) rc.capture_done[k] = static_cast<int32_t>(nbatches + 1);
                    captured = true;
                }
            }
            if (probe) {
                void* bp = nullptr;
                int64_t bb = 0;
                ctx.batch_ptr(br, &bp, &bb);
                cuda_check(cudaMemcpyAsync(probe + 16 * (nbatches % 1024), bp, 16,
                                           cudaMemcpyDeviceToHost, trainer),
                           "probe D2H");
                probe_bytes += 16;
            }
            for (uint64_t id : br.ids) {
                if (consumed_ids) consumed_ids[consumed] = id;
                all_ids.push_back(id);
                ++consumed;
            }
            if (batch_sizes) batch_sizes[nbatches] = br.n;
            if (timed) timed_samples += br.n;
            if (rc.scheduler) {
                cudaEvent_t ce = mk();
                cuda_check(cudaEventRecord(ce, trainer), "record consume");
                consume_q.push_back(ce);
            }
            if (ss != nullptr) {
                if (captured || probe != nullptr) {   // the consumer's wait also covers the reads queued here
                    if (br.ready == nullptr) br.ready = ctx.make_ready_event();
                    cuda_check(cudaEventRecord(br.ready, trainer), "record delivery");
                }
            } else {
                ctx.batch_release(b, trainer, rc.trainer_us > 0 || probe != nullptr || captured);
            }
            for (int64_t t : ts) ctx.ticket_release(t);
            if (ss != nullptr) ss->deliver(ss->user, b, br.n);
            ++nbatches;
            if (nbatches == rc.warmup_batches) {
                t_timed = mk();
                cuda_check(cudaEventRecord(t_timed, trainer), "record");
            }
            progressed = true;
            ph.lap(Phases::DELIVER);
        }
        // (5a) adaptive scheduler tick
        if (rc.scheduler) {
            const int64_t t = host_now_us();
            if (sched_prev_t == 0) sched_prev_t = sched_last = sched_t0 = t;
            const double dt = static_cast<double>(t - sched_prev_t);
            busy_integral += dt * static_cast<double>(inflight.size());
            workers_integral += dt * static_cast<double>(n_workers);
            sched_prev_t = t;
            if (t - sched_last >= sched_tick) {
                while (!consume_q.empty() && cudaEventQuery(consume_q.front()) == cudaSuccess)
                    consume_q.pop_front();
                sched_ema = 0.3 * static_cast<double>(consume_q.size()) + 0.7 * sched_ema;
                const double span = static_cast<double>(t - sched_last) * std::max(1, n_workers);
                const double c_usage = std::clamp(busy_integral / span, 0.0, 1.0);
                const int delta = lf_sched_delta(std::clamp(sched_ema, 0.0, q_max), c_usage, 2.0, 2.0, 0.7,
                                                 q_max, 2);
                n_workers = lf_sched_update(n_workers, delta, max_workers);
                busy_integral = 0.0;
                sched_last = t;
                ++sched_ticks;
            }
        }
        // (5) profiler maintenance (profiler_loop, profiler.cpp:108-121)
        if ((rc.policy == 1 || rc.policy == 2) && !prof.window.empty() && now - run_t0 >= rc.warmup_us &&
            now - last_update >= std::max<int64_t>(1, rc.update_interval_us)) {
            t_out = prof.update();
            last_update = now;
        }
        if (!progressed) {
            if (inflight.empty() && parked.empty() && fed == n && fast.empty() && slow.empty() &&
                !(sync && sync_next < n))
                fail(LFG_ERR_STATE, "shard stalled with samples unaccounted for");
        }
        idle_passes = progressed ? 0 : idle_passes + 1;
        if (lk.owns_lock()) {
            // between passes the consumer's batch calls take the context lock; a loop
            // that has waited a while (the consumer holds every batch buffer) naps
            lk.unlock();
            if (idle_passes > 256) std::this_thread::sleep_for(std::chrono::microseconds(20));
            else if (idle_passes > 0) std::this_thread::yield();
            lk.lock();
        } else if (!progressed) {
            std::this_thread::yield();
        }
        ph.lap(Phases::IDLE);
    }
    // every sample is consumed; groups whose samples were all handed on by their
    // stamps may still be finishing their last kernel: complete them
    while (!inflight.empty() || !parked.empty()) {
        for (auto* lst : {&inflight, &parked}) {
            for (size_t k = 0; k < lst->size();) {
                Group& g = ctx.groups[(*lst)[k]];
                if (ctx.poll_group(g)) {
                    finish_group(g, lst == &parked);
                    lst->erase(lst->begin() + static_cast<long>(k));
                } else {
                    ++k;
                }
            }
        }
        if (!inflight.empty() || !parked.empty()) {
            if (lk.owns_lock()) lk.unlock();
            std::this_thread::yield();
            if (ss != nullptr) lk.lock();
        }
    }
    ph.print(n, ctx.prof_group_ns - g_ns0, ctx.prof_launch_ns - l_ns0,
             static_cast<int64_t>(ctx.groups.size() - groups0));
    if (ph.on)
        std::fprintf(stderr, "[lfg shard] per group: views=%.0f desc=%.0f query=%.0f (%.1f queries) final=%.0f ns; %.1f loop passes\n",
                     (ctx.prof_views_ns - v_ns0) / double(std::max<size_t>(1, ctx.groups.size() - groups0)),
                     (ctx.prof_desc_ns - d_ns0) / double(std::max<size_t>(1, ctx.groups.size() - groups0)),
                     (ctx.prof_query_ns - q_ns0) / double(std::max<size_t>(1, ctx.groups.size() - groups0)),
                     double(ctx.prof_queries - nq0) / double(std::max<size_t>(1, ctx.groups.size() - groups0)),
                     (ctx.prof_final_ns - f_ns0) / double(std::max<size_t>(1, ctx.groups.size() - groups0)),
                     double(iters) / double(std::max<size_t>(1, ctx.groups.size() - groups0)));
    chain->est_group_us = est_group_us;
    ctx.forget_pinned();   // payload pages are re-validated by the next run (the caller may free them now)
    if (trace_on) {
        static const char* kinds[3] = {"fed", "done", "sealed"};
        std::fprintf(stderr, "[lfg trace] n=%lld:", static_cast<long long>(n));
        for (const auto& e : trace) std::fprintf(stderr, " %s%lld@%lld", kinds[e.kind], static_cast<long long>(e.id), static_cast<long long>(e.t_us));
        std::fprintf(stderr, " end@%lld\n", static_cast<long long>(host_now_us() - run_t0));
    }
    cudaEvent_t t_end = mk();
    cuda_check(cudaEventRecord(t_end, trainer), "record");
    cuda_check(cudaEventSynchronize(t_end), "sync");

    float el = 0;
    cuda_check(cudaEventElapsedTime(&el, t_timed, t_end), "elapsed");
    double busy = 0;
    for (auto& s : steps) {
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, s.first, s.second), "elapsed");
        busy += ms;
    }
    for (auto e : evs) cudaEventDestroy(e);
    if (probe) cudaFreeHost(probe);
    cudaStreamDestroy(trainer);

    // exactly-once audit (experiment.cpp:396-413)
    std::vector<uint64_t> want(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) want[i] = samples[i].id;
    std::sort(want.begin(), want.end());
    std::sort(all_ids.begin(), all_ids.end());
    int64_t dups = 0;
    for (size_t i = 1; i < all_ids.size(); ++i) dups += all_ids[i] == all_ids[i - 1];

    rep.samples = consumed;
    rep.batches = nbatches;
    rep.short_batches = 0;
    if (batch_sizes)
        for (int64_t i = 0; i < nbatches; ++i) rep.short_batches += batch_sizes[i] < B;
    rep.inplace_batches = ctx.counters.inplace_batches - c0.inplace_batches;
    rep.elapsed_ms = el;
    rep.timed_samples = static_cast<double>(timed_samples);
    rep.samples_per_s = el > 0 ? timed_samples / (el / 1000.0) : 0.0;
    rep.consumer_busy_ms = busy;
    rep.consumer_span_ms = el;
    rep.consumer_idle_frac = (rc.trainer_us > 0 && el > 0) ? 1.0 - busy / el : 1.0;
    rep.final_t_out_us = static_cast<double>(t_out >= kNoTimeoutUs ? -1 : t_out);
    rep.final_percentile = prof.pct;
    rep.pct_up = prof.up;
    rep.pct_down = prof.down;
    rep.profiled = prof.recorded;
    rep.exactly_once = (all_ids == want && dups == 0) ? 1 : 0;
    rep.duplicates = dups;
    rep.kernel_ms = kernel_ms;
    rep.h2d_bytes = ctx.counters.h2d_bytes - c0.h2d_bytes;
    rep.d2h_bytes = ctx.counters.d2h_bytes - c0.d2h_bytes + probe_bytes;
    rep.launches = ctx.counters.launches - c0.launches;
    rep.final_workers = n_workers;
    rep.sched_ticks = static_cast<int32_t>(sched_ticks);
    rep.mean_workers = workers_integral > 0 && sched_prev_t > sched_t0
                           ? workers_integral / static_cast<double>(sched_prev_t - sched_t0)
                           : static_cast<double>(n_workers);
    return LFG_OK;
}

}  // namespace lfg
