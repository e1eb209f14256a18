// lf_gpu.cpp -- the device branch of the reference-shaped API: process_sample,
// resume_slow, the batcher's seal and the consumer's release for chains whose
// transforms carry device ops.  Everything goes through the C ABI
// (include/lfgpu.h, liblfgpu.so); no CUDA types appear here.
//
// Realtime runtimes: process_sample submits the sample, then polls its
// per-stage CUDA events against t_out on the runtime clock (a microsecond
// tick via make_realtime_runtime_ticks(1000) makes device budgets
// representable).  A budget overrun classifies the sample slow and parks it
// in the temp queue with timeout_index = the first unfinished op; nothing is
// preempted or re-executed -- resume_slow waits for the completion event.
//
// Virtual runtimes (tests): device work is waited for synchronously and its
// device-measured duration is charged to the virtual clock, exactly like a
// synthetic cost model, so the reference's deterministic tests apply.
#include <cmath>
#include <cstring>
#include <map>
#include <unordered_map>
#include <mutex>
#include <thread>


#include "loadflow/api.hpp"

namespace loadflow {

namespace {

std::mutex g_mu;
std::vector<lfg_ctx*> g_shards;
// Compiled chains keyed by context and by the CONTENTS of the device op list
// (kind, params, size factor, barrier, name), not by the TransformChain's
// address: a chain destroyed and rebuilt at the same address, or edited after
// its first use, must never reuse a stale compiled chain.
std::map<std::pair<lfg_ctx*, std::string>, lfg_chain*> g_chains;

void check(int rc) {
    if (rc == LFG_OK) return;
    const std::string msg = lfg_last_error();
    switch (rc) {
        case LFG_ERR_INVALID: throw std::invalid_argument(msg);
        case LFG_ERR_STATE: throw std::logic_error(msg);
        case LFG_ERR_CLOSED: throw QueueClosedError(msg);
        default: throw std::runtime_error("lfgpu error " + std::to_string(rc) + ": " + msg);
    }
}

// A full output pool (LFG_ERR_AGAIN: every slot / batch buffer holds samples the
// batcher or consumer has not released yet) is back-pressure: the caller waits, as
// BoundedQueue::put blocks on a full queue (queue.hpp:57-59), instead of failing.
template <typename F>
void retry_full(F&& call) {
    for (int k = 0;; ++k) {
        const int rc = call();
        if (rc != LFG_ERR_AGAIN) {
            check(rc);
            return;
        }
        if (k < 64) std::this_thread::yield();
        else std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

lfg_ctx* ctx_of(const Sample& s) {
    lfg_ctx* c = gpu::shard_context(s.device.shard);
    if (c == nullptr) throw std::logic_error("device chain used without a bound GPU shard");
    return c;
}

lfg_chain* compiled(lfg_ctx* ctx, const TransformChain& chain) {
    std::vector<lfg_op> ops;
    for (const Transform& t : chain.transforms()) {
        lfg_op o;
        std::memset(&o, 0, sizeof(o));   // the key compares bytes: no padding garbage
        o.kind = t.device.op.kind;
        for (int k = 0; k < 8; ++k) o.param[k] = t.device.op.param[k];
        o.size_factor = t.size_factor;
        o.barrier = t.barrier;
        std::snprintf(o.name, sizeof(o.name), "%s", t.name.c_str());
        ops.push_back(o);
    }
    std::lock_guard<std::mutex> g(g_mu);
    auto key = std::make_pair(ctx, std::string(reinterpret_cast<const char*>(ops.data()),
                                               ops.size() * sizeof(lfg_op)));
    auto it = g_chains.find(key);
    if (it != g_chains.end()) return it->second;
    lfg_chain* h = nullptr;
    check(lfg_chain_create(ctx, ops.data(), static_cast<int>(ops.size()), &h));
    g_chains[key] = h;
    return h;
}

std::vector<DurationMs> device_costs(lfg_ctx* ctx, std::int64_t ticket, std::size_t n,
                                     std::int64_t tick_ns) {
    std::vector<double> us(n);
    int got = 0;
    check(lfg_exec_costs(ctx, ticket, us.data(), static_cast<int>(n), &got));
    std::vector<DurationMs> out(n);
    for (std::size_t i = 0; i < n; ++i)
        out[i] = static_cast<DurationMs>(std::llround(us[i] * 1000.0 / static_cast<double>(tick_ns)));
    return out;
}

void advance_to(Sample& s, std::size_t upto) {
    for (std::size_t i = s.next_index; i < upto; ++i) s.size_bytes *= s.chain->at(i).size_factor;
    s.next_index = upto;
}

}  // namespace

namespace gpu {

int bind_shard(lfg_ctx* ctx) {
    std::lock_guard<std::mutex> g(g_mu);
    g_shards.push_back(ctx);
    return static_cast<int>(g_shards.size()) - 1;
}

lfg_ctx* shard_context(int shard) {
    std::lock_guard<std::mutex> g(g_mu);
    return shard >= 0 && shard < static_cast<int>(g_shards.size()) ? g_shards[shard] : nullptr;
}

void unbind_all() {
    std::lock_guard<std::mutex> g(g_mu);
    for (auto& kv : g_chains) lfg_chain_destroy(kv.first.first, kv.second);
    g_chains.clear();
    g_shards.clear();
}

namespace {
Transform dev(const char* name, double factor, int kind, std::initializer_list<double> params) {
    Transform t;
    t.name = name;
    t.size_factor = factor;
    t.device.op.kind = kind;
    int i = 0;
    for (double p : params) t.device.op.param[i++] = p;
    return t;
}
}  // namespace

TransformChain img_seg_chain(int crop) {
    // proj/src/workloads.cpp:142-148, MLPerf 3D-UNet probabilities
    const double c = crop;
    return TransformChain({dev("RandomCrop", 0.0735, LFG_OP_RANDOM_CROP, {c, c, c}),
                           dev("RandomFlip", 1.0, LFG_OP_RANDOM_FLIP, {1.0 / 3.0}),
                           dev("RandomBrightness", 1.0, LFG_OP_RANDOM_BRIGHTNESS, {0.1, 0.7, 1.3}),
                           dev("GaussianNoise", 1.0, LFG_OP_GAUSSIAN_NOISE, {0.1, 0.1}),
                           dev("Cast", 1.0, LFG_OP_CAST, {})});
}

TransformChain obj_det_chain(int out) {
    // proj/src/workloads.cpp:151-156 with torchvision RandomResizedCrop defaults
    const double o = out;
    return TransformChain(
        {dev("Resize", 1.2, LFG_OP_RESIZE, {o, o, 0.08, 1.0, 3.0 / 4.0, 4.0 / 3.0}),
         dev("RandomHorizontalFlip", 1.0, LFG_OP_RANDOM_HFLIP, {0.5}),
         dev("ToTensor", 8.0, LFG_OP_TO_TENSOR, {}),
         dev("Normalize", 1.0, LFG_OP_NORMALIZE, {0.485, 0.456, 0.406, 0.229, 0.224, 0.225})});
}

void prepare_chain(const TransformChain& chain, int shard) {
    lfg_ctx* c = shard_context(shard);
    if (c == nullptr) throw std::logic_error("prepare_chain: no GPU shard bound");
    compiled(c, chain);
}

void seal_device_batch(Batch& b) {
    if (b.samples.empty() || b.samples.front().device.ticket < 0) return;
    lfg_ctx* ctx = ctx_of(b.samples.front());
    std::vector<lfg_ticket> ts;
    for (const Sample& s : b.samples) ts.push_back(s.device.ticket);
    lfg_batch h = -1;
    retry_full([&] { return lfg_seal_batch(ctx, ts.data(), static_cast<int>(ts.size()), &h); });
    for (lfg_ticket t : ts) check(lfg_ticket_release(ctx, t));
    b.device_batch = h;
}

lfg_run_report feed_shard(const TransformChain& chain, std::vector<Sample> samples, BatchQueue& out, Runtime& rt,
                          const lfg_run_config& cfg) {
    if (samples.empty()) {
        out.close();
        return lfg_run_report{};
    }
    lfg_ctx* ctx = ctx_of(samples.front());
    lfg_chain* ch = compiled(ctx, chain);
    std::vector<lfg_sample_desc> descs(samples.size());
    std::unordered_map<uint64_t, size_t> where;
    where.reserve(samples.size());
    for (size_t i = 0; i < samples.size(); ++i) {
        descs[i] = samples[i].device.desc;
        descs[i].id = samples[i].id;
        where.emplace(samples[i].id, i);
    }
    lfg_shard* sh = nullptr;
    check(lfg_shard_start(ctx, ch, descs.data(), static_cast<int64_t>(descs.size()), &cfg, &sh));
    std::vector<uint64_t> ids(static_cast<size_t>(std::max(1, 256)));
    int rc = LFG_OK;
    for (;;) {
        lfg_batch b = -1;
        int nb = 0;
        rc = lfg_shard_next_batch(sh, -1, &b, &nb);
        if (rc != LFG_OK) break;
        if (static_cast<size_t>(nb) > ids.size()) ids.resize(static_cast<size_t>(nb));
        void* p = nullptr;
        int64_t bytes = 0;
        int n = 0, inplace = 0;
        rc = lfg_batch_info(ctx, b, &p, &bytes, &n, ids.data(), &inplace);
        if (rc != LFG_OK) break;
        Batch batch;
        batch.samples.reserve(static_cast<size_t>(n));
        for (int k = 0; k < n; ++k) {
            const Sample& src = samples[where.at(ids[static_cast<size_t>(k)])];
            Sample s;   // the delivered sample's identity and accounting (its payload stays on the device)
            s.id = src.id;
            s.chain = src.chain;
            s.bytes_in = src.bytes_in;
            s.size_bytes = src.size_bytes;
            s.bytes_out = src.bytes_out;
            s.device.shard = src.device.shard;
            s.device.desc = descs[where.at(src.id)];
            batch.samples.push_back(std::move(s));
        }
        batch.sealed_at = rt.now();
        batch.device_batch = b;
        out.put(std::move(batch));   // blocks while the consumer is behind (back-pressure)
    }
    out.close();
    lfg_run_report rep{};
    const int frc = lfg_shard_finish(sh, &rep, nullptr, nullptr, nullptr);
    if (rc != LFG_ERR_CLOSED) check(rc);
    check(frc);
    return rep;
}

}  // namespace gpu

namespace detail {

RouteResult process_on_device(Sample s, DurationMs t_out, SampleQueue& fast_q, TempQueue& temp_q,
                              Runtime& rt) {
    lfg_ctx* ctx = ctx_of(s);
    lfg_chain* chain = compiled(ctx, *s.chain);
    const std::size_t n = s.chain->size();
    s.device.desc.id = s.id;
    retry_full([&] { return lfg_submit(ctx, chain, &s.device.desc, &s.device.ticket); });
    check(lfg_flush(ctx));
    RouteResult res;
    const TimeMs t0 = rt.now();

    auto park = [&](std::size_t done, DurationMs charged) {
        advance_to(s, done);
        s.classification = SampleClass::slow;
        res.route = Route::temp;
        res.foreground_ms = charged;
        res.timeout_index = done;
        temp_q.put(TempItem{std::move(s), done, res.exec_costs});
        return res;
    };

    if (rt.is_virtual()) {
        check(lfg_wait(ctx, s.device.ticket));
        const auto costs = device_costs(ctx, s.device.ticket, n, rt.tick_ns());
        DurationMs spent = 0;
        for (std::size_t i = 0; i < n; ++i) {
            if (spent + costs[i] > t_out) {
                rt.sleep(t_out - spent);
                return park(i, t_out);
            }
            spent += costs[i];
            rt.sleep(costs[i]);
            res.exec_costs.push_back(costs[i]);
        }
        res.foreground_ms = spent;
    } else {
        const double tick_us = static_cast<double>(rt.tick_ns()) / 1000.0;
        for (;;) {
            int ops_done = 0, complete = 0;
            std::int64_t el_us = 0;
            // block (no polling) until the sample's group finishes or its budget runs out
            const DurationMs left = t_out >= kNoTimeout ? kNoTimeout : t_out - (rt.now() - t0);
            const std::int64_t wait_us =
                left >= kNoTimeout ? 1000000 : std::max<std::int64_t>(1, static_cast<std::int64_t>(left * tick_us) + 1);
            check(lfg_wait_for(ctx, s.device.ticket, std::min<std::int64_t>(wait_us, 1000000), &complete));
            check(lfg_progress(ctx, s.device.ticket, &ops_done, &complete, &el_us));
            const DurationMs el = rt.now() - t0;
            if (complete) {
                res.exec_costs = device_costs(ctx, s.device.ticket, n, rt.tick_ns());
                if (el > t_out) {
                    // finished, but only observed after the budget: charge t_out, slow
                    res.exec_costs.clear();
                    return park(n, el);
                }
                res.foreground_ms = el;
                break;
            }
            if (el > t_out) return park(static_cast<std::size_t>(ops_done), el);
        }
    }
    advance_to(s, n);
    s.classification = SampleClass::fast;
    s.t_ready = rt.now();
    res.route = Route::fast;
    fast_q.put(std::move(s));
    return res;
}

void finish_on_device(Sample& s, std::vector<DurationMs>& costs, Runtime& rt) {
    lfg_ctx* ctx = ctx_of(s);
    check(lfg_wait(ctx, s.device.ticket));
    const auto all = device_costs(ctx, s.device.ticket, s.chain->size(), rt.tick_ns());
    if (rt.is_virtual()) {
        DurationMs rest = 0;
        for (std::size_t i = s.next_index; i < all.size(); ++i) rest += all[i];
        rt.sleep(rest);
    }
    for (std::size_t i = costs.size(); i < all.size(); ++i) costs.push_back(all[i]);
    advance_to(s, s.chain->size());
}

void release_device_batch(Batch& b) {
    if (b.device_batch < 0 || b.samples.empty()) return;
    check(lfg_batch_release(ctx_of(b.samples.front()), b.device_batch, nullptr));
    b.device_batch = -1;
}

}  // namespace detail

}  // namespace loadflow
