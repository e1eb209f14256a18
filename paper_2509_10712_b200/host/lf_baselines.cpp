// lf_baselines.cpp -- the reference's comparison baselines (proj/include/loadflow/
// baselines.hpp:12-47): the synchronous PyTorch-DataLoader-
// like loader with head-of-line blocking, Pecan's AutoOrder and the size
// heuristic.  The GPU counterpart of the sync loader is lfg_run_config.policy
// = 3 (csrc/shard.cpp): batch k = ids [kB, (k+1)B), sealed only when all its
// members are done, in batch order.
#include <algorithm>
#include <memory>
#include <stdexcept>

#include "loadflow/api.hpp"

namespace loadflow {

namespace {

// Shared by the worker actors and the publisher; lives as long as any actor.
struct SyncState {
    std::vector<Sample> samples;
    SyncLoaderConfig cfg;
    std::size_t n_batches = 0;
    std::size_t next_claim = 0;                  // next sample index to hand out
    std::size_t published = 0;                   // batches sealed so far
    std::vector<std::size_t> done;               // members finished, per batch
    std::vector<TimeMs> latest;                  // latest member completion, per batch
    std::unique_ptr<Mutex> mu;
    std::unique_ptr<Cond> cv;
    std::size_t batch_len(std::size_t k) const {
        return std::min(cfg.batch_size, samples.size() - k * cfg.batch_size);
    }
};

}  // namespace

// Workers claim samples strictly in id order, at most prefetch_factor batches per
// worker ahead of the oldest unpublished batch; the publisher seals batch k as soon
// as its last member completes and never before batch k - 1 (FIFO), so
// publish(k) = max(slowest member of k, publish(k - 1)).
void start_sync_loader(Runtime& rt, std::vector<Sample> samples, const SyncLoaderConfig& cfg,
                       BatchQueue& batch_q, std::vector<SyncBatchRecord>* records) {
    if (cfg.batch_size == 0 || cfg.n_workers < 1 || cfg.prefetch_factor < 1)
        throw std::invalid_argument("sync loader needs batch_size, n_workers, prefetch_factor >= 1");
    auto st = std::make_shared<SyncState>();
    st->samples = std::move(samples);
    st->cfg = cfg;
    st->n_batches = (st->samples.size() + cfg.batch_size - 1) / cfg.batch_size;
    st->done.assign(st->n_batches, 0);
    st->latest.assign(st->n_batches, 0);
    st->mu = rt.make_mutex();
    st->cv = rt.make_cond();
    const std::size_t window = static_cast<std::size_t>(cfg.prefetch_factor) * static_cast<std::size_t>(cfg.n_workers);

    for (int w = 0; w < cfg.n_workers; ++w) {
        rt.spawn("sync.worker." + std::to_string(w), [st, &rt, w, window] {
            Rng rng(0x5eedULL ^ (0x9e3779b97f4a7c15ULL * static_cast<std::uint64_t>(w + 1)));
            for (;;) {
                std::size_t i;
                {
                    LockGuard lk(*st->mu);
                    while (st->next_claim < st->samples.size() &&
                           st->next_claim / st->cfg.batch_size >= st->published + window)
                        st->cv->wait(*st->mu);
                    if (st->next_claim >= st->samples.size()) return;
                    i = st->next_claim++;
                }
                Sample& s = st->samples[i];
                apply_all_transforms(s, rt, rng);
                s.classification = SampleClass::fast;
                s.t_ready = rt.now();
                LockGuard lk(*st->mu);
                const std::size_t k = i / st->cfg.batch_size;
                st->done[k]++;
                st->latest[k] = std::max(st->latest[k], s.t_ready);
                st->cv->notify_all();
            }
        });
    }
    rt.spawn("sync.publisher", [st, &rt, &batch_q, records] {
        for (std::size_t k = 0; k < st->n_batches; ++k) {
            Batch b;
            {
                LockGuard lk(*st->mu);
                while (st->done[k] < st->batch_len(k)) st->cv->wait(*st->mu);
                const std::size_t first = k * st->cfg.batch_size;
                for (std::size_t i = first; i < first + st->batch_len(k); ++i)
                    b.samples.push_back(std::move(st->samples[i]));
                st->published = k + 1;
                st->cv->notify_all();
            }
            b.sealed_at = rt.now();
            if (records) records->push_back(SyncBatchRecord{k, b.sealed_at, st->latest[k]});
            batch_q.put(std::move(b));
        }
        batch_q.close();
    });
}

// Pecan AutoOrder: stable three-way partition (deflationary, neutral,
// inflationary) inside every barrier-free run; barriers stay where they are.
TransformChain autoorder(const TransformChain& chain) {
    auto cls = [](const Transform& t) { return t.size_factor < 1.0 ? 0 : (t.size_factor > 1.0 ? 2 : 1); };
    std::vector<Transform> out;
    out.reserve(chain.size());
    for (auto [first, last] : chain.sections()) {
        std::vector<Transform> run;
        for (std::size_t i = first; i < last; ++i) run.push_back(chain.at(i));
        if (!(run.size() == 1 && run[0].barrier))
            std::stable_sort(run.begin(), run.end(),
                             [&](const Transform& a, const Transform& b) { return cls(a) < cls(b); });
        for (auto& t : run) out.push_back(std::move(t));
    }
    return TransformChain(std::move(out));
}

SampleClass size_heuristic_classify(const Sample& sample, double size_cutoff_bytes) {
    if (!(size_cutoff_bytes > 0)) throw std::invalid_argument("size cutoff must be > 0");
    return sample.bytes_in > size_cutoff_bytes ? SampleClass::slow : SampleClass::fast;
}

}  // namespace loadflow
