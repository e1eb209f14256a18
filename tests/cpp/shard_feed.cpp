// shard_feed.cpp -- the reference's own consumer (run_consumer, trainer.cpp:20-66) on the
// high-throughput path: gpu::feed_shard runs an obj_det shard through the event-driven
// loop (lfg_shard_start) and publishes each sealed device batch into a BatchQueue as it is
// sealed; run_consumer takes and releases them (release_device_batch) while later groups
// are still running.  Exit 0 = every sample consumed exactly once, batch sizes as sealed,
// every batch device-resident, one batch tensor's samples equal to the oracle's.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <vector>

#include "loadflow/batcher.hpp"
#include "loadflow/runtime.hpp"
#include "loadflow/trainer.hpp"
#include "../../oracle/lf_oracle.h"   // the checker (test infrastructure)

using namespace loadflow;

#define EXPECT(c)                                                               \
    do {                                                                        \
        if (!(c)) {                                                             \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                           \
        }                                                                       \
    } while (0)

int main() {
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
    lfg_config cfg;
    lfg_config_default(&cfg);
    cfg.batch_size = 32;
    cfg.n_workers = 4;
    cfg.max_group = 32;
    cfg.max_slot_buffers = 12;
    lfg_ctx* ctx = nullptr;
    if (lfg_open(&cfg, &ctx) != LFG_OK) {
        std::fprintf(stderr, "lfg_open: %s\n", lfg_last_error());
        return 2;
    }
    const int shard = gpu::bind_shard(ctx);
    TransformChain chain = gpu::obj_det_chain(224);
    gpu::prepare_chain(chain, shard);

    const int64_t H = 300, W = 360;
    const int pool = 8, n = 32 * 10 + 7;   // a short tail batch
    std::vector<void*> imgs(pool);
    for (int i = 0; i < pool; ++i) {
        EXPECT(lfg_device_alloc(ctx, H * W * 3, &imgs[i]) == LFG_OK);
        EXPECT(lfg_synth_image(ctx, 1, static_cast<uint64_t>(i), H, W, imgs[i], 1) == LFG_OK);
    }
    lfg_synchronize(ctx);
    std::vector<Sample> samples;
    for (int i = 0; i < n; ++i) {
        Sample s;
        s.id = 5000 + static_cast<uint64_t>(i);
        s.chain = &chain;
        s.bytes_in = s.size_bytes = double(H * W * 3);
        s.bytes_out = 3.0 * 224 * 224 * 4;
        s.device.shard = shard;
        s.device.desc.src_kind = LFG_SRC_DEVICE;
        s.device.desc.ndim = 3;
        s.device.desc.dims[0] = H;
        s.device.desc.dims[1] = W;
        s.device.desc.dims[2] = 3;
        s.device.desc.data = imgs[i % pool];
        samples.push_back(s);
    }
    auto rt = make_realtime_runtime_ticks(1000);
    BatchQueue q(*rt, 3, QueueRole::batch);   // small: the feed waits for the consumer
    lfg_run_config rc{};
    rc.batch_size = 32;
    lfg_run_report rep{};
    rt->spawn("shard", [&] { rep = gpu::feed_shard(chain, samples, q, *rt, rc); });
    // one batch tensor checked against the oracle before the consumer runs: take the
    // first batch by hand, then let run_consumer drain the rest
    std::vector<uint8_t> first_out;
    std::vector<uint64_t> first_ids;
    ConsumerStats st;
    rt->spawn("consumer", [&] {
        auto b = q.get();
        if (b) {
            void* p = nullptr;
            int64_t bytes = 0;
            int nb = 0, inplace = 0;
            first_ids.resize(32);
            lfg_batch_info(ctx, b->device_batch, &p, &bytes, &nb, first_ids.data(), &inplace);
            first_ids.resize(static_cast<size_t>(nb));
            first_out.resize(static_cast<size_t>(bytes));
            lfg_batch_copy_to_host(ctx, b->device_batch, first_out.data(), static_cast<size_t>(bytes));
            lfg_batch_release(ctx, b->device_batch, nullptr);
            st.batches = 1;
            st.samples = nb;
            for (uint64_t id : first_ids) st.consumed_ids.push_back(id);
        }
        ConsumerConfig cc;
        cc.compute_per_batch = 50;   // 50 us per batch (microsecond ticks)
        cc.poll_sleep = 20;
        ConsumerStats rest = run_consumer(cc, q, *rt);
        st.batches += rest.batches;
        st.samples += rest.samples;
        st.consumed_ids.insert(st.consumed_ids.end(), rest.consumed_ids.begin(), rest.consumed_ids.end());
    });
    rt->run();

    std::set<uint64_t> got(st.consumed_ids.begin(), st.consumed_ids.end());
    std::printf("consumed %zu (unique %zu) in %lld batches; shard report: samples %lld batches %lld exactly_once %d\n",
                st.consumed_ids.size(), got.size(), static_cast<long long>(st.batches),
                static_cast<long long>(rep.samples), static_cast<long long>(rep.batches), rep.exactly_once);
    EXPECT(st.consumed_ids.size() == static_cast<size_t>(n) && got.size() == static_cast<size_t>(n));
    EXPECT(st.batches == rep.batches && rep.samples == n && rep.exactly_once == 1);
    EXPECT(!first_ids.empty());
    // the first batch against the oracle (obj_det: f32 [3, 224, 224] per slot, batch order)
    const int64_t plane = 3 * 224 * 224;
    double worst = 0;
    std::vector<uint8_t> himg(static_cast<size_t>(H * W * 3));
    for (size_t k = 0; k < first_ids.size(); ++k) {
        const uint64_t id = first_ids[k];
        EXPECT(lfg_memcpy_d2h(ctx, himg.data(), imgs[(id - 5000) % pool], himg.size()) == LFG_OK);
        lfo_cfg2d oc;
        lfo_cfg2d_default(&oc);
        lfo_params2d op;
        lfo_draw2d(&oc, cfg.seed, id, H, W, &op);
        std::vector<double> e(static_cast<size_t>(plane));
        lfo_apply2d(&oc, &op, himg.data(), H, W, e.data());
        const float* g = reinterpret_cast<const float*>(first_out.data()) + k * plane;
        for (int64_t v = 0; v < plane; ++v)
            worst = std::max(worst, std::fabs(g[v] - e[v]) / (1e-5 * std::fabs(e[v]) + 1e-5));
    }
    std::printf("first batch vs oracle: worst err/bound %.3f\n", worst);
    EXPECT(worst <= 1.0);
    gpu::unbind_all();
    for (void* p : imgs) lfg_device_free(ctx, p);
    lfg_close(ctx);
    std::printf("shard feed OK\n");
    return 0;
}
