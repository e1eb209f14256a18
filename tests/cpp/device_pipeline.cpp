// device_pipeline.cpp -- the reference-shaped C++ API driving the GPU path.
//
// Wires the Minato topology of proj/src/experiment.cpp:129-276 with this
// repo's loadflow headers, but with gpu::img_seg_chain() (transforms carrying
// device ops) and Sample::device payloads: process_sample submits to the CUDA
// library and classifies against t_out on a microsecond realtime clock,
// resume_slow waits on completion events, build_batches seals device batches,
// run_consumer releases them.  Some samples get a long synthetic device cost
// (a spin op in front of the chain) so the timeout path is exercised.
// Then four more samples go through process_sample's fast path, are sealed on the
// device (gpu::seal_device_batch), read back and compared with the CPU oracle
// (oracle/lf_oracle.c: labels bit-exact, image within 1e-5 relative + 1e-6).
// Exit code 0 = exactly-once delivery, fast/slow split as expected, every
// batch device-sealed, delivered outputs equal to the oracle's.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <set>
#include <vector>

#include "loadflow/balancer.hpp"
#include "loadflow/batcher.hpp"
#include "loadflow/runtime.hpp"
#include "loadflow/trainer.hpp"
#include "loadflow/worker_pool.hpp"
#include "../../oracle/lf_oracle.h"   // the checker (test infrastructure)

using namespace loadflow;

#define EXPECT(c)                                                   \
    do {                                                            \
        if (!(c)) {                                                 \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                               \
        }                                                           \
    } while (0)

int main() {
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);   // before the first CUDA call
    lfg_config cfg;
    lfg_config_default(&cfg);
    cfg.batch_size = 4;
    cfg.n_workers = 8;
    cfg.max_slot_buffers = 16;
    lfg_ctx* ctx = nullptr;
    if (lfg_open(&cfg, &ctx) != LFG_OK) {
        std::fprintf(stderr, "lfg_open: %s\n", lfg_last_error());
        return 2;
    }
    const int shard = gpu::bind_shard(ctx);

    // chain: a per-sample synthetic cost (spin) then the fused img_seg transforms
    TransformChain base = gpu::img_seg_chain(32);
    std::vector<Transform> ts;
    Transform spin;
    spin.name = "SampleCost";
    spin.device.op.kind = LFG_OP_SPIN;
    ts.push_back(spin);
    for (const auto& t : base.transforms()) ts.push_back(t);
    TransformChain chain(ts);
    gpu::prepare_chain(chain, shard);

    const int64_t D = 40, H = 48, W = 64, n = 64;
    void *img = nullptr, *lbl = nullptr;
    lfg_device_alloc(ctx, D * H * W * 4, &img);
    lfg_device_alloc(ctx, D * H * W, &lbl);
    lfg_synth_volume(ctx, 1, 0, D, H, W, img, lbl, 1);

    auto rt = make_realtime_runtime_ticks(1000);   // microsecond clock
    const int workers = 4;
    BoundedQueue<Sample> input(*rt, 100, QueueRole::input);
    std::vector<std::unique_ptr<SampleQueue>> fast, slow;
    std::vector<std::unique_ptr<TempQueue>> temp;
    std::vector<SampleQueue*> fp, sp;
    for (int i = 0; i < workers; ++i) {
        fast.push_back(std::make_unique<SampleQueue>(*rt, 100, QueueRole::fast));
        slow.push_back(std::make_unique<SampleQueue>(*rt, 100, QueueRole::slow));
        temp.push_back(std::make_unique<TempQueue>(*rt, 100, QueueRole::temp));
        fp.push_back(fast.back().get());
        sp.push_back(slow.back().get());
    }
    BatchQueue batch_q(*rt, 100, QueueRole::batch);
    const DurationMs t_out = 20'000;   // 20 ms budget (microsecond ticks)
    std::set<uint64_t> heavy;
    for (int64_t i = 5; i < n; i += 9) heavy.insert(i);
    std::atomic<int> n_fast{0}, n_slow{0}, bad_index{0};

    WorkerPool pool(*rt, PoolConfig{workers, workers}, input,
                    [&](int slot, Sample&& s) {
                        Rng rng(s.id);
                        const uint64_t id = s.id;
                        RouteResult r = process_sample(std::move(s), t_out, *fast[slot], *temp[slot], *rt, rng);
                        if (r.route == Route::fast) n_fast++;
                        else {
                            if (!heavy.count(id))
                                std::printf("unexpected slow: id %llu fg %lld us index %zu\n",
                                            (unsigned long long)id, (long long)r.foreground_ms,
                                            r.timeout_index);
                            n_slow++;
                            if (r.timeout_index > 1) bad_index++;   // still in the spin or the kernel
                        }
                    },
                    [&](int slot) {
                        fast[slot]->close();
                        temp[slot]->close();
                    });
    for (int i = 0; i < workers; ++i)
        rt->spawn("resume", [&, i] {
            Rng rng(i);
            resume_slow(*temp[i], *slow[i], *rt, rng);
            slow[i]->close();
        });
    rt->spawn("feeder", [&] {
        for (int64_t i = 0; i < n; ++i) {
            Sample s;
            s.id = static_cast<uint64_t>(i);
            s.chain = &chain;
            s.bytes_in = s.size_bytes = double(D * H * W * 5);
            s.bytes_out = 32.0 * 32 * 32 * 5;
            s.device.shard = shard;
            s.device.desc.src_kind = LFG_SRC_DEVICE;
            s.device.desc.ndim = 3;
            s.device.desc.dims[0] = D;
            s.device.desc.dims[1] = H;
            s.device.desc.dims[2] = W;
            s.device.desc.data = img;
            s.device.desc.aux = lbl;
            s.device.desc.spin_us[0] = heavy.count(i) ? 80'000 : 100;
            input.put(std::move(s));
        }
        input.close();
    });
    std::vector<int64_t> device_batches;
    rt->spawn("batcher", [&] { build_batches(fp, sp, batch_q, BatcherConfig{4, 1}, *rt); });
    ConsumerStats st;
    rt->spawn("consumer", [&] {
        ConsumerConfig cc;
        cc.compute_per_batch = 0;
        cc.poll_sleep = 50;
        st = run_consumer(cc, batch_q, *rt);
    });
    pool.start();
    rt->run();

    std::set<uint64_t> got(st.consumed_ids.begin(), st.consumed_ids.end());
    std::printf("consumed %zu (unique %zu) fast %d slow %d batches %lld\n", st.consumed_ids.size(),
                got.size(), n_fast.load(), n_slow.load(), (long long)st.batches);
    EXPECT(st.consumed_ids.size() == static_cast<size_t>(n));
    EXPECT(got.size() == static_cast<size_t>(n));
    EXPECT(n_slow.load() == static_cast<int>(heavy.size()));
    EXPECT(n_fast.load() == n - static_cast<int>(heavy.size()));
    EXPECT(bad_index.load() == 0);
    lfg_counters c;
    lfg_get_counters(ctx, &c);
    EXPECT(c.batches == st.batches);          // every batch was sealed on the device
    std::printf("device batches %lld (in place %lld, gathered %lld)\n", (long long)c.batches,
                (long long)c.inplace_batches, (long long)c.gathered_batches);

    // ---- delivered outputs against the oracle
    {
        const int64_t vox_in = D * H * W, vox = 32 * 32 * 32;
        std::vector<float> himg(static_cast<size_t>(vox_in));
        std::vector<uint8_t> hlbl(static_cast<size_t>(vox_in));
        EXPECT(lfg_memcpy_d2h(ctx, himg.data(), img, vox_in * 4) == LFG_OK);
        EXPECT(lfg_memcpy_d2h(ctx, hlbl.data(), lbl, vox_in) == LFG_OK);
        SampleQueue fq(*rt, 16, QueueRole::fast);
        TempQueue tq(*rt, 16, QueueRole::temp);
        Batch b;
        for (uint64_t id = 1000; id < 1004; ++id) {
            Sample s;
            s.id = id;
            s.chain = &chain;
            s.bytes_in = s.size_bytes = double(vox_in * 5);
            s.bytes_out = double(vox * 5);
            s.device.shard = shard;
            s.device.desc.src_kind = LFG_SRC_DEVICE;
            s.device.desc.ndim = 3;
            s.device.desc.dims[0] = D;
            s.device.desc.dims[1] = H;
            s.device.desc.dims[2] = W;
            s.device.desc.data = img;
            s.device.desc.aux = lbl;
            s.device.desc.spin_us[0] = 10;
            Rng rng(id);
            RouteResult r = process_sample(std::move(s), kNoTimeout, fq, tq, *rt, rng);
            EXPECT(r.route == Route::fast);
            auto got = fq.try_get();
            EXPECT(got.has_value());
            b.samples.push_back(std::move(*got));
        }
        gpu::seal_device_batch(b);
        EXPECT(b.device_batch >= 0);
        void* dp = nullptr;
        int64_t bytes = 0;
        int nb = 0, inplace = 0;
        uint64_t ids[4] = {};
        EXPECT(lfg_batch_info(ctx, b.device_batch, &dp, &bytes, &nb, ids, &inplace) == LFG_OK);
        EXPECT(nb == 4 && bytes >= 4 * vox * 5);
        std::vector<uint8_t> host(static_cast<size_t>(bytes));
        EXPECT(lfg_batch_copy_to_host(ctx, b.device_batch, host.data(), static_cast<size_t>(bytes)) == LFG_OK);
        const int64_t dims[3] = {D, H, W};
        double worst = 0.0;
        for (int k = 0; k < nb; ++k) {   // planar batch: [f32 image x 4][u8 label x 4]
            lfo_cfg3d oc;
            lfo_cfg3d_default(&oc);
            oc.crop[0] = oc.crop[1] = oc.crop[2] = 32;
            lfo_params3d op;
            lfo_draw3d(&oc, cfg.seed, ids[k], dims, &op);
            std::vector<double> e_img(static_cast<size_t>(vox));
            std::vector<uint8_t> e_lbl(static_cast<size_t>(vox));
            lfo_apply3d(&oc, &op, himg.data(), hlbl.data(), dims, e_img.data(), e_lbl.data());
            const float* g_img = reinterpret_cast<const float*>(host.data()) + k * vox;
            const uint8_t* g_lbl = host.data() + 4 * vox * 4 + k * vox;
            EXPECT(std::memcmp(g_lbl, e_lbl.data(), static_cast<size_t>(vox)) == 0);
            for (int64_t v = 0; v < vox; ++v) {
                const double err = std::fabs(g_img[v] - e_img[v]);
                worst = std::max(worst, err / (1e-5 * std::fabs(e_img[v]) + 1e-6));
            }
        }
        std::printf("delivered outputs vs oracle: worst err/bound %.3f\n", worst);
        EXPECT(worst <= 1.0);
        EXPECT(lfg_batch_release(ctx, b.device_batch, nullptr) == LFG_OK);
    }
    gpu::unbind_all();
    lfg_device_free(ctx, img);
    lfg_device_free(ctx, lbl);
    lfg_close(ctx);
    std::printf("device pipeline OK\n");
    return 0;
}
