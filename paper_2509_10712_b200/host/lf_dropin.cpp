// lf_dropin.cpp -- `loadflow_b200 dropin`: throughput of the DROP-IN path, i.e. the
// reference's own realtime Minato wiring (run_minato_pipeline, experiment.cpp:129-276:
// feeder -> WorkerPool of process_sample workers -> resume_slow -> build_batches ->
// run_consumer) over this repo's signature-compatible headers, with the transforms
// carrying device ops.  Each worker's process_sample submits its sample through the
// C ABI (lf_gpu.cpp process_on_device: lfg_submit + lfg_flush, then lfg_progress
// polls against t_out); with lfg_config.coalesce_us > 0 concurrent workers' samples
// share a launch group instead of one launch per sample.
//
//   loadflow_b200 dropin [--workers N] [--samples N] [--batch B] [--group G]
//                        [--coalesce-us U] [--t-out-us T] [--pool P] [--seed S] [--max-seconds M]
//
// Workload: C2 (obj_det RandomResizedCrop 224 + hflip + ToTensor + Normalize over
// HBM-resident u8 images of 256..512 px, Philox-synthesised on the device).
// Prints one JSON line: samples/s over the consumer's span (host clock), launches.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include <unistd.h>

#include "lfgpu.h"
#include "loadflow/balancer.hpp"
#include "loadflow/batcher.hpp"
#include "loadflow/runtime.hpp"
#include "loadflow/trainer.hpp"
#include "loadflow/worker_pool.hpp"

using namespace loadflow;

namespace {

void ck(int rc, const char* what) {
    if (rc != LFG_OK) throw std::runtime_error(std::string(what) + ": " + lfg_last_error());
}

}  // namespace

int cmd_dropin(int argc, char** argv) {
    int workers = 32, batch = 256, group = 64, pool_n = 256;
    int64_t samples = 20480, coalesce_us = 150, t_out_us = 0, max_seconds = 120;
    uint64_t seed = 1;
    for (int i = 2; i + 1 < argc; i += 2) {
        const std::string k = argv[i];
        const int64_t v = std::atoll(argv[i + 1]);
        if (k == "--workers") workers = static_cast<int>(v);
        else if (k == "--samples") samples = v;
        else if (k == "--batch") batch = static_cast<int>(v);
        else if (k == "--group") group = static_cast<int>(v);
        else if (k == "--coalesce-us") coalesce_us = v;
        else if (k == "--t-out-us") t_out_us = v;
        else if (k == "--pool") pool_n = static_cast<int>(v);
        else if (k == "--seed") seed = static_cast<uint64_t>(v);
        else if (k == "--max-seconds") max_seconds = v;
        else throw std::invalid_argument("dropin: unknown option " + k);
    }
    if (workers < 1 || samples < 1 || batch < 1 || group < 1 || pool_n < 1)
        throw std::invalid_argument("dropin: sizes must be positive");

    // a failed actor leaves the others waiting on its queues (as in the reference's
    // realtime wiring): bound the whole run instead of hanging
    if (max_seconds > 0) alarm(static_cast<unsigned>(max_seconds));
    lfg_config cfg;
    lfg_config_default(&cfg);
    cfg.batch_size = batch;
    cfg.n_workers = workers;
    cfg.max_group = group;
    cfg.max_slot_buffers = 24;
    cfg.coalesce_us = static_cast<int32_t>(coalesce_us);
    cfg.seed = seed;
    lfg_ctx* ctx = nullptr;
    ck(lfg_open(&cfg, &ctx), "lfg_open");
    const int shard = gpu::bind_shard(ctx);
    TransformChain chain = gpu::obj_det_chain(224);
    gpu::prepare_chain(chain, shard);

    // HBM-resident image pool (bench.py's C2 shapes: 256..512 px per side)
    std::mt19937_64 rs(seed);
    std::vector<void*> imgs(static_cast<size_t>(pool_n));
    std::vector<std::pair<int64_t, int64_t>> hw(static_cast<size_t>(pool_n));
    for (int i = 0; i < pool_n; ++i) {
        const int64_t H = 256 + static_cast<int64_t>(rs() % 257), W = 256 + static_cast<int64_t>(rs() % 257);
        hw[i] = {H, W};
        ck(lfg_device_alloc(ctx, static_cast<size_t>(H * W * 3), &imgs[i]), "device_alloc");
        ck(lfg_synth_image(ctx, seed, static_cast<uint64_t>(i), H, W, imgs[i], 1), "synth_image");
    }
    ck(lfg_synchronize(ctx), "synchronize");

    auto rt = make_realtime_runtime_ticks(1000);   // microsecond clock
    BoundedQueue<Sample> input(*rt, 4 * static_cast<size_t>(workers), QueueRole::input);
    std::vector<std::unique_ptr<SampleQueue>> fast, slow;
    std::vector<std::unique_ptr<TempQueue>> temp;
    std::vector<SampleQueue*> fp, sp;
    for (int i = 0; i < workers; ++i) {
        fast.push_back(std::make_unique<SampleQueue>(*rt, 4 * static_cast<size_t>(batch), QueueRole::fast));
        slow.push_back(std::make_unique<SampleQueue>(*rt, 4 * static_cast<size_t>(batch), QueueRole::slow));
        temp.push_back(std::make_unique<TempQueue>(*rt, 4 * static_cast<size_t>(batch), QueueRole::temp));
        fp.push_back(fast.back().get());
        sp.push_back(slow.back().get());
    }
    BatchQueue batch_q(*rt, 8, QueueRole::batch);
    const DurationMs t_out = t_out_us > 0 ? t_out_us : kNoTimeout;
    std::atomic<int64_t> n_fast{0}, n_slow{0};

    WorkerPool wp(*rt, PoolConfig{workers, workers}, input,
                  [&](int slot, Sample&& s) {
                      Rng rng(s.id);
                      RouteResult r = process_sample(std::move(s), t_out, *fast[slot], *temp[slot], *rt, rng);
                      (r.route == Route::fast ? n_fast : n_slow)++;
                  },
                  [&](int slot) {
                      fast[slot]->close();
                      temp[slot]->close();
                  });
    for (int i = 0; i < workers; ++i)
        rt->spawn("resume", [&, i] {
            Rng rng(static_cast<uint64_t>(i));
            resume_slow(*temp[i], *slow[i], *rt, rng);
            slow[i]->close();
        });
    rt->spawn("feeder", [&] {
        for (int64_t i = 0; i < samples; ++i) {
            Sample s;
            s.id = static_cast<uint64_t>(i);
            s.chain = &chain;
            const auto& d = hw[static_cast<size_t>(i % pool_n)];
            s.bytes_in = s.size_bytes = double(d.first * d.second * 3);
            s.bytes_out = 3.0 * 224 * 224 * 4;
            s.device.shard = shard;
            s.device.desc.src_kind = LFG_SRC_DEVICE;
            s.device.desc.ndim = 3;
            s.device.desc.dims[0] = d.first;
            s.device.desc.dims[1] = d.second;
            s.device.desc.dims[2] = 3;
            s.device.desc.data = imgs[static_cast<size_t>(i % pool_n)];
            input.put(std::move(s));
        }
        input.close();
    });
    rt->spawn("batcher", [&] { build_batches(fp, sp, batch_q, BatcherConfig{static_cast<size_t>(batch), 10}, *rt); });
    ConsumerStats st;
    rt->spawn("consumer", [&] {
        ConsumerConfig cc;
        cc.compute_per_batch = 0;
        cc.poll_sleep = 20;
        st = run_consumer(cc, batch_q, *rt);
    });
    lfg_counters c0;
    ck(lfg_get_counters(ctx, &c0), "counters");
    const auto w0 = std::chrono::steady_clock::now();
    wp.start();
    rt->run();
    const double wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    lfg_counters c1;
    ck(lfg_get_counters(ctx, &c1), "counters");

    const std::set<uint64_t> got(st.consumed_ids.begin(), st.consumed_ids.end());
    const bool exactly_once = got.size() == static_cast<size_t>(samples) &&
                              st.consumed_ids.size() == static_cast<size_t>(samples);
    const double launches = static_cast<double>(c1.launches - c0.launches);
    std::printf("{\"path\": \"drop-in C++ (run_minato_pipeline wiring, process_sample workers)\", "
                "\"value\": %.1f, \"unit\": \"samples/s\", \"samples\": %lld, \"wall_s\": %.4f, "
                "\"workers\": %d, \"batch\": %d, \"max_group\": %d, \"coalesce_us\": %lld, "
                "\"launches\": %.0f, \"samples_per_launch\": %.2f, \"fast\": %lld, \"slow\": %lld, "
                "\"batches\": %lld, \"inplace_batches\": %lld, \"exactly_once\": %s}\n",
                static_cast<double>(samples) / wall_s, static_cast<long long>(samples), wall_s, workers, batch,
                group, static_cast<long long>(coalesce_us), launches,
                launches > 0 ? static_cast<double>(samples) / launches : 0.0,
                static_cast<long long>(n_fast.load()), static_cast<long long>(n_slow.load()),
                static_cast<long long>(st.batches), static_cast<long long>(c1.inplace_batches - c0.inplace_batches),
                exactly_once ? "true" : "false");
    gpu::unbind_all();
    for (void* p : imgs) lfg_device_free(ctx, p);
    lfg_close(ctx);
    return exactly_once ? 0 : 3;
}
