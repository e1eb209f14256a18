// ref_harness.cpp -- the REFERENCE CPU loader timed on host cores (bench.py
// --impl reference and the cpu_baseline leg).  TEST/BENCH INFRASTRUCTURE.
//
// Links the reference library built from /root/reference/proj/src (ref.mk)
// and wires its realtime Minato pipeline the way run_minato_pipeline does
// (proj/src/experiment.cpp:129-276): feeder -> input queue -> WorkerPool slots
// running process_sample (real-function mode, balancer.cpp:42-77) -> per-slot
// fast/temp queues -> resume_slow actors -> slow queues -> build_batches ->
// run_consumer, with the Profiler's p75 timeout.  run_experiment itself only
// drives synthetic cost chains (workloads.cpp:14-20), so the wiring is
// restated here around real Transform::apply closures.
//
// The closures are the CPU oracle's transform arithmetic (lf_oracle.h) over the
// reference's fp64 Payload, one closure per reference transform name.
// Payload layout: [id, dims..., data...] (the header carries the sample id so
// per-sample parameters can be drawn: the reference apply() receives no id).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <mutex>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "lf_oracle.h"
#include "loadflow/balancer.hpp"
#include "loadflow/baselines.hpp"
#include "loadflow/batcher.hpp"
#include "loadflow/profiler.hpp"
#include "loadflow/runtime.hpp"
#include "loadflow/trainer.hpp"
#include "loadflow/worker_pool.hpp"

using namespace loadflow;

namespace {

constexpr uint64_t kSeed = 1;
constexpr int kHdr2d = 3;   // id, H, W
constexpr int kHdr3d = 4;   // id, D, H, W

// ---------------------------------------------------------------- obj_det chain
lfo_cfg2d g_c2;

Payload resize_step(Payload p) {   // Resize = RandomResizedCrop (bilinear) to 0..255 CHW
    const uint64_t id = (uint64_t)p[0];
    const int64_t H = (int64_t)p[1], W = (int64_t)p[2];
    lfo_params2d pr;
    lfo_draw2d(&g_c2, kSeed, id, H, W, &pr);
    const int64_t oh = g_c2.out_h, ow = g_c2.out_w;
    Payload out(kHdr2d + 3 * oh * ow);
    out[0] = p[0];
    out[1] = (double)oh;
    out[2] = (double)ow;
    const double* src = p.data() + kHdr2d;
    auto idx = [](int64_t d, int64_t in, int64_t o, int64_t& i0, int64_t& i1, double& l1) {
        double s = ((double)d + 0.5) * ((double)in / (double)o) - 0.5;
        if (s < 0) s = 0;
        int64_t a = (int64_t)std::floor(s);
        if (a > in - 1) a = in - 1;
        i0 = a;
        i1 = a < in - 1 ? a + 1 : a;
        l1 = s - (double)a;
    };
    for (int64_t y = 0; y < oh; ++y) {
        int64_t y0, y1;
        double ly;
        idx(y, pr.h, oh, y0, y1, ly);
        for (int64_t x = 0; x < ow; ++x) {
            int64_t x0, x1;
            double lx;
            idx(x, pr.w, ow, x0, x1, lx);
            for (int c = 0; c < 3; ++c) {
                auto px = [&](int64_t yy, int64_t xx) {
                    return src[((pr.top + yy) * W + pr.left + xx) * 3 + c];
                };
                const double v = (1 - ly) * ((1 - lx) * px(y0, x0) + lx * px(y0, x1)) +
                                 ly * ((1 - lx) * px(y1, x0) + lx * px(y1, x1));
                out[kHdr2d + (c * oh + y) * ow + x] = v;
            }
        }
    }
    return out;
}

Payload hflip_step(Payload p) {
    lfo_params2d pr;
    // the flip bit is the draw after the crop box on the same per-sample stream;
    // the crop box is re-drawn from the original image size kept below
    lfo_draw2d(&g_c2, kSeed, (uint64_t)p[0], (int64_t)p.back(), (int64_t)p[p.size() - 2], &pr);
    p.resize(p.size() - 2);
    if (pr.flip) {
        const int64_t oh = (int64_t)p[1], ow = (int64_t)p[2];
        for (int c = 0; c < 3; ++c)
            for (int64_t y = 0; y < oh; ++y) {
                double* row = p.data() + kHdr2d + (c * oh + y) * ow;
                std::reverse(row, row + ow);
            }
    }
    return p;
}

Payload to_tensor_step(Payload p) {
    for (size_t i = kHdr2d; i < p.size(); ++i) p[i] /= 255.0;
    return p;
}

Payload normalize_step(Payload p) {
    const int64_t plane = (int64_t)p[1] * (int64_t)p[2];
    for (int c = 0; c < 3; ++c)
        for (int64_t i = 0; i < plane; ++i) {
            double& v = p[kHdr2d + c * plane + i];
            v = (v - g_c2.mean[c]) / g_c2.std[c];
        }
    return p;
}

// ---------------------------------------------------------------- img_seg chain
lfo_cfg3d g_c3;

lfo_params3d params3d(const Payload& p, const int64_t dims[3]) {
    lfo_params3d pr;
    lfo_draw3d(&g_c3, kSeed, (uint64_t)p[0], dims, &pr);
    return pr;
}

// Payload after RandomCrop: [id, cd, ch, cw, D, H, W (original dims), img..., lbl...]
Payload crop_step(Payload p) {
    const int64_t dims[3] = {(int64_t)p[1], (int64_t)p[2], (int64_t)p[3]};
    lfo_params3d pr = params3d(p, dims);
    if (g_c3.has_fg && pr.fg) {   // foreground oversampling: scan the label volume
        const int64_t nv = dims[0] * dims[1] * dims[2];
        std::vector<uint8_t> lab((size_t)nv);
        for (int64_t i = 0; i < nv; ++i) lab[(size_t)i] = (uint8_t)p[kHdr3d + nv + i];
        int64_t off[3];
        if (lfo_fg_offsets(&pr, lab.data(), dims, off) == 0)
            for (int a = 0; a < 3; ++a) pr.off[a] = off[a];
    }
    const int64_t cd = g_c3.crop[0], ch = g_c3.crop[1], cw = g_c3.crop[2];
    const int64_t vox = cd * ch * cw, n = dims[0] * dims[1] * dims[2];
    Payload out(7 + 2 * vox, 0.0);
    out[0] = p[0];
    out[1] = cd; out[2] = ch; out[3] = cw;
    out[4] = dims[0]; out[5] = dims[1]; out[6] = dims[2];
    const double* img = p.data() + kHdr3d;
    const double* lbl = img + n;
    for (int64_t z = 0; z < cd; ++z)
        for (int64_t y = 0; y < ch; ++y)
            for (int64_t x = 0; x < cw; ++x) {
                const int64_t sz = pr.off[0] + z, sy = pr.off[1] + y, sx = pr.off[2] + x;
                if (sz >= dims[0] || sy >= dims[1] || sx >= dims[2]) continue;
                const int64_t si = (sz * dims[1] + sy) * dims[2] + sx, o = (z * ch + y) * cw + x;
                out[7 + o] = img[si];
                out[7 + vox + o] = lbl[si];
            }
    return out;
}

Payload flip_step(Payload p) {
    const int64_t dims[3] = {(int64_t)p[4], (int64_t)p[5], (int64_t)p[6]};
    const lfo_params3d pr = params3d(p, dims);
    const int64_t cd = (int64_t)p[1], ch = (int64_t)p[2], cw = (int64_t)p[3], vox = cd * ch * cw;
    Payload out(p.size());
    std::copy(p.begin(), p.begin() + 7, out.begin());
    for (int plane = 0; plane < 2; ++plane)
        for (int64_t z = 0; z < cd; ++z)
            for (int64_t y = 0; y < ch; ++y)
                for (int64_t x = 0; x < cw; ++x) {
                    const int64_t sz = pr.flip[0] ? cd - 1 - z : z, sy = pr.flip[1] ? ch - 1 - y : y,
                                  sx = pr.flip[2] ? cw - 1 - x : x;
                    out[7 + plane * vox + (z * ch + y) * cw + x] =
                        p[7 + plane * vox + (sz * ch + sy) * cw + sx];
                }
    return out;
}

Payload brightness_step(Payload p) {
    const int64_t dims[3] = {(int64_t)p[4], (int64_t)p[5], (int64_t)p[6]};
    const lfo_params3d pr = params3d(p, dims);
    const int64_t vox = (int64_t)(p[1] * p[2] * p[3]);
    for (int64_t i = 0; i < vox; ++i) p[7 + i] *= pr.scale;
    return p;
}

Payload noise_step(Payload p) {
    const int64_t dims[3] = {(int64_t)p[4], (int64_t)p[5], (int64_t)p[6]};
    const lfo_params3d pr = params3d(p, dims);
    if (pr.sigma == 0.0) return p;
    const int64_t vox = (int64_t)(p[1] * p[2] * p[3]);
    for (int64_t g = 0; g * 4 < vox; ++g) {
        double z[4];
        lfo_normals4((uint64_t)g, pr.key[0], pr.key[1], z);
        for (int j = 0; j < 4 && g * 4 + j < vox; ++j) p[7 + g * 4 + j] += pr.sigma * z[j];
    }
    return p;
}

Payload cast_step(Payload p) {
    const int64_t vox = (int64_t)(p[1] * p[2] * p[3]);
    for (int64_t i = 0; i < vox; ++i) p[7 + i] = (double)(float)p[7 + i];
    for (int64_t i = 0; i < vox; ++i) p[7 + vox + i] = (double)(uint8_t)p[7 + vox + i];
    return p;
}

Transform real(const char* name, double factor, std::function<Payload(Payload)> f) {
    Transform t;
    t.name = name;
    t.size_factor = factor;
    t.apply = std::move(f);
    return t;
}

int arg_int(int argc, char** argv, const char* key, int dflt) {
    for (int i = 1; i + 1 < argc; ++i)
        if (!std::strcmp(argv[i], key)) return std::atoi(argv[i + 1]);
    return dflt;
}
std::string arg_str(int argc, char** argv, const char* key, const char* dflt) {
    for (int i = 1; i + 1 < argc; ++i)
        if (!std::strcmp(argv[i], key)) return argv[i + 1];
    return dflt;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string wl = arg_str(argc, argv, "--workload", "rrc");
    const int steps = arg_int(argc, argv, "--steps", 10);
    const int warmup = arg_int(argc, argv, "--warmup", 2);
    const int cores = arg_int(argc, argv, "--workers", (int)std::max(1u, std::thread::hardware_concurrency()));
    const int max_s = arg_int(argc, argv, "--max-seconds", 150);
    const int feeders = std::max(1, arg_int(argc, argv, "--feeders", 4));
    // C5 sweep knobs: a heavy-tailed fraction of samples gets an
    // extra synthetic cost (a leading "SampleCost" transform that sleeps), the
    // consumer computes for trainer_ms per batch (trainer.hpp:15), and the
    // timeout is the Profiler's p75/p90 policy (pct = -1, default) or a fixed
    // nearest-rank percentile of the window (pct > 0) or none (pct = 0).
    const double heavy_frac = std::atof(arg_str(argc, argv, "--heavy-frac", "0").c_str());
    const int heavy_ms = arg_int(argc, argv, "--heavy-ms", 470);   // img_seg median cost, workloads.cpp:84-95
    const int trainer_ms = arg_int(argc, argv, "--trainer-ms", 0);
    const int pct = arg_int(argc, argv, "--pct", -1);
    const int prof_warmup_ms = arg_int(argc, argv, "--profiler-warmup-ms", 2000);
    // --loader sync: the reference's synchronous PyTorch-DataLoader-like loader
    // (start_sync_loader, baselines.cpp:12-151) instead of the Minato pipeline
    const bool sync = arg_str(argc, argv, "--loader", "minato") == "sync";
    const double p_fg = std::atof(arg_str(argc, argv, "--fg", "0").c_str());   // RandomCrop oversampling
    lfo_cfg2d_default(&g_c2);
    lfo_cfg3d_default(&g_c3);
    g_c3.has_fg = p_fg > 0;
    g_c3.p_fg = p_fg;
    const bool rrc = wl == "rrc";
    const int B = rrc ? 256 : 2;
    const int64_t n = (int64_t)(steps + warmup) * B;

    std::vector<Transform> heavy_ops;
    if (heavy_frac > 0) {
        heavy_ops.push_back(real("SampleCost", 1.0, [heavy_frac, heavy_ms](Payload p) {
            // heavy iff a per-id uniform < heavy_frac (the id rides in the payload header)
            std::mt19937_64 g(0x5eedULL ^ (0x9e3779b97f4a7c15ULL * ((uint64_t)p[0] + 1)));
            if ((double)(g() >> 11) * 0x1.0p-53 < heavy_frac)
                std::this_thread::sleep_for(std::chrono::milliseconds(heavy_ms));
            return p;
        }));
    }
    TransformChain chain(rrc ? std::vector<Transform>{real("Resize", 1.2, resize_step),
                                                      real("RandomHorizontalFlip", 1.0, hflip_step),
                                                      real("ToTensor", 8.0, to_tensor_step),
                                                      real("Normalize", 1.0, normalize_step)}
                             : std::vector<Transform>{real("RandomCrop", 0.0735, crop_step),
                                                      real("RandomFlip", 1.0, flip_step),
                                                      real("RandomBrightness", 1.0, brightness_step),
                                                      real("GaussianNoise", 1.0, noise_step),
                                                      real("Cast", 1.0, cast_step)});
    if (!heavy_ops.empty()) {
        std::vector<Transform> ts = heavy_ops;
        for (const auto& t : chain.transforms()) ts.push_back(t);
        chain = TransformChain(std::move(ts));
    }
    if (rrc) {
        // Resize needs the original (H, W) again at RandomHorizontalFlip to
        // re-derive the per-sample stream: carry it at the payload's tail
        chain.transforms()[heavy_ops.size()].apply = [](Payload p) {
            const double H = p[1], W = p[2];
            Payload out = resize_step(std::move(p));
            out.push_back(W);
            out.push_back(H);
            return out;
        };
    }

    // synthetic raw inputs: a small pool of distinct images / volumes
    std::mt19937_64 gen(7);
    const int pool = rrc ? 32 : 2;
    std::vector<std::vector<uint8_t>> images;
    std::vector<std::pair<int, int>> hw;
    std::vector<std::vector<float>> vols;
    std::vector<std::vector<uint8_t>> lbls;
    const int64_t D = 128, H3 = 384, W3 = 384;
    for (int i = 0; i < pool; ++i) {
        if (rrc) {
            const int h = 256 + (int)(gen() % 257), w = 256 + (int)(gen() % 257);
            std::vector<uint8_t> im((size_t)h * w * 3);
            for (auto& b : im) b = (uint8_t)gen();
            images.push_back(std::move(im));
            hw.emplace_back(h, w);
        } else {
            std::normal_distribution<float> nd;
            std::vector<float> v((size_t)(D * H3 * W3));
            std::vector<uint8_t> l(v.size());
            for (size_t k = 0; k < v.size(); ++k) {
                v[k] = nd(gen);
                l[k] = (uint8_t)(gen() % 3);
            }
            vols.push_back(std::move(v));
            lbls.push_back(std::move(l));
        }
    }

    auto rt = make_realtime_runtime();
    const std::size_t cap = 100;   // PAPER.md:831 queue capacity
    BoundedQueue<Sample> input(*rt, cap, QueueRole::input);
    std::vector<std::unique_ptr<SampleQueue>> fast, slow;
    std::vector<std::unique_ptr<TempQueue>> temp;
    std::vector<SampleQueue*> fast_p, slow_p;
    for (int i = 0; i < cores; ++i) {
        fast.push_back(std::make_unique<SampleQueue>(*rt, cap, QueueRole::fast));
        slow.push_back(std::make_unique<SampleQueue>(*rt, cap, QueueRole::slow));
        temp.push_back(std::make_unique<TempQueue>(*rt, cap, QueueRole::temp));
        fast_p.push_back(fast.back().get());
        slow_p.push_back(slow.back().get());
    }
    BatchQueue batch_q(*rt, cap, QueueRole::batch);
    TimeoutPolicy policy;
    ProfilerConfig pc;
    pc.warmup = prof_warmup_ms;   // ms; shortened from the 10 s default so the bounded run reaches p75
    Profiler prof(*rt, pc);
    std::vector<Rng> rngs;
    for (int i = 0; i < cores; ++i) rngs.emplace_back(kSeed ^ (0x9e3779b97f4a7c15ULL * (i + 1)));
    std::atomic<int64_t> n_slow{0};
    // per-sample totals for the fixed-percentile policy (--pct > 0)
    std::mutex win_mu;
    std::deque<DurationMs> win;
    auto record_total = [&](const std::vector<DurationMs>& c) {
        DurationMs t = 0;
        for (auto x : c) t += x;
        std::lock_guard<std::mutex> lk(win_mu);
        win.push_back(t);
        if (win.size() > pc.window) win.pop_front();
    };
    std::atomic<bool> give_up{false};
    const auto wall0 = std::chrono::steady_clock::now();

    WorkerPool pool_w(
        *rt, PoolConfig{cores, cores}, input,
        [&](int slot, Sample&& s) {
            const uint64_t id = s.id;
            const double sz = s.bytes_in;
            RouteResult r = process_sample(std::move(s), policy.timeout(), *fast[slot], *temp[slot],
                                           *rt, rngs[slot]);
            if (r.route == Route::fast) {
                record_total(r.exec_costs);
                prof.record(SampleStats::from_costs(id, sz, std::move(r.exec_costs), false));
            } else {
                n_slow++;
            }
        },
        [&](int slot) {
            fast[slot]->close();
            temp[slot]->close();
        });
    // The pool's inputs as fp64 payloads [id, dims..., data...], built once before the
    // clock starts; a fed sample copies its template (the feeder loads, the workers
    // transform -- experiment.cpp:221-228), so the feeders never bound the loader.
    std::vector<std::vector<double>> tmpl(static_cast<size_t>(pool));
    for (int q = 0; q < pool; ++q) {
        auto& t = tmpl[static_cast<size_t>(q)];
        if (rrc) {
            const auto& im = images[q];
            const auto [h, w] = hw[q];
            t.resize(kHdr2d + im.size());
            t[1] = h;
            t[2] = w;
            for (size_t k = 0; k < im.size(); ++k) t[kHdr2d + k] = im[k];
        } else {
            const auto& v = vols[q];
            const auto& l = lbls[q];
            t.resize(kHdr3d + 2 * v.size());
            t[1] = D;
            t[2] = H3;
            t[3] = W3;
            for (size_t k = 0; k < v.size(); ++k) t[kHdr3d + k] = v[k];
            for (size_t k = 0; k < l.size(); ++k) t[kHdr3d + v.size() + k] = l[k];
        }
    }
    auto make_payload_sample = [&](int64_t i) {
        Sample s;
        s.id = (uint64_t)i;
        s.chain = &chain;
        s.payload = tmpl[static_cast<size_t>(i % pool)];
        s.payload[0] = (double)i;
        s.bytes_in = s.size_bytes = (double)s.payload.size() * 8;
        s.t_enqueue = rt->now();
        return s;
    };
    // F feeder threads claim ids in order (one copy of a multi-MB payload each), the
    // last one to finish closes the input
    std::atomic<int64_t> next_id{0};
    std::atomic<int> feeders_left{feeders};
    if (!sync) {
    for (int i = 0; i < cores; ++i) {
        rt->spawn("resume." + std::to_string(i), [&, i] {
            Rng r(kSeed ^ (0xc2b2ae3d27d4eb4fULL * (i + 1)));
            resume_slow(*temp[i], *slow[i], *rt, r,
                        [&](const Sample& s, const std::vector<DurationMs>& c, DurationMs) {
                            record_total(c);
                            prof.record(SampleStats::from_costs(s.id, s.bytes_in, c, true));
                        });
            slow[i]->close();
        });
    }
    for (int f = 0; f < feeders; ++f)
        rt->spawn("feeder." + std::to_string(f), [&] {
            for (;;) {
                const int64_t i = next_id.fetch_add(1);
                if (i >= n) break;
                const auto el = std::chrono::steady_clock::now() - wall0;
                if (std::chrono::duration_cast<std::chrono::seconds>(el).count() > max_s) {
                    give_up = true;
                    break;
                }
                input.put(make_payload_sample(i));
            }
            if (feeders_left.fetch_sub(1) == 1) input.close();
        });
    }
    if (sync) {
        // all samples up front (start_sync_loader takes the stream by value)
        std::vector<Sample> all;
        for (int64_t i = 0; i < n; ++i) all.push_back(make_payload_sample(i));
        start_sync_loader(*rt, std::move(all), SyncLoaderConfig{(size_t)B, cores, 2}, batch_q);
    } else {
        rt->spawn("batcher", [&] {
            build_batches(fast_p, slow_p, batch_q, BatcherConfig{(size_t)B, 10}, *rt);
        });
    }
    ConsumerStats cs;
    rt->spawn("consumer", [&] {
        ConsumerConfig cc;
        cc.compute_per_batch = trainer_ms;   // 0: drain as fast as batches arrive (loader throughput)
        cs = run_consumer(cc, batch_q, *rt);
    });
    if (sync) {
    } else if (pct < 0) {
        rt->spawn("profiler", [&] { profiler_loop(prof, policy, *rt, [&] { return pool_w.stopped(); }); });
    } else if (pct > 0) {   // fixed percentile: the reference's percentile() over the window
        rt->spawn("profiler", [&] {
            rt->sleep(pc.warmup);
            while (!pool_w.stopped()) {
                std::vector<DurationMs> v;
                {
                    std::lock_guard<std::mutex> lk(win_mu);
                    v.assign(win.begin(), win.end());
                }
                if (!v.empty()) policy.set(percentile(std::move(v), pct), TimeoutPolicy::Source::configured);
                rt->sleep(pc.update_interval);
            }
        });
    }
    if (!sync) pool_w.start();
    rt->run();

    // timed window: batches after the warm-up ones (compute_end in ms)
    const auto& ev = cs.events;
    double value = 0, timed = 0, span_ms = 0;
    if ((int)ev.size() > warmup + 1) {
        const TimeMs t0 = ev[warmup - 1 < 0 ? 0 : warmup - 1].compute_end;
        for (size_t k = (size_t)warmup; k < ev.size(); ++k) timed += (double)ev[k].n_samples;
        span_ms = (double)(ev.back().compute_end - t0);
        value = span_ms > 0 ? timed / (span_ms / 1000.0) : 0;
    }
    std::printf("{\"value\": %.3f, \"unit\": \"samples/s\", \"cores\": %d, \"kind\": \"reference\", "
                "\"idle_frac\": %.4f, \"final_t_out_ms\": %lld, "
                "\"samples\": %.0f, \"span_ms\": %.0f, \"slow\": %lld, \"truncated\": %s, "
                "\"sample\": \"reference libloadflow (proj/src, realtime Minato wiring) with oracle "
                "transforms over fp64 Payload: %s, %lld samples fed (payloads pre-built, %d feeder threads), "
                "batch %d, %d workers\"}\n",
                value, cores, cs.idle_fraction(), (long long)policy.timeout(), timed, span_ms,
                (long long)n_slow.load(), give_up ? "true" : "false",
                rrc ? "RRC224+flip+ToTensor+Normalize on u8 3x(256..512)^2"
                    : "crop128^3+flip+brightness+noise+cast on 128x384x384",
                (long long)cs.samples, feeders, B, cores);
    return 0;
}
