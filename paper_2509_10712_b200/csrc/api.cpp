// api.cpp -- extern "C" entry points (include/lfgpu.h).  Every call takes the
// context lock, converts engine exceptions into LFG_ERR_* codes and records a
// thread-local message for lfg_last_error().
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"

namespace lfg {
int run_shard(Context& ctx, Chain* chain, const lfg_sample_desc* samples, int64_t n,
              const lfg_run_config& rc, lfg_run_report& rep, uint64_t* consumed_ids,
              int32_t* batch_sizes, int32_t* sample_class, const lfg_source* src = nullptr,
              const ShardStream* ss = nullptr);
}

using namespace lfg;

struct lfg_ctx {
    Context* impl;
};
struct lfg_chain {
    Chain* impl;
    lfg_ctx* ctx;
};
// A streaming shard run: the Algorithm-1 loop on its own thread, sealed batches
// queued for the consumer (the reference's BatchQueue between build_batches and
// run_consumer, batcher.cpp:50-58 / trainer.cpp:7-18).
struct lfg_shard {
    lfg_ctx* ctx = nullptr;
    std::vector<lfg_sample_desc> samples;
    lfg_run_config cfg{};
    std::thread th;
    std::mutex qm;
    std::condition_variable cv;
    std::deque<std::pair<int64_t, int>> q;   // (batch, samples), delivery order
    bool ended = false;
    int rc = LFG_OK;
    std::string err;
    lfg_run_report rep{};
    std::vector<uint64_t> ids;
    std::vector<int32_t> sizes, cls;
    // consumer-side ConsumerStats (trainer.hpp:30-47): host time blocked in next_batch
    std::chrono::steady_clock::time_point t_first, t_last;
    bool started = false;
    double wait_us = 0;
    int64_t taken = 0;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LFG_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return LFG_ERR_NOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LFG_ERR_STATE;
    }
}

void refuse_while_streaming(const Context& c) {
    if (c.streaming) fail(LFG_ERR_STATE, "a streaming shard run owns this context (lfg_shard_finish first)");
}

Context& C(lfg_ctx* ctx) {
    if (ctx == nullptr || ctx->impl == nullptr) fail(LFG_ERR_INVALID, "null context");
    cuda_check(cudaSetDevice(ctx->impl->cfg.device), "cudaSetDevice");
    return *ctx->impl;
}

// ---- host-side synthetic generators (same Philox streams as k_misc.cu) ----
inline void h_philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = uint64_t(0xD2511F53u) * c[0];
        const uint64_t p1 = uint64_t(0xCD9E8D57u) * c[2];
        const uint32_t n0 = uint32_t(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n2 = uint32_t(p0 >> 32) ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = uint32_t(p1);
        c[2] = n2;
        c[3] = uint32_t(p0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
inline void h_synth_rand(uint64_t seed, uint64_t id, uint64_t ctr, uint32_t stream, uint32_t o[4]) {
    const uint64_t k = seed * 0x9E3779B97F4A7C15ull ^ (id + 1) * 0xC2B2AE3D27D4EB4Full;
    o[0] = uint32_t(ctr);
    o[1] = uint32_t(ctr >> 32);
    o[2] = stream;
    o[3] = 0x5EEDu;
    h_philox(o, uint32_t(k), uint32_t(k >> 32));
}
inline void h_bm(uint32_t a, uint32_t b, float& z0, float& z1) {
    const double u1 = (double(a) + 0.5) * 0x1.0p-32, u2 = (double(b) + 0.5) * 0x1.0p-32;
    const double r = std::sqrt(-2.0 * std::log(u1));
    z0 = float(r * std::cos(2 * M_PI * u2));
    z1 = float(r * std::sin(2 * M_PI * u2));
}

template <typename F>
void parallel_for(int64_t n, F&& f) {
    const int nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int64_t i = t; i < n; i += nt) f(i);
        });
    for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

const char* lfg_last_error(void) { return g_last_error.c_str(); }
int lfg_abi_version(void) { return LFG_ABI_VERSION; }

int lfg_device_count(int* n) {
    return guarded([&] {
        if (!n) fail(LFG_ERR_INVALID, "null out");
        cudaError_t e = cudaGetDeviceCount(n);
        if (e != cudaSuccess) {
            *n = 0;
            cudaGetLastError();
        }
    });
}

void lfg_config_default(lfg_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->device = 0;
    cfg->n_workers = 12;          // PAPER.md:716, 829 (12 workers per GPU)
    cfg->max_group = 1;
    cfg->batch_size = 24;         // experiment.hpp:28 default
    cfg->max_slot_buffers = 8;
    cfg->seed = 1;                // workloads.hpp:31 default seed
}

int lfg_open(const lfg_config* cfg, lfg_ctx** out) {
    return guarded([&] {
        if (!cfg || !out) fail(LFG_ERR_INVALID, "null argument");
        auto* c = new lfg_ctx{nullptr};
        try {
            c->impl = new Context(*cfg);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int lfg_close(lfg_ctx* ctx) {
    return guarded([&] {
        if (!ctx) fail(LFG_ERR_INVALID, "null context");
        {
            std::lock_guard<std::mutex> g(ctx->impl->mu);
            refuse_while_streaming(*ctx->impl);
        }
        cudaSetDevice(ctx->impl->cfg.device);
        delete ctx->impl;
        delete ctx;
    });
}

int lfg_synchronize(lfg_ctx* ctx) {
    return guarded([&] {
        Context& c = C(ctx);
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        (void)c;
    });
}

int lfg_host_alloc(lfg_ctx* ctx, size_t bytes, void** out) {
    return guarded([&] {
        C(ctx);
        if (!out) fail(LFG_ERR_INVALID, "null out");
        cuda_check(cudaMallocHost(out, bytes ? bytes : 1), "cudaMallocHost");
    });
}
int lfg_host_free(lfg_ctx* ctx, void* p) {
    return guarded([&] {
        Context& c = C(ctx);
        {
            std::lock_guard<std::mutex> g(c.mu);
            c.forget_pinned();   // its pages may be reused for pageable memory
        }
        cuda_check(cudaFreeHost(p), "cudaFreeHost");
    });
}
int lfg_device_alloc(lfg_ctx* ctx, size_t bytes, void** out) {
    return guarded([&] {
        C(ctx);
        if (!out) fail(LFG_ERR_INVALID, "null out");
        cuda_check(cudaMalloc(out, bytes ? bytes : 1), "cudaMalloc");
    });
}
int lfg_device_free(lfg_ctx* ctx, void* p) {
    return guarded([&] {
        C(ctx);
        cuda_check(cudaFree(p), "cudaFree");
    });
}
int lfg_memcpy_h2d(lfg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        C(ctx);
        cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "H2D");
    });
}
int lfg_memcpy_d2h(lfg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        C(ctx);
        cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "D2H");
    });
}

int lfg_chain_create(lfg_ctx* ctx, const lfg_op* ops, int n_ops, lfg_chain** out) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!out) fail(LFG_ERR_INVALID, "null out");
        std::lock_guard<std::mutex> g(c.mu);
        Chain* ch = c.chain_create(ops, n_ops);
        *out = new lfg_chain{ch, ctx};
    });
}

int lfg_chain_destroy(lfg_ctx* ctx, lfg_chain* chain) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!chain) fail(LFG_ERR_INVALID, "null chain");
        std::lock_guard<std::mutex> g(c.mu);
        refuse_while_streaming(c);
        c.chain_destroy(chain->impl);
        delete chain;
    });
}

int lfg_chain_info(lfg_chain* chain, int* n_stages, int64_t* out_bytes, int* family) {
    return guarded([&] {
        if (!chain) fail(LFG_ERR_INVALID, "null chain");
        if (n_stages) *n_stages = static_cast<int>(chain->impl->stages.size());
        if (out_bytes) *out_bytes = chain->impl->out_bytes;
        if (family) *family = chain->impl->fam;
    });
}

int lfg_chain_stage(lfg_chain* chain, int s, int* first_op, int* last_op) {
    return guarded([&] {
        if (!chain) fail(LFG_ERR_INVALID, "null chain");
        const auto& st = chain->impl->stages;
        if (s < 0 || s >= static_cast<int>(st.size())) fail(LFG_ERR_INVALID, "stage out of range");
        if (first_op) *first_op = st[s].first_op;
        if (last_op) *last_op = st[s].last_op;
    });
}

int lfg_draw_params(lfg_chain* chain, uint64_t seed, const lfg_sample_desc* s, double* out,
                    int cap, int* n_out) {
    return guarded([&] {
        if (!chain || !s || !out) fail(LFG_ERR_INVALID, "null argument");
        const Chain& c = *chain->impl;
        std::vector<double> v;
        if (c.fam == FAM_IMG3D) {
            Params3D p;
            draw_3d(c, seed, s->id, s->dims, p);
            v = {double(p.off[0]), double(p.off[1]), double(p.off[2]), double(p.flip[0]),
                 double(p.flip[1]), double(p.flip[2]), p.scale, p.sigma, double(p.key[0]),
                 double(p.key[1]), double(p.win[0]), double(p.win[1]), double(p.win[2]), p.contrast,
                 double(p.fg), p.u_cls, p.u_adj[0], p.u_adj[1], p.u_adj[2]};
        } else if (c.fam == FAM_RRC2D) {
            Params2D p;
            draw_2d(c, seed, s->id, s->dims[0], s->dims[1], p);
            v = {double(p.top), double(p.left), double(p.h), double(p.w), double(p.flip)};
        } else {
            ParamsSp p;
            draw_sp(c, seed, s->id, s->dims[0], p);
            v.push_back(p.T);
            v.push_back(c.n_fmask);
            for (int i = 0; i < c.n_fmask; ++i) {
                v.push_back(p.f_lo[i]);
                v.push_back(p.f_w[i]);
            }
            v.push_back(c.n_tmask);
            for (int i = 0; i < c.n_tmask; ++i) {
                v.push_back(p.t_lo[i]);
                v.push_back(p.t_w[i]);
            }
        }
        if (static_cast<int>(v.size()) > cap) fail(LFG_ERR_INVALID, "params buffer too small");
        std::memcpy(out, v.data(), v.size() * sizeof(double));
        if (n_out) *n_out = static_cast<int>(v.size());
    });
}

int lfg_rng_outputs(uint64_t seed, uint64_t id, int n, uint64_t* out) {
    return guarded([&] {
        if (n < 0 || (n > 0 && !out)) fail(LFG_ERR_INVALID, "bad output buffer");
        rng_outputs(seed, id, n, out);
    });
}

int lfg_submit(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* s, lfg_ticket* out) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!chain || !s || !out) fail(LFG_ERR_INVALID, "null argument");
        std::lock_guard<std::mutex> g(c.mu);
        refuse_while_streaming(c);
        *out = c.submit(chain->impl, *s);
    });
}

int lfg_flush(lfg_ctx* ctx) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        c.flush_due();
    });
}

int lfg_progress(lfg_ctx* ctx, lfg_ticket t, int* ops_done, int* complete, int64_t* elapsed_us) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        c.progress(t, ops_done, complete, elapsed_us);
    });
}

int lfg_wait(lfg_ctx* ctx, lfg_ticket t) {
    // Never block while holding the context lock: a slow sample's wait (the
    // resume path) would stall every other thread's progress polls and push
    // their fast samples past t_out.  Launch under the lock, then poll.
    return guarded([&] {
        Context& c = C(ctx);
        {
            std::lock_guard<std::mutex> g(c.mu);
            if (c.launch_if_pending(t)) return;
        }
        for (int spins = 0;; ++spins) {
            {
                std::lock_guard<std::mutex> g(c.mu);
                c.group_of(t);   // validates the ticket
                if (c.sample_ready(t)) return;   // its own stamp, or the whole group
            }
            if (spins < 64) std::this_thread::yield();
            else std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    });
}

int lfg_wait_for(lfg_ctx* ctx, lfg_ticket t, int64_t timeout_us, int* complete) {
    // Blocks (without the context lock) until the ticket's sample finished or the
    // timeout passed.  A coalescing group still open is launched once due; launched
    // groups wake their waiters through the completion notice (coalesce_us > 0),
    // otherwise the wait polls.
    return guarded([&] {
        Context& c = C(ctx);
        if (!complete) fail(LFG_ERR_INVALID, "null out");
        *complete = 0;
        const int64_t deadline = host_now_us() + std::max<int64_t>(0, timeout_us);
        for (;;) {
            int64_t serial = 0, due = 0;
            {
                std::lock_guard<std::mutex> g(c.mu);
                Group& gr = c.group_of(t);
                const int64_t now = host_now_us();
                if (!gr.launched && !gr.complete && c.cfg.coalesce_us > 0 && now - gr.t_open_us >= c.cfg.coalesce_us)
                    c.launch_if_pending(t);
                if (gr.launched && c.group_done_notified(gr.serial)) c.poll_group(gr);
                if (c.sample_ready(t)) {
                    *complete = 1;
                    return;
                }
                serial = gr.launched ? gr.serial : 0;
                due = gr.launched ? 0 : gr.t_open_us + std::max(1, c.cfg.coalesce_us);
            }
            const int64_t now = host_now_us();
            if (now >= deadline) return;
            int64_t until = deadline;
            if (serial == 0) until = std::min(until, std::max(due, now + 1));   // wake to launch it when due
            if (serial > 0 && c.cfg.coalesce_us > 0) {
                const int w = static_cast<int>(serial & (Context::kDoneWaits - 1));
                std::unique_lock<std::mutex> lk(c.done_mu_[w]);
                c.done_cv_[w].wait_for(lk, std::chrono::microseconds(until - now),
                                       [&] { return c.group_done_notified(serial); });
            } else {
                std::this_thread::sleep_for(std::chrono::microseconds(std::min<int64_t>(until - now, 20)));
            }
        }
    });
}

int lfg_exec_costs(lfg_ctx* ctx, lfg_ticket t, double* costs_us, int cap, int* n_out) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!costs_us) fail(LFG_ERR_INVALID, "null out");
        std::lock_guard<std::mutex> g(c.mu);
        const int n = c.exec_costs(t, costs_us, cap);
        if (n_out) *n_out = n;
    });
}

int lfg_ticket_output(lfg_ctx* ctx, lfg_ticket t, void* host_dst, size_t bytes) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!host_dst) fail(LFG_ERR_INVALID, "null out");
        std::lock_guard<std::mutex> g(c.mu);
        c.ticket_output(t, host_dst, bytes);
    });
}

int lfg_ticket_release(lfg_ctx* ctx, lfg_ticket t) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        c.ticket_release(t);
    });
}

int lfg_seal_batch(lfg_ctx* ctx, const lfg_ticket* tickets, int n, lfg_batch* out) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!tickets || !out) fail(LFG_ERR_INVALID, "null argument");
        std::lock_guard<std::mutex> g(c.mu);
        refuse_while_streaming(c);
        *out = c.seal(tickets, n);
    });
}

int lfg_batch_info(lfg_ctx* ctx, lfg_batch b, void** dev_ptr, int64_t* bytes, int* n,
                   uint64_t* ids, int* in_place) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        BatchRec& br = c.batch(b);
        if (n) *n = br.n;
        if (ids) std::memcpy(ids, br.ids.data(), br.ids.size() * sizeof(uint64_t));
        if (in_place) *in_place = br.in_place ? 1 : 0;
        if (dev_ptr || bytes) {
            void* p = nullptr;
            int64_t by = 0;
            c.batch_ptr(br, &p, &by);  // planar [plane0: cap x p0][plane1: cap x p1]
            if (dev_ptr) *dev_ptr = p;
            if (bytes) *bytes = by;
        }
    });
}

int lfg_batch_wait_stream(lfg_ctx* ctx, lfg_batch b, void* stream) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        c.batch_wait_stream(b, static_cast<cudaStream_t>(stream));
    });
}

int lfg_batch_lengths(lfg_ctx* ctx, lfg_batch b, int32_t* lengths, int32_t* t_max) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        BatchRec& br = c.batch(b);
        if (br.chain->fam != FAM_SPEECH) fail(LFG_ERR_INVALID, "lengths exist for speech batches only");
        if (lengths) std::memcpy(lengths, br.rows.data(), br.rows.size() * sizeof(int32_t));
        if (t_max) *t_max = br.t_max;
    });
}

int lfg_batch_copy_to_host(lfg_ctx* ctx, lfg_batch b, void* host_dst, size_t bytes) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!host_dst) fail(LFG_ERR_INVALID, "null out");
        std::lock_guard<std::mutex> g(c.mu);
        BatchRec& br = c.batch(b);
        const Chain& ch = *br.chain;
        void* p = nullptr;
        int64_t by = 0;
        c.batch_ptr(br, &p, &by);
        if (ch.fam == FAM_SPEECH) {   // time-major [t_max, n, stack * 80]
            const int64_t need = int64_t(br.t_max) * br.n * ch.stack * ch.n_mels * 4;
            if (static_cast<int64_t>(bytes) < need) fail(LFG_ERR_INVALID, "host buffer too small");
            if (br.ready) cuda_check(cudaEventSynchronize(br.ready), "batch ready");
            cuda_check(cudaMemcpy(host_dst, p, need, cudaMemcpyDeviceToHost), "D2H batch");
            c.counters.d2h_bytes += need;
            return;
        }
        const int64_t need = static_cast<int64_t>(br.n) * ch.out_bytes;
        if (static_cast<int64_t>(bytes) < need) fail(LFG_ERR_INVALID, "host buffer too small");
        if (br.ready) cuda_check(cudaEventSynchronize(br.ready), "batch ready");
        char* d = static_cast<char*>(host_dst);
        const int64_t cap = c.cfg.batch_size;
        cuda_check(cudaMemcpy(d, p, br.n * ch.plane_bytes[0], cudaMemcpyDeviceToHost), "D2H batch");
        if (ch.nplanes > 1)
            cuda_check(cudaMemcpy(d + br.n * ch.plane_bytes[0],
                                  static_cast<char*>(p) + cap * ch.plane_bytes[0],
                                  br.n * ch.plane_bytes[1], cudaMemcpyDeviceToHost),
                       "D2H batch");
        c.counters.d2h_bytes += need;
    });
}

int lfg_batch_release(lfg_ctx* ctx, lfg_batch b, void* stream) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        c.batch_release(b, static_cast<cudaStream_t>(stream));
    });
}

int lfg_trainer_step(lfg_ctx* ctx, lfg_batch b, void* stream, int64_t us) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        c.trainer_step(b, static_cast<cudaStream_t>(stream), us);
    });
}

int lfg_synth_volume(lfg_ctx* ctx, uint64_t seed, uint64_t id, int64_t D, int64_t H, int64_t W,
                     void* img_f32, void* lbl_u8, int on_device) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!img_f32 || !lbl_u8 || D < 1 || H < 1 || W < 1) fail(LFG_ERR_INVALID, "bad volume");
        if (on_device) {
            cuda_check(launch_synth_volume(seed, id, D, H, W, static_cast<float*>(img_f32),
                                           static_cast<uint8_t*>(lbl_u8), c.aux_stream),
                       "synth volume");
            cuda_check(cudaStreamSynchronize(c.aux_stream), "synth sync");
            return;
        }
        float* img = static_cast<float*>(img_f32);
        uint8_t* lbl = static_cast<uint8_t*>(lbl_u8);
        const int64_t n = D * H * W;
        const int64_t chunks = (n + 4 * 65536 - 1) / (4 * 65536);
        parallel_for(chunks, [&](int64_t ck) {
            for (int64_t q = ck * 65536; q < std::min<int64_t>((ck + 1) * 65536, (n + 3) / 4); ++q) {
                uint32_t r[4];
                h_synth_rand(seed, id, uint64_t(q), 1u, r);
                float z[4];
                h_bm(r[0], r[1], z[0], z[1]);
                h_bm(r[2], r[3], z[2], z[3]);
                for (int j = 0; j < 4; ++j) {
                    const int64_t v = q * 4 + j;
                    if (v >= n) break;
                    img[v] = z[j];
                    const int64_t x = v % W, y = (v / W) % H, zz = v / (W * H);
                    const float dz = (zz - 0.5f * D) / (0.25f * D), dy = (y - 0.5f * H) / (0.25f * H),
                                dx = (x - 0.5f * W) / (0.25f * W);
                    const float tz = (zz - 0.55f * D) / (0.08f * D), ty = (y - 0.45f * H) / (0.08f * H),
                                tx = (x - 0.5f * W) / (0.08f * W);
                    const float e = dz * dz + dy * dy + dx * dx, t = tz * tz + ty * ty + tx * tx;
                    lbl[v] = t <= 1.0f ? 2 : (e <= 1.0f ? 1 : 0);
                }
            }
        });
    });
}

int lfg_synth_image(lfg_ctx* ctx, uint64_t seed, uint64_t id, int64_t H, int64_t W, void* hwc_u8,
                    int on_device) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!hwc_u8 || H < 1 || W < 1) fail(LFG_ERR_INVALID, "bad image");
        if (on_device) {
            cuda_check(launch_synth_image(seed, id, H, W, static_cast<uint8_t*>(hwc_u8), c.aux_stream),
                       "synth image");
            cuda_check(cudaStreamSynchronize(c.aux_stream), "synth sync");
            return;
        }
        uint8_t* out = static_cast<uint8_t*>(hwc_u8);
        const int64_t n = H * W * 3;
        for (int64_t q = 0; q * 16 < n; ++q) {
            uint32_t r[4];
            h_synth_rand(seed, id, uint64_t(q), 2u, r);
            for (int j = 0; j < 16; ++j) {
                const int64_t v = q * 16 + j;
                if (v < n) out[v] = uint8_t(r[j >> 2] >> (8 * (j & 3)));
            }
        }
    });
}

int lfg_synth_waveform(lfg_ctx* ctx, uint64_t seed, uint64_t id, int64_t L, void* wav_f32,
                       int on_device) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!wav_f32 || L < 1) fail(LFG_ERR_INVALID, "bad waveform");
        if (on_device) {
            cuda_check(launch_synth_waveform(seed, id, L, static_cast<float*>(wav_f32), c.aux_stream),
                       "synth waveform");
            cuda_check(cudaStreamSynchronize(c.aux_stream), "synth sync");
            return;
        }
        float* wav = static_cast<float*>(wav_f32);
        uint32_t f[4];
        h_synth_rand(seed, id, 0xFFFFFFFFull, 3u, f);
        const double f1 = 100.0 + (f[0] % 700u), f2 = 300.0 + (f[1] % 1500u), f3 = 1000.0 + (f[2] % 5000u);
        for (int64_t q = 0; q * 4 < L; ++q) {
            uint32_t r[4];
            h_synth_rand(seed, id, uint64_t(q), 4u, r);
            float z[4];
            h_bm(r[0], r[1], z[0], z[1]);
            h_bm(r[2], r[3], z[2], z[3]);
            for (int j = 0; j < 4; ++j) {
                const int64_t v = q * 4 + j;
                if (v >= L) break;
                const double t = double(v) / 16000.0;
                wav[v] = float(0.5 * std::sin(2 * M_PI * f1 * t) + 0.3 * std::sin(2 * M_PI * f2 * t) +
                               0.2 * std::sin(2 * M_PI * f3 * t) + 0.01 * z[j]);
            }
        }
    });
}

int lfg_get_counters(lfg_ctx* ctx, lfg_counters* out) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!out) fail(LFG_ERR_INVALID, "null out");
        std::lock_guard<std::mutex> g(c.mu);
        *out = c.counters;
    });
}

int lfg_time_kernels(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* samples, int n,
                     double* mean_ms, int64_t* launches, int64_t* bytes, int64_t* flops) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!chain || !samples || !mean_ms || !launches || !bytes || !flops) fail(LFG_ERR_INVALID, "null argument");
        std::lock_guard<std::mutex> g(c.mu);
        refuse_while_streaming(c);
        c.time_kernels(chain->impl, samples, n, mean_ms, launches, bytes, flops);
    });
}

int lfg_set_serial(lfg_ctx* ctx, int serial) {
    return guarded([&] {
        Context& c = C(ctx);
        std::lock_guard<std::mutex> g(c.mu);
        c.serial = serial != 0;
    });
}

int lfg_run_shard(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* samples, int64_t n,
                  const lfg_run_config* cfg, lfg_run_report* report, uint64_t* consumed_ids,
                  int32_t* batch_sizes, int32_t* sample_class) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!chain || !cfg || !report) fail(LFG_ERR_INVALID, "null argument");
        std::lock_guard<std::mutex> g(c.mu);
        refuse_while_streaming(c);
        run_shard(c, chain->impl, samples, n, *cfg, *report, consumed_ids, batch_sizes,
                  sample_class);
    });
}

int lfg_run_shard_source(lfg_ctx* ctx, lfg_chain* chain, const lfg_source* src, int64_t n,
                         const lfg_run_config* cfg, lfg_run_report* report, uint64_t* consumed_ids,
                         int32_t* batch_sizes, int32_t* sample_class) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!chain || !cfg || !report || !src) fail(LFG_ERR_INVALID, "null argument");
        std::lock_guard<std::mutex> g(c.mu);
        refuse_while_streaming(c);
        run_shard(c, chain->impl, nullptr, n, *cfg, *report, consumed_ids, batch_sizes, sample_class, src);
    });
}

namespace {
void shard_deliver(void* user, int64_t b, int n) {
    auto* sh = static_cast<lfg_shard*>(user);
    {
        std::lock_guard<std::mutex> g(sh->qm);
        sh->q.emplace_back(b, n);
    }
    sh->cv.notify_one();
}
}  // namespace

int lfg_shard_start(lfg_ctx* ctx, lfg_chain* chain, const lfg_sample_desc* samples, int64_t n,
                    const lfg_run_config* cfg, lfg_shard** out) {
    return guarded([&] {
        Context& c = C(ctx);
        if (!chain || !cfg || !out || n < 0 || (n > 0 && !samples)) fail(LFG_ERR_INVALID, "null argument");
        *out = nullptr;
        {
            std::lock_guard<std::mutex> g(c.mu);
            if (c.streaming) fail(LFG_ERR_STATE, "a streaming shard run is already active on this context");
            c.streaming = true;
        }
        struct Unclaim {   // until the run's thread owns the flag, a throw hands it back
            Context* c;
            ~Unclaim() {
                if (c) {
                    std::lock_guard<std::mutex> g(c->mu);
                    c->streaming = false;
                }
            }
        } unclaim{&c};
        auto sh = std::make_unique<lfg_shard>();
        sh->ctx = ctx;
        sh->samples.assign(samples, samples + n);
        sh->cfg = *cfg;
        sh->cfg.trainer_us = 0;   // the caller is the trainer
        sh->ids.resize(static_cast<size_t>(n));
        sh->sizes.resize(static_cast<size_t>(n));
        sh->cls.resize(static_cast<size_t>(n));
        lfg_shard* p = sh.get();
        Chain* ch = chain->impl;
        p->th = std::thread([p, ch, n] {
            Context& cx = *p->ctx->impl;
            int rc = LFG_OK;
            std::string err;
            try {
                cuda_check(cudaSetDevice(cx.cfg.device), "cudaSetDevice");
                ShardStream ss;
                ss.lock = &cx.mu;
                ss.deliver = shard_deliver;
                ss.user = p;
                run_shard(cx, ch, p->samples.data(), n, p->cfg, p->rep, p->ids.data(), p->sizes.data(),
                          p->cls.data(), nullptr, &ss);
            } catch (const Error& e) {
                rc = e.code;
                err = e.msg;
            } catch (const std::exception& e) {
                rc = LFG_ERR_STATE;
                err = e.what();
            }
            {
                std::lock_guard<std::mutex> g(cx.mu);
                cx.streaming = false;
            }
            {
                std::lock_guard<std::mutex> g(p->qm);
                p->rc = rc;
                p->err = err;
                p->ended = true;
            }
            p->cv.notify_all();
        });
        unclaim.c = nullptr;
        *out = sh.release();
    });
}

int lfg_shard_next_batch(lfg_shard* sh, int64_t timeout_us, lfg_batch* out, int* n) {
    return guarded([&] {
        if (!sh || !out) fail(LFG_ERR_INVALID, "null argument");
        const auto t0 = std::chrono::steady_clock::now();
        if (!sh->started) {
            sh->started = true;
            sh->t_first = t0;
        }
        std::unique_lock<std::mutex> lk(sh->qm);
        auto have = [&] { return !sh->q.empty() || sh->ended; };
        if (timeout_us < 0) sh->cv.wait(lk, have);
        else sh->cv.wait_for(lk, std::chrono::microseconds(timeout_us), have);
        const auto t1 = std::chrono::steady_clock::now();
        sh->wait_us += std::chrono::duration<double, std::micro>(t1 - t0).count();
        sh->t_last = t1;
        if (!sh->q.empty()) {
            *out = sh->q.front().first;
            if (n) *n = sh->q.front().second;
            sh->q.pop_front();
            ++sh->taken;
            return;
        }
        if (!sh->ended) fail(LFG_ERR_AGAIN, "no batch sealed within the timeout");
        if (sh->rc != LFG_OK) fail(sh->rc, "shard run failed: " + sh->err);
        fail(LFG_ERR_CLOSED, "end of stream: every sample was delivered");
    });
}

int lfg_shard_finish(lfg_shard* sh, lfg_run_report* report, uint64_t* consumed_ids, int32_t* batch_sizes,
                     int32_t* sample_class) {
    if (!sh) {
        g_last_error = "null shard";
        return LFG_ERR_INVALID;
    }
    // drain: batches the consumer never took go back to the pool as they arrive
    for (;;) {
        std::pair<int64_t, int> b{-1, 0};
        bool end = false;
        {
            std::unique_lock<std::mutex> lk(sh->qm);
            sh->cv.wait(lk, [&] { return !sh->q.empty() || sh->ended; });
            if (!sh->q.empty()) {
                b = sh->q.front();
                sh->q.pop_front();
            } else {
                end = true;
            }
        }
        if (end) break;
        lfg_batch_release(sh->ctx, b.first, nullptr);
    }
    if (sh->th.joinable()) sh->th.join();
    const int rc = sh->rc;
    if (rc == LFG_OK) {
        const int64_t n = static_cast<int64_t>(sh->samples.size());
        if (report) {
            *report = sh->rep;
            // consumer idle as ConsumerStats counts it: time blocked waiting for a batch
            // over the consumer's span (first next_batch call .. last return)
            const double span = sh->started ? std::chrono::duration<double, std::micro>(sh->t_last - sh->t_first).count() : 0.0;
            report->consumer_span_ms = span / 1000.0;
            report->consumer_busy_ms = std::max(0.0, span - sh->wait_us) / 1000.0;
            report->consumer_idle_frac = span > 0 ? std::min(1.0, sh->wait_us / span) : 1.0;
        }
        if (consumed_ids) std::copy(sh->ids.begin(), sh->ids.begin() + std::min<int64_t>(n, sh->rep.samples), consumed_ids);
        if (batch_sizes) std::copy(sh->sizes.begin(), sh->sizes.begin() + std::min<int64_t>(n, sh->rep.batches), batch_sizes);
        if (sample_class) std::copy(sh->cls.begin(), sh->cls.end(), sample_class);
    } else {
        g_last_error = "shard run failed: " + sh->err;
    }
    delete sh;
    return rc;
}

}  // extern "C"
