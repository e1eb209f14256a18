// engine.cpp -- launch groups, tickets, output slot buffers and batch sealing.
//
// Reference mapping (proj/):
//   submit + launch_group  <- process_sample's transform loop (src/balancer.cpp:42-77)
//                             on a WorkerPool slot (src/worker_pool.cpp:63-98)
//   poll_group / progress  <- the cooperative budget check after each transform
//                             (balancer.cpp:55); here one CUDA event per fused stage
//   seal                   <- build_batches' seal_and_publish (src/batcher.cpp:50-58)
//   batch_release          <- the consumer dropping its Batch (src/trainer.cpp:20-66)
#include "engine.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <optional>

namespace lfg {

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fail(LFG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

int64_t host_now_us() {
    using namespace std::chrono;
    return duration_cast<microseconds>(steady_clock::now().time_since_epoch()).count();
}

static int64_t rows_touched(int64_t h, int oh);

// ------------------------------------------------------------------ params
// Per-sample generator: the reference's Rng (std::mt19937_64, sample.hpp:25)
// seeded with experiment.cpp:163's mixing constant keyed by sample id.
namespace {
// std::mt19937_64, bit-exact, evaluated lazily.  A sample draws at most a few
// dozen numbers, but std::mt19937_64 seeds all 312 state words and twists all of
// them before its first output (~1.3 us).  Output k < 156 depends only on the
// seeded words k, k + 1 and k + 156 (the twist reads x[k + 156] before it is
// rewritten), so this generator seeds words on demand (157 + k of them) and
// twists one word per output; from output 156 on it falls back to the library
// generator advanced to the same position.
class LazyMt64 {
public:
    explicit LazyMt64(uint64_t seed) : seeded_(1) { x_[0] = seed; }
    uint64_t operator()() {
        if (k_ >= kM) {
            if (!full_) {
                full_.emplace(x_[0]);
                full_->discard(static_cast<unsigned long long>(k_));
            }
            ++k_;
            return (*full_)();
        }
        const int need = k_ + kM + 1;
        while (seeded_ < need) {
            const uint64_t p = x_[seeded_ - 1];
            x_[seeded_] = 6364136223846793005ULL * (p ^ (p >> 62)) + static_cast<uint64_t>(seeded_);
            ++seeded_;
        }
        const uint64_t y = (x_[k_] & 0xFFFFFFFF80000000ULL) | (x_[k_ + 1] & 0x7FFFFFFFULL);
        uint64_t z = x_[k_ + kM] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        ++k_;
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        z ^= z >> 43;
        return z;
    }

private:
    static constexpr int kM = 156;
    uint64_t x_[312];
    int seeded_;
    int k_ = 0;
    std::optional<std::mt19937_64> full_;
};

struct SampleRng {
    LazyMt64 g;
    SampleRng(uint64_t seed, uint64_t id) : g(seed ^ (0x9e3779b97f4a7c15ULL * (id + 1ULL))) {}
    double unif01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    int64_t randint(int64_t lo, int64_t hi) {
        const double u = unif01();
        const int64_t span = hi - lo + 1;
        int64_t k = static_cast<int64_t>(std::floor(u * static_cast<double>(span)));
        if (k >= span) k = span - 1;
        return lo + k;
    }
    double uniform(double a, double b) { return a + (b - a) * unif01(); }
};
}  // namespace

// Draw order (chain order; oracle/lf_oracle.c lfo_draw3d): RandomCrop offset
// uniforms, [its foreground draws: apply, class, 3 placements], [RandomZoom3D
// apply + factor], flips, brightness, [RandomContrast
// apply + factor], noise, Philox key.  The offset is floor(u * (room + 1)) once
// the window edge is known -- randint(0, room) of the plain chain.
void draw_3d(const Chain& c, uint64_t seed, uint64_t id, const int64_t dims[3], Params3D& p) {
    SampleRng r(seed, id);
    double u_off[3];
    for (int a = 0; a < 3; ++a) u_off[a] = r.unif01();
    p.fg = 0;
    p.u_cls = 0.0;
    p.u_adj[0] = p.u_adj[1] = p.u_adj[2] = 0.0;
    if (c.has_fg) {   // RandomCrop's foreground draws
        p.fg = r.unif01() < c.p_fg;
        p.u_cls = r.unif01();
        for (int a = 0; a < 3; ++a) p.u_adj[a] = r.unif01();
    }
    for (int a = 0; a < 3; ++a) p.win[a] = c.crop[a];
    if (c.has_zoom) {
        const bool z_apply = r.unif01() < c.p_zoom;
        const double zf = r.uniform(c.z_lo, c.z_hi);
        if (z_apply)
            for (int a = 0; a < 3; ++a)
                p.win[a] = std::max<int64_t>(1, static_cast<int64_t>(std::floor(c.crop[a] * zf + 0.5)));
    }
    for (int a = 0; a < 3; ++a) {
        const int64_t room = dims[a] - p.win[a];
        const int64_t span = (room > 0 ? room : 0) + 1;
        const int64_t k = static_cast<int64_t>(std::floor(u_off[a] * static_cast<double>(span)));
        p.off[a] = k >= span ? span - 1 : k;
    }
    for (int a = 0; a < 3; ++a) p.flip[a] = r.unif01() < c.p_flip;
    const bool b_apply = r.unif01() < c.p_bright;
    const double b_factor = r.uniform(c.b_lo, c.b_hi);
    p.scale = b_apply ? b_factor : 1.0;
    p.contrast = 1.0;
    if (c.has_contrast) {
        const bool c_apply = r.unif01() < c.p_contrast;
        const double c_factor = r.uniform(c.c_lo, c.c_hi);
        if (c_apply) p.contrast = c_factor;
    }
    const bool n_apply = r.unif01() < c.p_noise;
    const double n_std = r.uniform(0.0, c.noise_max);
    const uint64_t key = r.g();
    p.sigma = n_apply ? n_std : 0.0;
    p.key[0] = static_cast<uint32_t>(key);
    p.key[1] = static_cast<uint32_t>(key >> 32);
}

void draw_2d(const Chain& c, uint64_t seed, uint64_t id, int64_t H, int64_t W, Params2D& p) {
    // torchvision RandomResizedCrop.get_params restated on the per-sample Rng
    SampleRng r(seed, id);
    const double area = static_cast<double>(H) * static_cast<double>(W);
    const double lr0 = std::log(c.ratio_lo), lr1 = std::log(c.ratio_hi);
    bool found = false;
    for (int t = 0; t < 10 && !found; ++t) {
        const double target = area * r.uniform(c.scale_lo, c.scale_hi);
        const double aspect = std::exp(r.uniform(lr0, lr1));
        const int64_t w = static_cast<int64_t>(std::nearbyint(std::sqrt(target * aspect)));
        const int64_t h = static_cast<int64_t>(std::nearbyint(std::sqrt(target / aspect)));
        if (w > 0 && w <= W && h > 0 && h <= H) {
            p.top = r.randint(0, H - h);
            p.left = r.randint(0, W - w);
            p.h = h;
            p.w = w;
            found = true;
        }
    }
    if (!found) {
        const double in_ratio = static_cast<double>(W) / static_cast<double>(H);
        int64_t w = W, h = H;
        if (in_ratio < c.ratio_lo) {
            h = static_cast<int64_t>(std::nearbyint(static_cast<double>(w) / c.ratio_lo));
        } else if (in_ratio > c.ratio_hi) {
            w = static_cast<int64_t>(std::nearbyint(static_cast<double>(h) * c.ratio_hi));
        }
        p.top = (H - h) / 2;
        p.left = (W - w) / 2;
        p.h = h;
        p.w = w;
    }
    p.flip = r.unif01() < c.p_hflip;
    p.rows_touched = rows_touched(p.h, c.oh);
}

void draw_sp(const Chain& c, uint64_t seed, uint64_t id, int64_t L, ParamsSp& p) {
    SampleRng r(seed, id);
    p.T = static_cast<int>(1 + L / c.hop);
    for (int i = 0; i < c.n_fmask; ++i) {
        int w = static_cast<int>(r.randint(0, c.fmask_max));
        if (w > c.n_mels) w = c.n_mels;
        p.f_w[i] = w;
        p.f_lo[i] = static_cast<int>(r.randint(0, c.n_mels - w));
    }
    const int tmax = static_cast<int>(std::floor(c.tmask_frac * p.T));
    for (int i = 0; i < c.n_tmask; ++i) {
        const int w = static_cast<int>(r.randint(0, tmax));
        p.t_w[i] = w;
        const int room = p.T - w;
        p.t_lo[i] = static_cast<int>(r.randint(0, room > 0 ? room : 0));
    }
}

// Algorithmic HBM bytes of K3 for one sample: the distinct source rows the
// bilinear taps touch (exact, from the same index formula the kernel uses)
// times the crop-box row bytes, plus the f32 output.
int64_t rrc_algo_bytes(const Chain& c, const Params2D& p) {
    return p.rows_touched * p.w * 3 + c.out_bytes;
}

static int64_t rows_touched(int64_t h, int oh) {
    int64_t rows = 0, last = -1;
    const double scale = static_cast<double>(h) / oh;
    for (int y = 0; y < oh; ++y) {
        double src = (y + 0.5) * scale - 0.5;
        if (src < 0) src = 0;
        int64_t a = static_cast<int64_t>(std::floor(src));
        if (a > h - 1) a = h - 1;
        const int64_t b = a < h - 1 ? a + 1 : a;
        if (a > last) ++rows;
        if (b > a && b > last) ++rows;
        last = std::max(last, b);
    }
    return rows;
}

int64_t Chain::algo_bytes_per_sample(const lfg_sample_desc& s) const {
    switch (fam) {
        case FAM_IMG3D: {
            const int64_t vox = int64_t(crop[0]) * crop[1] * crop[2];
            return vox * 10;  // read f32 + u8, write f32 + u8 (zoomed windows: img3d_algo_bytes)
        }
        case FAM_RRC2D: {
            (void)s;
            return out_bytes;  // write side; the read side is added per sample by the caller
        }
        case FAM_SPEECH:
            return wav_bytes * s.dims[0] + out_bytes;
        default:
            return 0;
    }
}

// ------------------------------------------------------------------ worker threads
WorkerThreads::WorkerThreads(int n) {
    for (int w = 0; w < n; ++w)
        th_.emplace_back([this, w] {
            uint64_t seen = 0;
            for (;;) {
                std::function<void(int)> f;
                {
                    std::unique_lock<std::mutex> l(m_);
                    cv_.wait(l, [&] { return quit_ || gen_ != seen; });
                    if (quit_) return;
                    seen = gen_;
                    f = job_;
                }
                f(w);
                std::lock_guard<std::mutex> l(m_);
                if (--busy_ == 0) idle_.notify_all();
            }
        });
}

WorkerThreads::~WorkerThreads() {
    {
        std::lock_guard<std::mutex> l(m_);
        quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
}

void WorkerThreads::run(std::function<void(int)> f) {
    std::lock_guard<std::mutex> l(m_);
    job_ = std::move(f);
    busy_ = static_cast<int>(th_.size());
    ++gen_;
    cv_.notify_all();
}

void WorkerThreads::wait() {
    std::unique_lock<std::mutex> l(m_);
    idle_.wait(l, [&] { return busy_ == 0; });
    job_ = nullptr;
}

// ------------------------------------------------------------------ context
Context::Context(const lfg_config& c) : cfg(c) {
    if (cfg.n_workers < 1) fail(LFG_ERR_INVALID, "n_workers must be >= 1");
    if (cfg.batch_size < 1) fail(LFG_ERR_INVALID, "batch_size must be >= 1");
    if (cfg.max_group < 1) fail(LFG_ERR_INVALID, "max_group must be >= 1");
    if (cfg.max_slot_buffers < 2) fail(LFG_ERR_INVALID, "max_slot_buffers must be >= 2");
    if (cfg.batch_size > kMaxGather) fail(LFG_ERR_INVALID, "batch_size must be <= 256");
    cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice");
    cuda_check(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, cfg.device),
               "sm count");
    // (A/B experiment) L2 -> DRAM fetch granularity hint in bytes (LFG_L2_FETCH=32|64|128)
    if (const char* e = std::getenv("LFG_L2_FETCH")) {
        size_t v = 0;
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(std::atoi(e)));
        cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
        std::fprintf(stderr, "[lfg] L2 fetch granularity %zu\n", v);
    }
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    cuda_check(cudaStreamCreateWithPriority(&seal_stream, cudaStreamNonBlocking, hi), "seal stream");
    cuda_check(cudaStreamCreateWithFlags(&aux_stream, cudaStreamNonBlocking), "aux stream");
    side_streams_.resize(4);
    for (auto& ss : side_streams_) cuda_check(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking), "side stream");
    // Nothing that can implicitly synchronise the device (stream / event /
    // buffer creation) may run inside the shard loop: a blocked host loop
    // would push in-flight samples past t_out.  Pools are created up front.
    // Stream pool = the hardware work queues minus the seal / aux / trainer
    // streams (and one spare), so no two launch groups share a queue: a parked
    // (slow) group must not create a false dependency for the fast groups behind
    // it.  The queue count is the process's CUDA_DEVICE_MAX_CONNECTIONS (CUDA's
    // default 8 if unset), which CUDA reads when the device context is created;
    // the library never sets it -- applications that want up to 28 concurrent
    // launch groups export CUDA_DEVICE_MAX_CONNECTIONS=32 before their first CUDA
    // call (bench.py, the tests and the CLI do).  The shard's in-flight group
    // limit is capped at the pool size.
    {
        int conn = 8;
        if (const char* e = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS")) conn = std::atoi(e);
        stream_pool = std::clamp(conn - 4, 4, kMaxStreamPool);
    }
    for (int i = 0; i < stream_pool; ++i) {
        cudaStream_t s;
        cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        streams_.push_back(s);
        if (i > 0) free_streams_.push_back(static_cast<int>(streams_.size()) - 1);
    }
    cuda_check(warm_stage(), "load stage kernel");
    cuda_check(warm_img3d(), "load img3d kernel");
    cuda_check(warm_img3d_zoom(), "load img3d zoom kernels");
    cuda_check(cudaMalloc(&csum_, kCsumSlots * sizeof(double)), "contrast sums");
    cuda_check(cudaMalloc(&fg_box_, size_t(kFgSlots) * kMax3D * 48 * sizeof(int32_t)), "fg boxes");
    cuda_check(cudaMalloc(&fg_offs_, size_t(kFgSlots) * kMax3D * sizeof(int4)), "fg offsets");
    cuda_check(warm_rrc2d(), "load rrc2d kernel");
    cuda_check(warm_misc(), "load misc kernels");
    cuda_check(warm_speech(), "load speech kernels");
    if (const char* e = std::getenv("LFG_IMG3D_TMA")) img3d_tma_ = std::atoi(e) != 0;
    for (int i = 0; i < 512; ++i) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        free_events_.push_back(e);
        cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        free_tevents_.push_back(e);
    }
    // per-sample completion stamps: host-mapped words the kernels write, device counters
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&stamp_host_), kStampSlots * sizeof(uint64_t),
                             cudaHostAllocMapped | cudaHostAllocPortable),
               "stamp words");
    std::memset(stamp_host_, 0, kStampSlots * sizeof(uint64_t));
    cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&stamp_dev_), stamp_host_, 0), "stamp words");
    cuda_check(cudaMalloc(&stamp_cnt_, kStampSlots * sizeof(uint32_t)), "stamp counters");
    cuda_check(cudaMemset(stamp_cnt_, 0, kStampSlots * sizeof(uint32_t)), "stamp counters");
    // Host tables of shard runs, faulted in once here (a run of up to kPrefault samples
    // then takes no page fault on its ticket or parameter tables; larger runs grow them)
    {
        constexpr size_t kPrefault = size_t(1) << 16;
        tickets.resize(kPrefault);
        tickets.clear();
        pre_store.resize(kPrefault);
        std::memset(static_cast<void*>(pre_store.data()), 0, kPrefault * sizeof(PreDraw));
        groups.reserve(kPrefault / 8);
    }
    done_ring_.reset(new std::atomic<int64_t>[kDoneSlots]);
    for (int i = 0; i < kDoneSlots; ++i) done_ring_[i].store(0, std::memory_order_relaxed);
    // draw workers: half the host threads (the shard loop and the trainer keep theirs), <= 16
    workers = std::make_unique<WorkerThreads>(
        static_cast<int>(std::clamp(std::thread::hardware_concurrency() / 2, 1u, 16u)));
}

Context::~Context() {
    cudaSetDevice(cfg.device);
    cudaDeviceSynchronize();
    for (auto& g : groups) for (auto e : g.ev) if (e) cudaEventDestroy(e);
    for (auto& b : batches) if (b.ready) cudaEventDestroy(b.ready);
    for (auto e : free_events_) cudaEventDestroy(e);
    for (auto e : free_tevents_) cudaEventDestroy(e);
    for (auto& b : bufs_) {
        for (auto e : b.pending) cudaEventDestroy(e);
        cudaFree(b.base);
    }
    for (auto& r : raws_) cudaFree(r.ptr);
    if (raw_pool_ != nullptr) cudaMemPoolDestroy(raw_pool_);
    if (stamp_host_) cudaFreeHost(stamp_host_);
    if (stamp_cnt_) cudaFree(stamp_cnt_);
    if (csum_) cudaFree(csum_);
    if (fg_box_) cudaFree(fg_box_);
    if (fg_offs_) cudaFree(fg_offs_);
    if (out_tab_) cudaFree(out_tab_);
    for (auto s : streams_) cudaStreamDestroy(s);
    cudaStreamDestroy(seal_stream);
    cudaStreamDestroy(aux_stream);
    for (auto ss : side_streams_) cudaStreamDestroy(ss);
    speech_tables_destroy(speech_);
}

cudaEvent_t Context::get_event(bool timed) {
    auto& pool = timed ? free_tevents_ : free_events_;
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cuda_check(timed ? cudaEventCreate(&e) : cudaEventCreateWithFlags(&e, cudaEventDisableTiming),
               "cudaEventCreate");
    return e;
}

void Context::put_event(cudaEvent_t e, bool timed) { (timed ? free_tevents_ : free_events_).push_back(e); }

int Context::get_stream() {
    if (serial) return 0;   // stream 0 is reserved for serial (roofline) mode
    if (!free_streams_.empty()) {
        int i = free_streams_.back();
        free_streams_.pop_back();
        return i;
    }
    cudaStream_t s;
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    streams_.push_back(s);
    return static_cast<int>(streams_.size()) - 1;
}

// ------------------------------------------------------------------ chains
namespace {
int rank_of(int kind, Family& fam) {
    switch (kind) {
        case LFG_OP_RANDOM_CROP: fam = FAM_IMG3D; return 1;
        case LFG_OP_RANDOM_ZOOM3D: fam = FAM_IMG3D; return 2;
        case LFG_OP_RANDOM_FLIP: fam = FAM_IMG3D; return 3;
        case LFG_OP_RANDOM_BRIGHTNESS: fam = FAM_IMG3D; return 4;
        case LFG_OP_RANDOM_CONTRAST: fam = FAM_IMG3D; return 5;
        case LFG_OP_GAUSSIAN_NOISE: fam = FAM_IMG3D; return 6;
        case LFG_OP_CAST: fam = FAM_IMG3D; return 7;
        case LFG_OP_RESIZE: fam = FAM_RRC2D; return 1;
        case LFG_OP_RANDOM_HFLIP: fam = FAM_RRC2D; return 2;
        case LFG_OP_TO_TENSOR: fam = FAM_RRC2D; return 3;
        case LFG_OP_NORMALIZE: fam = FAM_RRC2D; return 4;
        case LFG_OP_PAD: fam = FAM_SPEECH; return 1;
        case LFG_OP_SPEC_AUGMENT: fam = FAM_SPEECH; return 2;
        case LFG_OP_FILTER_BANK: fam = FAM_SPEECH; return 3;
        case LFG_OP_FRAME_SPLICING: fam = FAM_SPEECH; return 4;
        case LFG_OP_PERMUTE_AUDIO: fam = FAM_SPEECH; return 5;
        default: return -1;
    }
}
double pdef(double v, double d) { return v != 0.0 ? v : d; }
}  // namespace

Chain* Context::chain_create(const lfg_op* ops, int n) {
    if (ops == nullptr || n < 1) fail(LFG_ERR_INVALID, "chain needs >= 1 op");
    auto c = std::make_unique<Chain>();
    c->ops.assign(ops, ops + n);
    int last_rank = 0;
    int first_tf = -1, last_tf = -1;
    bool has_anchor = false, has_norm = false;
    for (int i = 0; i < n; ++i) {
        const lfg_op& o = ops[i];
        if (!(o.size_factor > 0.0)) fail(LFG_ERR_INVALID, "op size_factor must be > 0");
        if (o.kind == LFG_OP_SPIN) {
            if (c->n_spin >= 4) fail(LFG_ERR_UNSUPPORTED, "at most 4 spin ops per chain");
            c->n_spin++;
            continue;
        }
        Family f = FAM_NONE;
        const int rk = rank_of(o.kind, f);
        if (rk < 0) fail(LFG_ERR_INVALID, "unknown op kind " + std::to_string(o.kind));
        if (c->fam != FAM_NONE && c->fam != f) fail(LFG_ERR_UNSUPPORTED, "ops from two chain families");
        c->fam = f;
        if (rk <= last_rank) {
            fail(LFG_ERR_UNSUPPORTED,
                 "op order not fusable (the fused kernel applies the reference chain order)");
        }
        last_rank = rk;
        if (first_tf < 0) first_tf = i;
        last_tf = i;
        const double* p = o.param;
        switch (o.kind) {
            case LFG_OP_RANDOM_CROP:
                for (int a = 0; a < 3; ++a) c->crop[a] = p[a] > 0 ? static_cast<int>(p[a]) : 128;
                if (p[3] < 0 || p[3] > 1) fail(LFG_ERR_INVALID, "RandomCrop foreground probability must be in [0, 1]");
                c->has_fg = p[3] > 0;
                c->p_fg = p[3];
                has_anchor = true;
                break;
            case LFG_OP_RANDOM_FLIP: c->p_flip = p[0]; break;
            case LFG_OP_RANDOM_BRIGHTNESS:
                c->p_bright = p[0];
                c->b_lo = pdef(p[1], 0.7);
                c->b_hi = pdef(p[2], 1.3);
                break;
            case LFG_OP_GAUSSIAN_NOISE:
                c->p_noise = p[0];
                c->noise_max = pdef(p[1], 0.1);
                break;
            case LFG_OP_RANDOM_ZOOM3D:
                c->has_zoom = true;
                c->p_zoom = p[0];
                c->z_lo = pdef(p[1], 0.8);
                c->z_hi = pdef(p[2], 1.2);
                if (!(c->z_lo > 0 && c->z_hi >= c->z_lo && c->z_hi <= 2.0))
                    fail(LFG_ERR_INVALID, "RandomZoom3D range must satisfy 0 < lo <= hi <= 2");
                break;
            case LFG_OP_RANDOM_CONTRAST:
                c->has_contrast = true;
                c->p_contrast = p[0];
                c->c_lo = pdef(p[1], 0.75);
                c->c_hi = pdef(p[2], 1.25);
                break;
            case LFG_OP_CAST: break;
            case LFG_OP_RESIZE:
                c->oh = p[0] > 0 ? static_cast<int>(p[0]) : 224;
                c->ow = p[1] > 0 ? static_cast<int>(p[1]) : 224;
                c->scale_lo = pdef(p[2], 0.08);
                c->scale_hi = pdef(p[3], 1.0);
                c->ratio_lo = pdef(p[4], 3.0 / 4.0);
                c->ratio_hi = pdef(p[5], 4.0 / 3.0);
                has_anchor = true;
                break;
            case LFG_OP_RANDOM_HFLIP: c->p_hflip = p[0]; break;
            case LFG_OP_TO_TENSOR: c->to_tensor = true; break;
            case LFG_OP_NORMALIZE:
                for (int k = 0; k < 3; ++k) {
                    c->mean[k] = p[k];
                    c->std[k] = p[3 + k];
                    if (!(c->std[k] > 0)) fail(LFG_ERR_INVALID, "normalize std must be > 0");
                }
                has_norm = true;
                break;
            case LFG_OP_PAD: break;
            case LFG_OP_SPEC_AUGMENT:
                c->n_fmask = static_cast<int>(p[0]);
                c->fmask_max = static_cast<int>(p[1]);
                c->n_tmask = static_cast<int>(p[2]);
                c->tmask_frac = p[3];
                if (c->n_fmask < 0 || c->n_fmask > 2 || c->n_tmask < 0 || c->n_tmask > 10)
                    fail(LFG_ERR_UNSUPPORTED, "SpecAugment supports <= 2 freq and <= 10 time masks");
                break;
            case LFG_OP_FILTER_BANK:
                if ((p[0] != 0 && p[0] != 512) || (p[1] != 0 && p[1] != 320) ||
                    (p[2] != 0 && p[2] != 160) || (p[3] != 0 && p[3] != 80))
                    fail(LFG_ERR_UNSUPPORTED, "FilterBank kernel is built for n_fft 512, win 320, hop 160, 80 mels");
                if (p[4] > 0) c->max_L = static_cast<int64_t>(p[4]);
                // param[5]: the waveform's sample type, LFG_DT_F32 (0 = default) or LFG_DT_I16
                // (16-bit PCM, the reference's speech bytes_in = 2 B per sample,
                // workloads.cpp:115; converted on the device as s / 32768, exactly)
                if (p[5] != 0 && p[5] != LFG_DT_F32 && p[5] != LFG_DT_I16)
                    fail(LFG_ERR_UNSUPPORTED, "FilterBank input type must be LFG_DT_F32 or LFG_DT_I16");
                c->wav_bytes = p[5] == LFG_DT_I16 ? 2 : 4;
                has_anchor = true;
                break;
            case LFG_OP_FRAME_SPLICING:
                c->stack = p[0] > 0 ? static_cast<int>(p[0]) : 3;
                break;
            case LFG_OP_PERMUTE_AUDIO: break;
        }
    }
    if (c->fam == FAM_NONE) fail(LFG_ERR_UNSUPPORTED, "chain has no device transform");
    if (!has_anchor) {
        fail(LFG_ERR_UNSUPPORTED,
             "chain must contain its shape-defining op (RandomCrop / Resize / FilterBank)");
    }
    if (has_norm && c->fam == FAM_RRC2D && !c->to_tensor) {
        fail(LFG_ERR_UNSUPPORTED, "Normalize requires ToTensor before it");
    }
    if (c->fam == FAM_IMG3D) {
        for (int a = 0; a < 3; ++a)
            if (c->crop[a] < 1 || c->crop[a] > 1024) fail(LFG_ERR_INVALID, "crop out of range");
        if (c->crop[2] % 4 != 0) fail(LFG_ERR_UNSUPPORTED, "crop width must be a multiple of 4");
        const int64_t vox = int64_t(c->crop[0]) * c->crop[1] * c->crop[2];
        c->nplanes = 2;
        c->plane_bytes[0] = vox * 4;
        c->plane_bytes[1] = ((vox + 15) / 16) * 16;
    } else if (c->fam == FAM_RRC2D) {
        if (c->oh < 1 || c->ow < 2 || c->ow > 256 || (c->ow & 1) || c->oh > 4096)
            fail(LFG_ERR_UNSUPPORTED, "Resize output width must be even and <= 256");
        c->nplanes = 1;
        // slot stride rounded up to 16 B: K12 gathers in 16-B words (3*oh*ow*4 is
        // 8 mod 16 when oh is odd and ow = 2 mod 4); the 3 planes fill the first
        // 3*oh*ow*4 bytes of each slot
        c->plane_bytes[0] = (int64_t(3) * c->oh * c->ow * 4 + 15) / 16 * 16;
    } else {
        bool splice = false;
        for (int i = 0; i < n; ++i) splice |= ops[i].kind == LFG_OP_FRAME_SPLICING;
        if (!splice) c->stack = 1;
        if (c->stack < 1 || speech_frames_per_cta() % c->stack != 0)
            fail(LFG_ERR_UNSUPPORTED, "FrameSplicing stack must divide 126 (1, 2, 3, 6, 7, 9, ...)");
        if (c->max_L < 2 || c->max_L > (1 << 24)) fail(LFG_ERR_INVALID, "FilterBank max length out of range");
        if (speech_ == nullptr) cuda_check(speech_tables_create(&speech_), "speech tables");
        const int64_t t_max = 1 + c->max_L / c->hop;
        const int64_t rows = (t_max + c->stack - 1) / c->stack;
        c->nplanes = 1;
        c->plane_bytes[0] = rows * c->stack * c->n_mels * 4;   // time-major [T'_max, stack * 80]
    }
    c->out_bytes = c->plane_bytes[0] + c->plane_bytes[1];
    // stages: leading spins, the fused stage (with interleaved spins), trailing spins
    int spin_slot = 0;
    for (int i = 0; i < n; ++i) {
        if (ops[i].kind == LFG_OP_SPIN && (i < first_tf || i > last_tf)) {
            Stage s{ST_SPIN, i, i + 1, {spin_slot++}};
            c->stages.push_back(s);
        } else if (i == first_tf) {
            Stage s{c->fam == FAM_IMG3D ? ST_IMG3D : (c->fam == FAM_RRC2D ? ST_RRC2D : ST_SPEECH),
                    first_tf, last_tf + 1, {}};
            for (int k = first_tf; k <= last_tf; ++k)
                if (ops[k].kind == LFG_OP_SPIN) s.spin_ops.push_back(spin_slot++);
            c->stages.push_back(s);
            i = last_tf;
        }
    }
    c->spin_last = c->stages.back().kind == ST_SPIN || !c->stages.back().spin_ops.empty();
    chains_.push_back(std::move(c));
    reserve_bufs(chains_.back().get());
    return chains_.back().get();
}

void Context::chain_destroy(Chain* c) {
    for (auto& g : groups) {
        if (g.chain != c || g.complete || poll_group(g)) continue;
        // a group whose samples all completed (stamps) may still be retiring its last
        // kernel: wait for it; a group with unfinished samples is a caller error
        bool ready = g.launched;
        for (int64_t t : g.tickets) ready = ready && sample_ready(t);
        if (!ready) fail(LFG_ERR_STATE, "chain has samples in flight");
        cuda_check(cudaEventSynchronize(g.ev.back()), "group completion");
        poll_group(g);
    }
    for (size_t i = 0; i < chains_.size(); ++i) {
        if (chains_[i].get() == c) {
            open_buf_.erase(c);
            open_group_[0].erase(c);
            open_group_[1].erase(c);
            // orphan the chain's buffers: a later chain may be allocated at the
            // same address, so buffers must never be matched by a stale pointer
            for (auto& b : bufs_) {
                if (b.chain != c) continue;
                b.chain = nullptr;
                b.open = false;
                b.assigned = b.live = 0;
            }
            chains_.erase(chains_.begin() + static_cast<long>(i));
            return;
        }
    }
    fail(LFG_ERR_INVALID, "unknown chain");
}

// ------------------------------------------------------------------ slot buffers
bool Context::buf_reusable(SlotBuf& b) {
    if (b.open || b.in_batch || b.live > 0) return false;
    while (!b.pending.empty()) {
        cudaError_t q = cudaEventQuery(b.pending.back());
        if (q == cudaErrorNotReady) return false;
        cuda_check(q, "pending event");
        put_event(b.pending.back());
        b.pending.pop_back();
    }
    return true;
}

bool Context::chain_alive(const Chain* c) const {
    for (auto& ch : chains_)
        if (ch.get() == c) return true;
    return false;
}

// All output buffers of a chain are created when the chain is (the shard loop
// never allocates): max_slot_buffers sample-slot buffers plus max_slot_buffers
// gather (collation target) buffers, bounded separately so stragglers pinning
// slot buffers can never starve a seal of its destination.  Idle buffers of
// destroyed chains are recycled first.
void Context::reserve_bufs(const Chain* c) {
    const int64_t need = static_cast<int64_t>(cfg.batch_size) * c->out_bytes;
    for (int role = 0; role < 2; ++role) {
        int have = 0;
        for (auto& b : bufs_) {
            if (have >= cfg.max_slot_buffers) break;
            if (b.gather_role != (role == 1) || chain_alive(b.chain)) continue;
            if (b.bytes < need || !buf_reusable(b)) continue;
            b.chain = c;
            b.cap = cfg.batch_size;
            b.assigned = b.live = 0;
            b.open = b.in_batch = false;
            ++have;
        }
        for (; have < cfg.max_slot_buffers; ++have) {
            SlotBuf b;
            cuda_check(cudaMalloc(&b.base, static_cast<size_t>(need)), "cudaMalloc(output buffer)");
            b.cap = cfg.batch_size;
            b.chain = c;
            b.bytes = need;
            b.gather_role = role == 1;
            bufs_.push_back(b);
        }
    }
    sync_out_tab();
}

// The device table of slot-buffer bases (K3's packed descriptors name a buffer by
// its index); rewritten whenever buffers are created -- at chain creation, never
// inside the shard loop.
void Context::sync_out_tab() {
    if (bufs_.size() > static_cast<size_t>(kMaxRrcBufs))
        fail(LFG_ERR_UNSUPPORTED, "more than 4096 output buffers in one context");
    if (out_tab_ == nullptr)
        cuda_check(cudaMalloc(&out_tab_, kMaxRrcBufs * sizeof(float*)), "output buffer table");
    std::vector<float*> h(bufs_.size());
    for (size_t i = 0; i < bufs_.size(); ++i) h[i] = reinterpret_cast<float*>(bufs_[i].base);
    cuda_check(cudaMemcpy(out_tab_, h.data(), h.size() * sizeof(float*), cudaMemcpyHostToDevice),
               "output buffer table");
}

// Round-robin from the buffer after the last one handed out: the oldest
// buffer is the likeliest to be free, so usually the first candidate is taken
// after at most one event query (a full scan with queries costs microseconds).
int Context::alloc_buf(const Chain* c, bool for_batch) {
    const size_t nb = bufs_.size();
    size_t& cur = alloc_cursor_[for_batch ? 1 : 0];
    for (size_t k = 0; k < nb; ++k) {
        const size_t i = (cur + 1 + k) % nb;
        SlotBuf& b = bufs_[i];
        if (b.gather_role != for_batch || b.chain != c) continue;
        if (buf_reusable(b)) {
            b.assigned = 0;
            b.live = 0;
            b.open = !for_batch;
            b.in_batch = for_batch;
            cur = i;
            return static_cast<int>(i);
        }
    }
    fail(LFG_ERR_AGAIN, "all output buffers are in use (consume or release batches)");
}

void Context::assign_slot(Ticket& t, const Chain* c) {
    auto it = open_buf_.find(c);
    int bi = it == open_buf_.end() ? -1 : it->second;
    if (bi < 0 || !bufs_[bi].open || bufs_[bi].assigned >= bufs_[bi].cap) {
        if (bi >= 0) bufs_[bi].open = false;
        bi = alloc_buf(c, false);
        open_buf_[c] = bi;
    }
    SlotBuf& b = bufs_[bi];
    t.buf = bi;
    t.pos = b.assigned++;
    b.live++;
    if (b.assigned == b.cap) {
        b.open = false;
        open_buf_.erase(c);
    }
}

char* Context::slot_ptr(const Ticket& t, int plane) const {
    const SlotBuf& b = bufs_[t.buf];
    const Chain* c = b.chain;
    const int64_t plane_off = plane == 0 ? 0 : static_cast<int64_t>(b.cap) * c->plane_bytes[0];
    return b.base + plane_off + static_cast<int64_t>(t.pos) * c->plane_bytes[plane];
}

// ------------------------------------------------------------------ raw staging
// Raw staging buffers (pinned-host groups) are pooled.  A new buffer is stream-ordered
// (cudaMallocAsync on the group's stream: unlike cudaMalloc it never synchronises the
// device, which would stall every in-flight group) and sized with headroom, so groups a
// little larger than the pooled buffers do not allocate again.
int64_t Context::get_raw(int64_t bytes, cudaStream_t st) {
    int64_t best = -1;
    for (size_t k = 0; k < free_raws_.size(); ++k) {
        const int64_t i = free_raws_[k];
        if (raws_[i].cap >= bytes && (best < 0 || raws_[i].cap < raws_[best].cap)) best = i;
    }
    if (best >= 0) {
        free_raws_.erase(std::find(free_raws_.begin(), free_raws_.end(), best));
        return best;
    }
    RawBuf r;
    constexpr int64_t kRound = int64_t(4) << 20;
    r.cap = (std::max<int64_t>(bytes + bytes / 4, int64_t(8) << 20) + kRound - 1) / kRound * kRound;
    static const bool trace = std::getenv("LFG_SHARD_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (raw_pool_ == nullptr) {
        // The context's own stream-ordered pool (the device's default pool and its
        // settings stay untouched).  Growing a pool maps physical memory (~1 ms per
        // 64 MB): at the first staged group it is grown once for every launch-group
        // stream and kept (release threshold: never), so later groups -- inside a timed
        // run -- carve their buffers from memory the pool already holds.
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = cfg.device;
        cuda_check(cudaMemPoolCreate(&raw_pool_, &props), "raw staging pool");
        uint64_t keep = UINT64_MAX;
        cuda_check(cudaMemPoolSetAttribute(raw_pool_, cudaMemPoolAttrReleaseThreshold, &keep), "pool threshold");
        void* prime = nullptr;
        const size_t total = static_cast<size_t>(r.cap) * static_cast<size_t>(std::min(stream_pool, 32));
        if (cudaMallocFromPoolAsync(&prime, total, raw_pool_, st) == cudaSuccess) cudaFreeAsync(prime, st);
        else cudaGetLastError();   // (not enough free HBM to hold it all: grow on demand)
    }
    cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&r.ptr), static_cast<size_t>(r.cap), raw_pool_, st),
               "cudaMallocFromPoolAsync(raw staging)");
    if (trace)
        std::fprintf(stderr, "[lfg trace] raw staging +%lld MB (pool %zu) in %.0f us\n",
                     static_cast<long long>(r.cap >> 20), raws_.size() + 1,
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    raws_.push_back(r);
    return static_cast<int64_t>(raws_.size()) - 1;
}

static int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

// Algorithmic bytes of K1 / K4 for one sample: the window voxels inside the
// source, read once (f32 + u8), and the crop written (f32 + u8).  Without
// RandomZoom3D the window is the crop: 128^3 * 10 B.
int64_t img3d_algo_bytes(const Chain& c, const Ticket& t) {
    if (!c.has_zoom) return c.algo_bytes_per_sample(t.desc());
    int64_t in = 5;
    for (int a = 0; a < 3; ++a)
        in *= std::max<int64_t>(0, std::min<int64_t>(t.p3().win[a], t.desc().dims[a] - t.p3().off[a]));
    return in + int64_t(c.crop[0]) * c.crop[1] * c.crop[2] * 5;
}

// Geometry of the bytes a sample's chain reads, as strided boxes (K0 copies
// them from pinned host memory; see kernels.h for the row-skew convention).
struct Box {
    const char* src;
    int64_t src_py, src_pz;
    int32_t row_bytes, ny, nz;
    int plane;               // 0: image / primary payload, 1: label
    int64_t dst_py() const { return 16 * ((static_cast<int64_t>(row_bytes) + 30) / 16); }
    int64_t bytes() const { return dst_py() * ny * nz; }
};

static int boxes_of(const Chain& c, const Ticket& t, Box out[2], int64_t wd[3]) {
    const lfg_sample_desc& s = t.desc();
    wd[0] = wd[1] = wd[2] = 0;
    if (c.fam == FAM_IMG3D) {
        const int64_t H = s.dims[1], W = s.dims[2];
        if (c.has_fg && t.p3().fg) {
            // a foreground-biased crop's window depends on the label scan: stage the
            // label volume only; K0w pulls the image window once K2 resolved it
            for (int a = 0; a < 3; ++a) wd[a] = s.dims[a];
            out[0] = Box{static_cast<const char*>(s.aux), W, H * W, static_cast<int32_t>(W),
                         static_cast<int32_t>(H), static_cast<int32_t>(s.dims[0]), 1};
            return 1;
        }
        for (int a = 0; a < 3; ++a) wd[a] = std::min<int64_t>(t.p3().win[a], s.dims[a] - t.p3().off[a]);
        const int64_t first = (t.p3().off[0] * H + t.p3().off[1]) * W + t.p3().off[2];
        out[0] = Box{static_cast<const char*>(s.data) + first * 4, W * 4, H * W * 4,
                     static_cast<int32_t>(wd[2] * 4), static_cast<int32_t>(wd[1]),
                     static_cast<int32_t>(wd[0]), 0};
        out[1] = Box{static_cast<const char*>(s.aux) + first, W, H * W, static_cast<int32_t>(wd[2]),
                     static_cast<int32_t>(wd[1]), static_cast<int32_t>(wd[0]), 1};
        return 2;
    }
    if (c.fam == FAM_RRC2D) {
        const int64_t W = s.dims[1];
        out[0] = Box{static_cast<const char*>(s.data) + (t.p2().top * W + t.p2().left) * 3, W * 3, 0,
                     static_cast<int32_t>(t.p2().w * 3), static_cast<int32_t>(t.p2().h), 1, 0};
        return 1;
    }
    out[0] = Box{static_cast<const char*>(s.data), 0, 0, static_cast<int32_t>(s.dims[0] * c.wav_bytes), 1, 1, 0};
    return 1;
}

// a foreground-crop sample's compact window (K0w): image rows padded to 4 floats,
// label rows to 16 bytes
static int64_t fg_window_bytes(const Params3D& p) {
    const int64_t rows = p.win[0] * p.win[1];
    return align256(4 * rows * ((p.win[2] + 3) / 4 * 4)) + align256(rows * ((p.win[2] + 15) / 16 * 16));
}

int64_t Context::stage_raw_bytes(const Chain& c, const Ticket& t) const {
    Box b[2];
    int64_t wd[3];
    const int nb = boxes_of(c, t, b, wd);
    int64_t total = 0;
    for (int i = 0; i < nb; ++i) total += align256(b[i].bytes());
    if (c.fam == FAM_IMG3D && c.has_fg && t.p3().fg) total += fg_window_bytes(t.p3());
    return total;
}

// ------------------------------------------------------------------ submit
void draw_params(const Chain& c, uint64_t seed, const lfg_sample_desc& s, PreDraw& out) {
    if (c.fam == FAM_IMG3D) {
        out.p3 = Params3D{};
        draw_3d(c, seed, s.id, s.dims, out.p3);
    } else if (c.fam == FAM_RRC2D) {
        out.p2 = Params2D{};
        draw_2d(c, seed, s.id, s.dims[0], s.dims[1], out.p2);
    } else {
        out.ps = ParamsSp{};
        draw_sp(c, seed, s.id, s.dims[0], out.ps);
    }
}

int64_t Context::submit(Chain* c, const lfg_sample_desc& s, const PreDraw* pre) {
    if (c == nullptr) fail(LFG_ERR_INVALID, "null chain");
    if (s.data == nullptr) fail(LFG_ERR_INVALID, "sample has no payload");
    if (s.src_kind != LFG_SRC_DEVICE && s.src_kind != LFG_SRC_HOST_PINNED)
        fail(LFG_ERR_INVALID, "bad src_kind");
    if (c->fam == FAM_IMG3D) {
        if (s.ndim != 3 || s.aux == nullptr) fail(LFG_ERR_INVALID, "img_seg sample needs a D,H,W volume and a label");
        for (int a = 0; a < 3; ++a)
            if (s.dims[a] < 1 || s.dims[a] > (1 << 20)) fail(LFG_ERR_INVALID, "volume dims out of range");
    } else if (c->fam == FAM_RRC2D) {
        if (s.ndim != 3 || s.dims[2] != 3 || s.dims[0] < 1 || s.dims[1] < 1 || s.dims[0] > 65535 ||
            s.dims[1] > 65535)
            fail(LFG_ERR_INVALID, "obj_det sample needs an H,W,3 image (H, W <= 65535)");
    } else {
        // reflect padding by n_fft/2 needs L > n_fft/2 (torch.stft center=True has the same rule)
        if (s.ndim != 1 || s.dims[0] < c->n_fft / 2 + 1 || s.dims[0] > c->max_L)
            fail(LFG_ERR_INVALID, "speech sample needs a waveform of length in [n_fft/2 + 1, max_L]");
        if (reinterpret_cast<uintptr_t>(s.data) % static_cast<uintptr_t>(c->wav_bytes) != 0)
            fail(LFG_ERR_INVALID, "waveform pointer is not aligned to its sample type");
    }
    if (s.src_kind == LFG_SRC_HOST_PINNED) {
        // K0 reads the payload over PCIe through its UVA mapping: it must be pinned
        for (const void* p : {s.data, s.aux}) {
            if (p == nullptr) continue;
            // a page that held a validated pinned address stays pinned while the caller's
            // buffer lives (allocations are page-granular): one driver query per page
            const uintptr_t page = reinterpret_cast<uintptr_t>(p) >> 12;
            if (pinned_pages_.count(page)) continue;
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeHost) {
                cudaGetLastError();
                fail(LFG_ERR_INVALID, "LFG_SRC_HOST_PINNED payload is not pinned host memory");
            }
            if (pinned_pages_.size() > (size_t(1) << 20)) pinned_pages_.clear();
            pinned_pages_.insert(page);
        }
    }
    for (int k = 0; k < c->n_spin; ++k)
        if (s.spin_us[k] < 0) fail(LFG_ERR_STATE, "negative transform cost");  // balancer.cpp:16
    // Tickets point at the sample's descriptor and drawn parameters.  The shard
    // runner passes its run arrays (they outlive the run's tickets); a sample
    // submitted through the ABI is copied into context-owned storage.
    const lfg_sample_desc* sp = &s;
    bool owned = false;
    if (pre == nullptr) {
        owned_.emplace_back();
        owned_.back().first = s;
        draw_params(*c, cfg.seed, s, owned_.back().second);
        sp = &owned_.back().first;
        pre = &owned_.back().second;
        owned = true;
    }
    // the ticket is built in place (submit runs once per sample)
    const int64_t ti = static_cast<int64_t>(tickets.size());
    // its completion stamp slot (ticket index mod the ring) must be free: the ticket
    // that used it last, kStampSlots earlier, has finished
    if (ti >= kStampSlots && !groups[tickets[ti - kStampSlots].group].complete &&
        !poll_group(groups[tickets[ti - kStampSlots].group]))
        fail(LFG_ERR_AGAIN, "completion stamp ring full (a sample 2^20 submissions old is still running)");
    if (c->spin_last || stamp_transforms) stamp_host_[ti & (kStampSlots - 1)] = 0;
    tickets.emplace_back();
    Ticket& t = tickets.back();
    t.id = s.id;
    t.dp = sp;
    t.pp = pre;
    try {
        assign_slot(t, c);
    } catch (...) {
        tickets.pop_back();
        if (owned) owned_.pop_back();
        throw;
    }
    auto& og = open_group_[s.src_kind == LFG_SRC_DEVICE ? 0 : 1];
    auto it = og.find(c);
    int64_t gi;
    if (it == og.end()) {
        gi = static_cast<int64_t>(groups.size());
        groups.emplace_back();
        Group& ng = groups.back();
        ng.id = gi;
        ng.chain = c;
        ng.src_kind = s.src_kind;
        ng.tickets.reserve(static_cast<size_t>(std::max(1, cfg.max_group)));
        if (cfg.coalesce_us > 0) ng.t_open_us = host_now_us();
        og[c] = gi;
    } else {
        gi = it->second;
    }
    t.group = gi;
    t.idx = static_cast<int>(groups[gi].tickets.size());
    Group& g = groups[gi];
    g.tickets.push_back(ti);
    g.refs++;
    counters.submitted++;
    const int cap = c->fam == FAM_IMG3D ? kMax3D : (c->fam == FAM_RRC2D ? kMax2D : kMaxSp);
    if (static_cast<int>(g.tickets.size()) >= std::min(cfg.max_group, cap)) {
        og.erase(c);
        if (defer_launch) deferred_.push_back(gi);
        else launch_group(g);
    }
    return ti;
}

int64_t Context::open_group_count() const {
    return static_cast<int64_t>(open_group_[0].size() + open_group_[1].size());
}

bool Context::recycle_tables() {
    if (!deferred_.empty() || open_group_count() != 0) return false;
    for (const Group& g : groups)
        if (!g.complete || g.refs != 0) return false;
    for (const Ticket& t : tickets)
        if (!t.released) return false;
    tickets.clear();
    groups.clear();
    owned_.clear();
    return true;
}

void Context::flush() {
    for (int64_t gi : deferred_) launch_group(groups[gi]);
    deferred_.clear();
    for (auto& og : open_group_) {
        for (auto& kv : og) launch_group(groups[kv.second]);
        og.clear();
    }
}

void Context::flush_due() {
    if (cfg.coalesce_us <= 0) {
        flush();
        return;
    }
    for (int64_t gi : deferred_) launch_group(groups[gi]);
    deferred_.clear();
    const int64_t now = host_now_us();
    for (auto& og : open_group_) {
        std::vector<const Chain*> due;
        for (auto& kv : og)
            if (now - groups[kv.second].t_open_us >= cfg.coalesce_us) due.push_back(kv.first);
        for (const Chain* c : due) {
            const int64_t gi = og.find(c)->second;
            og.erase(c);
            launch_group(groups[gi]);
        }
    }
}

// Roofline timing of a chain's transform kernels: all samples are submitted
// first (launches deferred), then every launch group is issued back to back on
// one stream behind a device-side gate, so the per-stage CUDA events bracket kernel
// time only -- no host submission gaps or launch-call time.  Returns the mean device time of one transform-stage launch.
void Context::time_kernels(Chain* c, const lfg_sample_desc* s, int n, double* mean_ms,
                           int64_t* launches, int64_t* bytes, int64_t* flops) {
    if (n < 1) fail(LFG_ERR_INVALID, "no samples to time");
    const int64_t fit = int64_t(cfg.max_slot_buffers - 1) * cfg.batch_size;
    if (n > fit) n = static_cast<int>(fit);
    cuda_check(cudaDeviceSynchronize(), "sync");
    const lfg_counters c0 = counters;
    const bool timed0 = time_groups;
    time_groups = true;
    serial = true;
    defer_launch = true;
    std::vector<int64_t> ts;
    try {
        for (int i = 0; i < n; ++i) ts.push_back(submit(c, s[i]));
        for (auto& og : open_group_) {
            for (auto& kv : og)
                if (groups[kv.second].chain == c) deferred_.push_back(kv.second);
            og.erase(c);
        }
        defer_launch = false;
        // Hold stream 0 with a device spin while the host issues the groups: each stage's
        // start event then fires when the previous launch ends instead of when the host
        // gets to it, so the events bracket the kernel and not the host's launch call
        // (the 256-image K3 launch prepares ~20-40 us of descriptors on the host and its
        // launch call costs ~8 us with the large parameter block).  The spin is sized well
        // above the host's issue time; it sits outside every stage's events.
        const int64_t gate_ns = 500'000 + 250'000 * static_cast<int64_t>(deferred_.size());
        cuda_check(launch_trainer_spin(std::min<int64_t>(gate_ns, 50'000'000), 1, streams_[0]), "timing gate");
        flush();
    } catch (...) {
        serial = defer_launch = false;
        time_groups = timed0;
        throw;
    }
    serial = false;
    time_groups = timed0;
    cuda_check(cudaDeviceSynchronize(), "sync");
    double ms = 0;
    int64_t nl = 0;
    std::vector<int64_t> seen;
    for (int64_t t : ts) {
        Group& g = groups[tickets[t].group];
        if (std::find(seen.begin(), seen.end(), g.id) != seen.end()) continue;
        seen.push_back(g.id);
        poll_group(g);
        for (size_t k = 0; k < c->stages.size(); ++k)
            if (c->stages[k].kind != ST_SPIN) {
                ms += g.stage_ms[k];
                ++nl;
            }
    }
    for (int64_t t : ts) ticket_release(t);
    *mean_ms = nl ? ms / nl : 0.0;
    *launches = nl;
    *bytes = counters.kernel_bytes - c0.kernel_bytes;
    *flops = counters.reserved[1] - c0.reserved[1];
}

void Context::launch_group(Group& g) {
    const auto t_enter = std::chrono::steady_clock::now();
    const Chain& c = *g.chain;
    g.stream_idx = get_stream();
    g.stream = streams_[g.stream_idx];
    const int nst = static_cast<int>(c.stages.size());
    g.ev.resize(nst + 1);
    g.timed = time_groups;
    for (auto& e : g.ev) e = get_event(g.timed);
    cudaStream_t st = g.stream;
    // The start event goes in immediately before the group's first device
    // operation, after the host has built that operation's parameters: stage
    // times (timeout classification, the roofline) then measure device work,
    // not host-side launch preparation (TMA map encoding, descriptor fills).
    bool started = false;
    auto start = [&] {
        if (!started) {
            if (g.timed) cuda_check(cudaEventRecord(g.ev[0], st), "record start");
            started = true;
        }
    };
    const int n = static_cast<int>(g.tickets.size());
    const bool staged = g.src_kind == LFG_SRC_HOST_PINNED;
    auto lap = [&](double& acc, std::chrono::steady_clock::time_point& t0) {
        if (!prof_on) return;
        const auto t1 = std::chrono::steady_clock::now();
        acc += std::chrono::duration<double, std::nano>(t1 - t0).count();
        t0 = t1;
    };
    auto t_lap = std::chrono::steady_clock::now();

    // Host-pinned payloads: K0 pulls exactly the boxes the chain reads over
    // PCIe into one staging buffer (part of the group's first stage).
    struct View {
        const char* p[2];
        int64_t py[2], pz[2];
        int32_t sk0[2], sky[2], skz[2];
        int64_t sdim[3], off[3];
    };
    // per-thread scratch: no allocation or clearing per group
    static thread_local std::vector<View> views;
    if (static_cast<int>(views.size()) < n) views.resize(static_cast<size_t>(n));
    if (staged) {
        int64_t total = 0;
        for (int i = 0; i < n; ++i) total += stage_raw_bytes(c, tickets[g.tickets[i]]);
        g.raw_idx = get_raw(total, st);
        char* dst = raws_[g.raw_idx].ptr;
        StageLaunch SL{};
        for (int i = 0; i < n; ++i) {
            Ticket& t = tickets[g.tickets[i]];
            View& v = views[i];
            Box b[2];
            int64_t wd[3];
            const int nb = boxes_of(c, t, b, wd);
            v.p[0] = v.p[1] = nullptr;
            for (int k = 0; k < nb; ++k) {
                const int pl = b[k].plane;
                StageDesc& d = SL.d[SL.n++];
                d.src = b[k].src;
                d.dst = dst;
                d.src_py = b[k].src_py;
                d.src_pz = b[k].src_pz;
                d.dst_py = b[k].dst_py();
                d.dst_pz = b[k].dst_py() * b[k].ny;
                d.row_bytes = b[k].row_bytes;
                d.ny = b[k].ny;
                d.nz = b[k].nz;
                const uintptr_t sa = reinterpret_cast<uintptr_t>(b[k].src);
                const int esz = (c.fam == FAM_IMG3D && pl == 0) ? 4 : 1;  // skew unit
                v.p[pl] = dst;
                v.py[pl] = d.dst_py / esz;
                v.pz[pl] = d.dst_pz / esz;
                v.sk0[pl] = static_cast<int32_t>((sa & 15) / esz);
                v.sky[pl] = static_cast<int32_t>((b[k].src_py & 15) / esz);
                v.skz[pl] = static_cast<int32_t>((b[k].src_pz & 15) / esz);
                counters.h2d_bytes += static_cast<int64_t>(b[k].row_bytes) * b[k].ny * b[k].nz;
                dst += align256(b[k].bytes());
            }
            if (c.fam == FAM_SPEECH) {
                // a waveform is one K0 row (read over PCIe with the group's other
                // boxes in the same launch); the kernel reads it at its skew
                v.p[0] += v.sk0[0];
                continue;
            }
            const bool whole = c.fam == FAM_IMG3D && c.has_fg && t.p3().fg;   // see boxes_of
            if (whole) {   // the K0w compact window follows the staged label volume
                v.p[0] = dst;
                v.py[0] = v.pz[0] = 0;
                v.sk0[0] = v.sky[0] = v.skz[0] = 0;
                dst += fg_window_bytes(t.p3());
            }
            for (int a = 0; a < 3; ++a) {
                v.sdim[a] = wd[a];
                v.off[a] = whole ? t.p3().off[a] : 0;
            }
        }
        if (SL.n > 0) {
            start();
            cuda_check(launch_stage(SL, st), "stage launch");
            counters.launches++;
        }
    } else if (c.fam != FAM_RRC2D) {   // (obj_det reads its HBM-resident boxes straight from the tickets)
        for (int i = 0; i < n; ++i) {
            Ticket& t = tickets[g.tickets[i]];
            View& v = views[i];
            std::memset(&v, 0, sizeof(v));
            const lfg_sample_desc& s = t.desc();
            if (c.fam == FAM_IMG3D) {
                v.p[0] = static_cast<const char*>(s.data);
                v.p[1] = static_cast<const char*>(s.aux);
                v.py[0] = v.py[1] = s.dims[2];
                v.pz[0] = v.pz[1] = s.dims[1] * s.dims[2];
                for (int a = 0; a < 3; ++a) {
                    v.sdim[a] = s.dims[a];
                    v.off[a] = t.p3().off[a];
                }
            } else {
                v.p[0] = static_cast<const char*>(s.data);
            }
        }
    }

    // The group's last kernel carries the per-sample completion stamps.
    const StampRef stamps{stamp_cnt_, stamp_dev_};
    const auto slot_of = [&](int i) { return static_cast<int32_t>(g.tickets[i] & (kStampSlots - 1)); };
    g.stamped = c.spin_last || stamp_transforms;
    g.got.assign(static_cast<size_t>(n), 0);
    g.n_got = g.scan_from = 0;
    g.part_ev = nullptr;
    g.part_idx.clear();
    g.part_done = g.part_handed = false;
    g.part_ms = 0.0f;
    lap(prof_views_ns, t_lap);
    auto launch_spins = [&](int slot, bool stamp) {
        SpinLaunch L{};
        L.n = n;
        for (int i = 0; i < n; ++i) L.ns[i] = tickets[g.tickets[i]].desc().spin_us[slot] * 1000;
        if (stamp) {
            L.st = stamps;
            for (int i = 0; i < n; ++i) L.slot[i] = slot_of(i);
        }
        start();
        cuda_check(launch_spin(L, st), "spin launch");
        counters.launches++;
    };

    for (int s = 0; s < nst; ++s) {
        const Stage& S = c.stages[s];
        // this stage's transform kernel is the group's last kernel (and stamps)
        const bool stamp_here = s == nst - 1 && S.spin_ops.empty() && stamp_transforms;
        if (S.kind == ST_SPIN) {
            launch_spins(S.spin_ops[0], s == nst - 1);
        } else if (S.kind == ST_IMG3D) {
            Img3dLaunch L{};
            if (stamp_here) L.st = stamps;
            for (int a = 0; a < 3; ++a) L.crop[a] = c.crop[a];
            L.n = n;
            // TMA tile path: HBM-resident volumes with 16-B aligned rows
            bool tma = !staged && img3d_tma_ && !c.has_zoom;
            for (int i = 0; i < n && tma; ++i) {
                const lfg_sample_desc& sd = tickets[g.tickets[i]].desc();
                tma = img3d_tma_ok(sd.data, sd.aux, sd.dims, c.crop) &&
                      img3d_encode_maps(L, i, sd.data, sd.aux, sd.dims) == cudaSuccess;
            }
            L.tma = tma ? 1 : 0;
            const auto t_l = std::chrono::steady_clock::now();
            for (int i = 0; i < n; ++i) {
                Ticket& t = tickets[g.tickets[i]];
                const View& v = views[i];
                Img3dDesc& d = L.d[i];
                d.img = reinterpret_cast<const float*>(v.p[0]);
                d.lbl = reinterpret_cast<const uint8_t*>(v.p[1]);
                d.out_img = reinterpret_cast<float*>(slot_ptr(t, 0));
                d.out_lbl = reinterpret_cast<uint8_t*>(slot_ptr(t, 1));
                d.img_py = v.py[0];
                d.img_pz = v.pz[0];
                d.lbl_py = v.py[1];
                d.lbl_pz = v.pz[1];
                d.img_sk0 = v.sk0[0];
                d.img_sky = v.sky[0];
                d.img_skz = v.skz[0];
                d.lbl_sk0 = v.sk0[1];
                d.lbl_sky = v.sky[1];
                d.lbl_skz = v.skz[1];
                for (int a = 0; a < 3; ++a) {
                    d.sdim[a] = static_cast<int32_t>(v.sdim[a]);
                    d.off[a] = static_cast<int32_t>(v.off[a]);
                }
                d.flip = t.p3().flip[0] | (t.p3().flip[1] << 1) | (t.p3().flip[2] << 2);
                d.scale = static_cast<float>(t.p3().scale);
                d.sigma = static_cast<float>(t.p3().sigma);
                d.key0 = t.p3().key[0];
                d.key1 = t.p3().key[1];
                for (int a = 0; a < 3; ++a) {
                    d.win[a] = static_cast<int32_t>(t.p3().win[a]);
                    d.zscale[a] = static_cast<double>(t.p3().win[a]) / static_cast<double>(c.crop[a]);
                }
                d.contrast = static_cast<float>(t.p3().contrast);
                d.csum = nullptr;
                d.contrast_on = t.p3().contrast != 1.0;
                d.slot = slot_of(i);
                counters.kernel_bytes += img3d_algo_bytes(c, t);
            }
            // RandomContrast (K5 sums each contrasted sample's crop first) then K1 / K4
            // over the launch `Lx` (the whole group, or one part of a split group)
            auto contrast_and_transform = [&](Img3dLaunch& Lx) {
                if (c.has_contrast) {
                    int n_c = 0;
                    for (int i = 0; i < Lx.n; ++i) {
                        Img3dDesc& d = Lx.d[i];
                        if (!d.contrast_on) continue;
                        d.csum = csum_ + csum_next_;
                        csum_next_ = (csum_next_ + 1) % kCsumSlots;
                        ++n_c;
                        counters.kernel_bytes += int64_t(4) * std::min(d.win[0], d.sdim[0] - d.off[0]) *
                                                 std::min(d.win[1], d.sdim[1] - d.off[1]) *
                                                 std::min(d.win[2], d.sdim[2] - d.off[2]);
                    }
                    if (n_c > 0) {
                        start();
                        for (int i = 0; i < Lx.n; ++i)
                            if (Lx.d[i].csum != nullptr)
                                cuda_check(cudaMemsetAsync(const_cast<double*>(Lx.d[i].csum), 0, sizeof(double), st),
                                           "csum reset");
                        cuda_check(launch_img3d_mean(Lx, st), "img3d mean launch");
                        counters.launches++;
                    }
                }
                start();
                if (c.has_zoom) cuda_check(launch_img3d_zoom(Lx, st), "img3d zoom launch");
                else cuda_check(launch_img3d(Lx, st), "img3d launch");
                counters.launches++;
            };
            int n_fg = 0;
            for (int i = 0; i < n && c.has_fg; ++i) n_fg += tickets[g.tickets[i]].p3().fg != 0;
            if (n_fg == 0) {
                contrast_and_transform(L);
            } else {
                // RandomCrop foreground oversampling (K2).  The group splits: its plain
                // samples run first and complete at a sub-launch event, so they never
                // wait for the label scans; then K2 scans the label volumes of the
                // samples that drew it, resolves their window origins, and K1 / K4
                // crops them (from pinned memory K0w first pulls just those windows).
                std::vector<int> plain, fgi;
                for (int i = 0; i < n; ++i) (tickets[g.tickets[i]].p3().fg ? fgi : plain).push_back(i);
                auto subset = [&](const std::vector<int>& idx) {
                    std::unique_ptr<Img3dLaunch> X(new Img3dLaunch(L));
                    X->n = static_cast<int32_t>(idx.size());
                    for (size_t j = 0; j < idx.size(); ++j) {
                        X->d[j] = L.d[idx[j]];
                        X->tm_img[j] = L.tm_img[idx[j]];
                        X->tm_lbl[j] = L.tm_lbl[idx[j]];
                    }
                    return X;
                };
                auto Lf = subset(fgi);
                FgLaunch F{};
                for (size_t j = 0; j < fgi.size(); ++j) {
                    const Params3D& p3 = tickets[g.tickets[fgi[j]]].p3();
                    F.d[j].fg = 1;
                    F.d[j].u_cls = p3.u_cls;
                    for (int a = 0; a < 3; ++a) F.d[j].u_adj[a] = p3.u_adj[a];
                    counters.kernel_bytes += Lf->d[j].lbl_pz * Lf->d[j].sdim[0];   // the label volume, once
                }
                const int slot = fg_next_;
                fg_next_ = (fg_next_ + 1) % kFgSlots;
                int32_t* box = fg_box_ + size_t(slot) * kMax3D * 48;
                int4* offs = fg_offs_ + size_t(slot) * kMax3D;
                start();
                // The label scans (K2) fork onto a side stream and run concurrently with
                // the plain samples' K1 on the group's stream; the group's stream joins
                // them before the foreground crops.
                cudaStream_t side = side_streams_[static_cast<size_t>(side_next_++) % side_streams_.size()];
                cudaEvent_t fork = get_event();
                cuda_check(cudaEventRecord(fork, st), "record fork");
                cuda_check(cudaStreamWaitEvent(side, fork, 0), "fork");
                put_event(fork);   // (the wait captured the record; the event may be reused)
                // mins ([kMax3D][8][3]) preset large, maxs (the next block) to -1
                cuda_check(cudaMemsetAsync(box, 0x7f, kMax3D * 24 * sizeof(int32_t), side), "fg box reset");
                cuda_check(cudaMemsetAsync(box + kMax3D * 24, 0xff, kMax3D * 24 * sizeof(int32_t), side),
                           "fg box reset");
                cuda_check(launch_fg_scan(*Lf, F, box, side), "fg scan launch");
                cuda_check(launch_fg_offsets(*Lf, F, box, offs, side), "fg offsets launch");
                counters.launches += 2;
                cudaEvent_t join = get_event();
                cuda_check(cudaEventRecord(join, side), "record join");
                if (!plain.empty()) {   // the plain samples complete at a sub-launch event
                    auto Lp = subset(plain);
                    contrast_and_transform(*Lp);
                    g.part_ev = get_event(g.timed);
                    cuda_check(cudaEventRecord(g.part_ev, st), "record plain part");
                    g.part_idx = plain;
                }
                cuda_check(cudaStreamWaitEvent(st, join, 0), "join");
                put_event(join);
                if (staged) {
                    // K0w: the windows at the resolved origins, from pinned host memory
                    // (image) and the staged label volume (label), into compact windows
                    WindowLaunch W{};
                    W.n = Lf->n;
                    W.offs = offs;
                    for (int j = 0; j < Lf->n; ++j) {
                        const Ticket& t = tickets[g.tickets[fgi[j]]];
                        const View& v = views[fgi[j]];
                        WindowDesc& w = W.d[j];
                        Img3dDesc& d = Lf->d[j];
                        w.img_host = static_cast<const float*>(t.desc().data);
                        w.lbl = d.lbl;
                        w.lbl_py = d.lbl_py;
                        w.lbl_pz = d.lbl_pz;
                        w.lbl_sk0 = d.lbl_sk0;
                        w.lbl_sky = d.lbl_sky;
                        w.lbl_skz = d.lbl_skz;
                        for (int a = 0; a < 3; ++a) {
                            w.dims[a] = static_cast<int32_t>(t.desc().dims[a]);
                            w.win[a] = d.win[a];
                        }
                        w.img_pitch = (d.win[2] + 3) / 4 * 4;
                        w.lbl_pitch = (d.win[2] + 15) / 16 * 16;
                        w.dst_img = reinterpret_cast<float*>(const_cast<char*>(v.p[0]));
                        w.dst_lbl = reinterpret_cast<uint8_t*>(const_cast<char*>(v.p[0])) +
                                    align256(int64_t(4) * w.img_pitch * d.win[1] * d.win[0]);
                        counters.h2d_bytes += int64_t(4) * d.win[0] * d.win[1] *
                                              std::max<int64_t>(0, std::min<int64_t>(d.win[2], t.desc().dims[2]));
                        // K1 / K4 read the compact window: origin 0, all of it valid
                        d.img = w.dst_img;
                        d.lbl = w.dst_lbl;
                        d.img_py = w.img_pitch;
                        d.img_pz = int64_t(w.img_pitch) * d.win[1];
                        d.lbl_py = w.lbl_pitch;
                        d.lbl_pz = int64_t(w.lbl_pitch) * d.win[1];
                        d.img_sk0 = d.img_sky = d.img_skz = d.lbl_sk0 = d.lbl_sky = d.lbl_skz = 0;
                        for (int a = 0; a < 3; ++a) {
                            d.sdim[a] = d.win[a];
                            d.off[a] = 0;
                        }
                    }
                    cuda_check(launch_stage_window(W, st), "window stage launch");
                    counters.launches++;
                    Lf->offs = nullptr;
                } else {
                    Lf->offs = offs;
                }
                contrast_and_transform(*Lf);
            }
            prof_launch_ns += std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t_l).count();
        } else if (S.kind == ST_RRC2D) {
            RrcLaunch L{};
            L.oh = c.oh;
            L.ow = c.ow;
            for (int k = 0; k < 3; ++k) {
                const double a = (c.to_tensor ? 1.0 / 255.0 : 1.0) / c.std[k];
                L.a[k] = static_cast<float>(a);
                L.b[k] = static_cast<float>(-c.mean[k] / c.std[k]);
            }
            L.n = n;
            L.out_tab = out_tab_;
            L.out_stride = c.plane_bytes[0] / 4;
            L.slot_base = slot_of(0);
            if (stamp_here) {   // image i stamps slot_base + i: the group's tickets must be consecutive
                bool consecutive = true;
                for (int i = 1; i < n && consecutive; ++i) consecutive = slot_of(i) == L.slot_base + i;
                if (consecutive) L.st = stamps;
                else g.stamped = false;   // (the group completes as a whole)
            }
            for (int i = 0; i < n; ++i) {
                const Ticket& t = tickets[g.tickets[i]];
                const Params2D& p = t.p2();
                bool ok;
                if (staged) {   // the K0-staged box (skewed rows)
                    const View& v = views[i];
                    ok = rrc_pack(L.d[i], v.p[0], v.sk0[0], v.sky[0], static_cast<int>(v.py[0]), static_cast<int>(p.h),
                                  static_cast<int>(p.w), p.flip, t.pos, t.buf);
                } else {        // the crop box inside the HBM-resident HWC image
                    const lfg_sample_desc& sd = t.desc();
                    ok = rrc_pack(L.d[i], static_cast<const uint8_t*>(sd.data) + (p.top * sd.dims[1] + p.left) * 3, 0, 0,
                                  static_cast<int>(sd.dims[1] * 3), static_cast<int>(p.h), static_cast<int>(p.w), p.flip,
                                  t.pos, t.buf);
                }
                if (!ok) fail(LFG_ERR_UNSUPPORTED, "obj_det sample does not fit the packed K3 descriptor");
                counters.kernel_bytes += rrc_algo_bytes(c, p);
            }
            lap(prof_desc_ns, t_lap);
            const auto t_l = std::chrono::steady_clock::now();
            start();
            cuda_check(launch_rrc2d(L, st), "rrc2d launch");
            prof_launch_ns += std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t_l).count();
            counters.launches++;
        } else {
            SpLaunch L{};
            L.n = n;
            L.n_fmask = c.n_fmask;
            L.n_tmask = c.n_tmask;
            L.stack = c.stack;
            L.pcm16 = c.wav_bytes == 2;
            if (stamp_here) L.st = stamps;
            for (int i = 0; i < n; ++i) {
                Ticket& t = tickets[g.tickets[i]];
                SpDesc& d = L.d[i];
                d.slot = slot_of(i);
                d.wav = views[i].p[0];
                d.out = reinterpret_cast<float*>(slot_ptr(t, 0));
                d.L = static_cast<int32_t>(t.desc().dims[0]);
                d.T = t.ps().T;
                for (int k = 0; k < c.n_fmask; ++k) {
                    d.f_lo[k] = t.ps().f_lo[k];
                    d.f_w[k] = t.ps().f_w[k];
                }
                for (int k = 0; k < c.n_tmask; ++k) {
                    d.t_lo[k] = t.ps().t_lo[k];
                    d.t_w[k] = t.ps().t_w[k];
                }
                counters.kernel_bytes += c.wav_bytes * t.desc().dims[0] +
                                         4 * int64_t((t.ps().T + c.stack - 1) / c.stack) * c.stack * c.n_mels;
                counters.reserved[1] += int64_t(t.ps().T) * 2 * kTapsDft * 512 * 3;   // tensor FLOPs
            }
            start();
            cuda_check(launch_speech(L, speech_, st), "speech launch");
            counters.launches++;
        }
        for (size_t k = 0; k < S.spin_ops.size(); ++k)
            launch_spins(S.spin_ops[k], s == nst - 1 && k + 1 == S.spin_ops.size());
        start();
        cuda_check(cudaEventRecord(g.ev[s + 1], st), "record stage end");
    }
    g.launched = true;
    g.t_launch_us = host_now_us();
    g.serial = ++launch_serial_;
    if (cfg.coalesce_us > 0) {
        struct DoneMsg {
            Context* ctx;
            int64_t serial;
        };
        auto* msg = new DoneMsg{this, g.serial};
        cuda_check(cudaLaunchHostFunc(
                       st,
                       [](void* p) {
                           auto* m = static_cast<DoneMsg*>(p);
                           Context* cx = m->ctx;
                           const int w = static_cast<int>(m->serial & (kDoneWaits - 1));
                           {
                               std::lock_guard<std::mutex> lk(cx->done_mu_[w]);
                               cx->done_ring_[m->serial & (kDoneSlots - 1)].store(m->serial, std::memory_order_release);
                           }
                           cx->done_cv_[w].notify_all();
                           delete m;
                       },
                       msg),
                   "group completion notice");
    }
    prof_group_ns += std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t_enter).count();
}

// ------------------------------------------------------------------ progress
Group& Context::group_of(int64_t t) {
    if (t < 0 || t >= static_cast<int64_t>(tickets.size())) fail(LFG_ERR_INVALID, "unknown ticket");
    if (tickets[t].released) fail(LFG_ERR_INVALID, "ticket already released");
    return groups[tickets[t].group];
}

bool Context::poll_group(Group& g) {
    if (g.complete) return true;
    if (!g.launched) return false;
    const int nst = static_cast<int>(g.chain->stages.size());
    while (g.stages_done < nst) {
        std::chrono::steady_clock::time_point t0;
        if (prof_on) t0 = std::chrono::steady_clock::now();
        cudaError_t q = cudaEventQuery(g.ev[g.stages_done + 1]);
        if (prof_on) {
            prof_query_ns += std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
            ++prof_queries;
        }
        if (q == cudaErrorNotReady) return false;
        cuda_check(q, "stage event");
        g.stages_done++;
    }
    g.complete = true;
    std::chrono::steady_clock::time_point t1;
    if (prof_on) t1 = std::chrono::steady_clock::now();
    finalize_group_timing(g);
    if (prof_on) prof_final_ns += std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t1).count();
    counters.completed += static_cast<int64_t>(g.tickets.size());
    if (g.stream_idx != 0) free_streams_.push_back(g.stream_idx);
    if (g.raw_idx >= 0) {
        free_raws_.push_back(g.raw_idx);
        g.raw_idx = -1;
    }
    return true;
}

void Context::finalize_group_timing(Group& g) {
    const int nst = static_cast<int>(g.chain->stages.size());
    g.stage_ms.assign(nst, 0.0f);
    for (int s = 0; s < nst && g.timed; ++s) {
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, g.ev[s], g.ev[s + 1]), "stage time");
        g.stage_ms[s] = ms;
    }
    if (g.part_ev != nullptr) {
        if (g.timed) cuda_check(cudaEventElapsedTime(&g.part_ms, g.ev[0], g.part_ev), "part time");
        put_event(g.part_ev, g.timed);
        g.part_ev = nullptr;
        g.part_done = true;
    }
    for (auto e : g.ev) put_event(e, g.timed);
    g.ev.clear();
}

void Context::progress(int64_t t, int* ops_done, int* complete, int64_t* elapsed_us) {
    Group& g = group_of(t);
    const int64_t now = host_now_us();
    // a coalescing group still open launches once its deadline passed
    if (!g.launched && !g.complete && cfg.coalesce_us > 0 && now - g.t_open_us >= cfg.coalesce_us)
        launch_if_pending(t);
    // Per-sample pollers (process_sample workers) share launch groups: the group's
    // events are queried at most once per 2 us however many of its samples' workers
    // poll (an event query costs ~1.5 us under the context lock)
    if (!g.complete && now - g.t_query_us >= 2) {
        g.t_query_us = now;
        poll_group(g);
    }
    const bool done = sample_ready(t);   // its own stamp, or the whole group
    const auto& st = g.chain->stages;
    const int od = g.stages_done > 0 ? st[g.stages_done - 1].last_op : 0;
    if (ops_done) *ops_done = done ? static_cast<int>(g.chain->ops.size()) : od;
    if (complete) *complete = done ? 1 : 0;
    if (elapsed_us) *elapsed_us = g.launched ? host_now_us() - g.t_launch_us : 0;
}

bool Context::launch_if_pending(int64_t t) {
    Group& g = group_of(t);
    if (!g.launched) {
        for (auto& og : open_group_)
            for (auto it = og.begin(); it != og.end(); ++it)
                if (it->second == g.id) { og.erase(it); break; }
        launch_group(g);
    }
    return poll_group(g);
}

void Context::wait(int64_t t) {
    Group& g = group_of(t);
    if (!launch_if_pending(t)) {
        cuda_check(cudaEventSynchronize(g.ev.back()), "wait");
        poll_group(g);
    }
}

int Context::exec_costs(int64_t t, double* out, int cap) {
    Group& g = group_of(t);
    if (!sample_ready(t)) fail(LFG_ERR_STATE, "sample not complete");
    const int nops = static_cast<int>(g.chain->ops.size());
    if (cap < nops) fail(LFG_ERR_INVALID, "cost buffer too small");
    for (int i = 0; i < nops; ++i) out[i] = 0.0;
    if (!g.complete) {
        // the sample finished before its group: no stage events yet, so its cost is
        // the wall time from the group's launch to now (the realtime runtime's clock),
        // attributed to the last op
        out[nops - 1] = static_cast<double>(host_now_us() - g.t_launch_us);
        return nops;
    }
    for (size_t s = 0; s < g.stage_ms.size(); ++s)
        out[g.chain->stages[s].last_op - 1] = 1000.0 * g.stage_ms[s];
    return nops;
}

void Context::ticket_output(int64_t t, void* dst, size_t bytes) {
    Group& g = group_of(t);
    Ticket& tk = tickets[t];
    if (!sample_ready(t)) fail(LFG_ERR_STATE, "sample not complete");
    if (tk.consumed) fail(LFG_ERR_STATE, "sample already sealed into a batch");
    const Chain& c = *g.chain;
    if (bytes < static_cast<size_t>(c.plane_bytes[0] + (c.nplanes > 1 ? c.plane_bytes[1] : 0)))
        fail(LFG_ERR_INVALID, "output buffer too small");
    char* d = static_cast<char*>(dst);
    cuda_check(cudaMemcpy(d, slot_ptr(tk, 0), c.plane_bytes[0], cudaMemcpyDeviceToHost), "D2H output");
    if (c.nplanes > 1)
        cuda_check(cudaMemcpy(d + c.plane_bytes[0], slot_ptr(tk, 1), c.plane_bytes[1],
                              cudaMemcpyDeviceToHost),
                   "D2H output");
    counters.d2h_bytes += c.out_bytes;
}

void Context::ticket_release(int64_t t) {
    Group& g = group_of(t);
    Ticket& tk = tickets[t];
    if (!tk.consumed) {
        if (!sample_ready(t)) fail(LFG_ERR_STATE, "cannot release an in-flight sample");
        bufs_[tk.buf].live--;
        tk.consumed = true;
    }
    tk.released = true;
    g.refs--;
}

// ------------------------------------------------------------------ seal
int64_t Context::seal(const int64_t* ts, int n) {
    if (n < 1) fail(LFG_ERR_INVALID, "empty batch");
    if (n > cfg.batch_size) fail(LFG_ERR_INVALID, "batch larger than batch_size");
    const Chain* c = nullptr;
    bool same_buf = true;
    for (int i = 0; i < n; ++i) {
        if (ts[i] < 0 || ts[i] >= static_cast<int64_t>(tickets.size())) fail(LFG_ERR_INVALID, "unknown ticket");
        Ticket& t = tickets[ts[i]];
        if (t.released || t.consumed) fail(LFG_ERR_INVALID, "ticket already sealed or released");
        Group& g = groups[t.group];
        if (!sample_ready(ts[i])) fail(LFG_ERR_STATE, "cannot seal an incomplete sample");
        if (c == nullptr) c = g.chain;
        if (g.chain != c) fail(LFG_ERR_INVALID, "batch mixes chains");
        if (t.buf != tickets[ts[0]].buf) same_buf = false;
    }
    // duplicate check in O(n): mark, test, unmark
    for (int i = 0; i < n; ++i) {
        Ticket& t = tickets[ts[i]];
        if (t.in_seal) {
            for (int j = 0; j < i; ++j) tickets[ts[j]].in_seal = false;
            fail(LFG_ERR_INVALID, "duplicate ticket in batch");
        }
        t.in_seal = true;
    }
    for (int i = 0; i < n; ++i) tickets[ts[i]].in_seal = false;
    const int b0 = tickets[ts[0]].buf;
    // speech batches are time-major (PermuteAudio), so they are always collated
    const bool in_place = c->fam != FAM_SPEECH && same_buf && bufs_[b0].assigned == n &&
                          !bufs_[b0].in_batch;

    BatchRec br;
    br.chain = c;
    br.n = n;
    br.in_place = in_place;
    // the seal stream waits for every distinct producing group
    std::vector<int64_t> gs;
    for (int i = 0; i < n; ++i) gs.push_back(tickets[ts[i]].group);
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
    (void)gs;  // every sample is complete (its stamp landed: its outputs are written and
               // published device-wide) -- no device wait needed

    if (in_place) {
        SlotBuf& b = bufs_[b0];
        if (b.open) {
            b.open = false;
            auto it = open_buf_.find(c);
            if (it != open_buf_.end() && it->second == b0) open_buf_.erase(it);
        }
        b.in_batch = true;
        br.buf = b0;
        br.ids.assign(n, 0);
        for (int i = 0; i < n; ++i) br.ids[tickets[ts[i]].pos] = tickets[ts[i]].id;
        counters.inplace_batches++;
    } else {
        const int nb = alloc_buf(c, true);
        br.buf = nb;
        GatherLaunch L{};
        L.nplanes = c->nplanes;
        L.plane_bytes[0] = c->plane_bytes[0];
        L.plane_bytes[1] = c->plane_bytes[1];
        L.dst = bufs_[nb].base;
        L.dst_plane_stride = static_cast<int64_t>(bufs_[nb].cap) * c->plane_bytes[0];
        L.n = n;
        br.ids.resize(n);
        std::vector<int> src_bufs;
        for (int i = 0; i < n; ++i) {
            Ticket& t = tickets[ts[i]];
            L.src[i] = slot_ptr(t, 0);
            L.src_plane_stride[i] = c->nplanes > 1 ? slot_ptr(t, 1) - slot_ptr(t, 0) : 0;
            br.ids[i] = t.id;
            src_bufs.push_back(t.buf);
        }
        if (c->fam == FAM_SPEECH) {
            // PermuteAudio + Pad: time-major [T'_max, n, stack * 80], zero-padded
            SpCollate SC{};
            SC.n = n;
            SC.width = c->stack * c->n_mels;
            for (int i = 0; i < n; ++i) {
                const Ticket& t = tickets[ts[i]];
                SC.rows[i] = (t.ps().T + c->stack - 1) / c->stack;
                SC.src[i] = reinterpret_cast<const float*>(L.src[i]);
                SC.t_max = std::max(SC.t_max, SC.rows[i]);
            }
            SC.dst = reinterpret_cast<float*>(bufs_[nb].base);
            br.t_max = SC.t_max;
            br.rows.assign(SC.rows, SC.rows + n);
            cuda_check(launch_speech_collate(SC, seal_stream), "collate launch");
            counters.reserved[0] += 2 * static_cast<int64_t>(SC.t_max) * n * SC.width * 4;
        } else {
            cuda_check(launch_gather(L, seal_stream), "gather launch");
            counters.reserved[0] += 2 * static_cast<int64_t>(n) * c->out_bytes;  // gather bytes
        }
        counters.launches++;
        std::sort(src_bufs.begin(), src_bufs.end());
        src_bufs.erase(std::unique(src_bufs.begin(), src_bufs.end()), src_bufs.end());
        for (int sb : src_bufs) {
            cudaEvent_t e = get_event();
            cuda_check(cudaEventRecord(e, seal_stream), "record gather");
            bufs_[sb].pending.push_back(e);
        }
        for (int i = 0; i < n; ++i) bufs_[tickets[ts[i]].buf].live--;
        counters.gathered_batches++;
    }
    // An in-place batch is ready the moment it is sealed: every sample was seen
    // complete above, so there is nothing for a consumer stream to wait on.
    if (!in_place) {
        br.ready = get_event();
        cuda_check(cudaEventRecord(br.ready, seal_stream), "record batch ready");
    }
    for (int i = 0; i < n; ++i) {
        Ticket& t = tickets[ts[i]];
        t.consumed = true;
    }
    counters.batches++;
    if (n < cfg.batch_size) counters.short_batches++;
    batches.push_back(std::move(br));
    return static_cast<int64_t>(batches.size()) - 1;
}

BatchRec& Context::batch(int64_t b) {
    if (b < 0 || b >= static_cast<int64_t>(batches.size())) fail(LFG_ERR_INVALID, "unknown batch");
    if (batches[b].released) fail(LFG_ERR_INVALID, "batch already released");
    return batches[b];
}

void Context::batch_wait_stream(int64_t b, cudaStream_t s) {
    BatchRec& br = batch(b);
    if (br.ready) cuda_check(cudaStreamWaitEvent(s, br.ready, 0), "batch wait");
}

// `readers`: work that reads the batch may still be queued on `s`, so the
// buffer is reused only after an event recorded there; the shard runner
// passes false when it enqueued nothing for the batch.
void Context::batch_release(int64_t b, cudaStream_t s, bool readers) {
    BatchRec& br = batch(b);
    SlotBuf& buf = bufs_[br.buf];
    if (readers) {
        cudaEvent_t e = get_event();
        cuda_check(cudaEventRecord(e, s), "record batch release");
        buf.pending.push_back(e);
    }
    buf.in_batch = false;
    if (br.in_place) buf.live -= br.n;
    br.released = true;
    // the ready event also covers work queued before it on the delivering stream (a
    // streaming run's captures / probe): the buffer is reused only after it, too
    if (br.ready) buf.pending.push_back(br.ready);
    br.ready = nullptr;
}

void Context::trainer_step(int64_t b, cudaStream_t s, int64_t us) {
    batch_wait_stream(b, s);
    if (us > 0) {
        cuda_check(launch_trainer_spin(us * 1000, 1, s), "trainer step");
        counters.launches++;
    }
}

int64_t Context::capture_sample(int64_t b, int pos, char* dst, int64_t cap_bytes, cudaStream_t s) {
    BatchRec& br = batch(b);
    const Chain& c = *br.chain;
    if (pos < 0 || pos >= br.n) fail(LFG_ERR_INVALID, "capture position out of range");
    const SlotBuf& buf = bufs_[br.buf];
    batch_wait_stream(b, s);
    if (c.fam == FAM_SPEECH) {   // time-major [t_max, n, width]: the sample's rows, packed
        const int64_t w = int64_t(c.stack) * c.n_mels * 4;
        const int64_t rows = br.rows[pos];
        if (rows * w > cap_bytes) fail(LFG_ERR_INVALID, "capture stride too small");
        cuda_check(cudaMemcpy2DAsync(dst, w, buf.base + pos * w, w * br.n, w, rows, cudaMemcpyDeviceToHost, s),
                   "capture D2H");
        return rows * w;
    }
    const int64_t p0 = c.plane_bytes[0], p1 = c.nplanes > 1 ? c.plane_bytes[1] : 0;
    if (p0 + p1 > cap_bytes) fail(LFG_ERR_INVALID, "capture stride too small");
    cuda_check(cudaMemcpyAsync(dst, buf.base + pos * p0, p0, cudaMemcpyDeviceToHost, s), "capture D2H");
    if (p1 > 0)
        cuda_check(cudaMemcpyAsync(dst + p0, buf.base + int64_t(buf.cap) * p0 + pos * p1, p1,
                                   cudaMemcpyDeviceToHost, s),
                   "capture D2H");
    return p0 + p1;
}

void rng_outputs(uint64_t seed, uint64_t id, int n, uint64_t* out) {
    SampleRng r(seed, id);
    for (int i = 0; i < n; ++i) out[i] = r.g();
}

}  // namespace lfg
