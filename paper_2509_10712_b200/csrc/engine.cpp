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
#include <cstring>

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

// ------------------------------------------------------------------ params
// Per-sample generator: the reference's Rng (std::mt19937_64, sample.hpp:25)
// seeded with experiment.cpp:163's mixing constant keyed by sample id.
namespace {
struct SampleRng {
    std::mt19937_64 g;
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

void draw_3d(const Chain& c, uint64_t seed, uint64_t id, const int64_t dims[3], Params3D& p) {
    SampleRng r(seed, id);
    for (int a = 0; a < 3; ++a) {
        const int64_t room = dims[a] - c.crop[a];
        p.off[a] = r.randint(0, room > 0 ? room : 0);
    }
    for (int a = 0; a < 3; ++a) p.flip[a] = r.unif01() < c.p_flip;
    const bool b_apply = r.unif01() < c.p_bright;
    const double b_factor = r.uniform(c.b_lo, c.b_hi);
    p.scale = b_apply ? b_factor : 1.0;
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

int64_t Chain::algo_bytes_per_sample(const lfg_sample_desc& s) const {
    switch (fam) {
        case FAM_IMG3D: {
            const int64_t vox = int64_t(crop[0]) * crop[1] * crop[2];
            return vox * 10;  // read f32 + u8, write f32 + u8
        }
        case FAM_RRC2D: {
            (void)s;
            return out_bytes;  // write side; the read side is added per sample by the caller
        }
        case FAM_SPEECH:
            return 4 * s.dims[0] + out_bytes;
        default:
            return 0;
    }
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
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    cuda_check(cudaStreamCreateWithPriority(&seal_stream, cudaStreamNonBlocking, hi), "seal stream");
    cuda_check(cudaStreamCreateWithFlags(&aux_stream, cudaStreamNonBlocking), "aux stream");
}

Context::~Context() {
    cudaSetDevice(cfg.device);
    cudaDeviceSynchronize();
    for (auto& g : groups) for (auto e : g.ev) if (e) cudaEventDestroy(e);
    for (auto& b : batches) if (b.ready) cudaEventDestroy(b.ready);
    for (auto e : free_events_) cudaEventDestroy(e);
    for (auto& b : bufs_) {
        for (auto e : b.pending) cudaEventDestroy(e);
        cudaFree(b.base);
    }
    for (auto& r : raws_) cudaFree(r.ptr);
    for (auto s : streams_) cudaStreamDestroy(s);
    cudaStreamDestroy(seal_stream);
    cudaStreamDestroy(aux_stream);
}

cudaEvent_t Context::get_event() {
    if (!free_events_.empty()) {
        cudaEvent_t e = free_events_.back();
        free_events_.pop_back();
        return e;
    }
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void Context::put_event(cudaEvent_t e) { free_events_.push_back(e); }

int Context::get_stream() {
    if (serial) {
        if (streams_.empty()) {
            cudaStream_t s;
            cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
            streams_.push_back(s);
        }
        return 0;
    }
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
        case LFG_OP_RANDOM_FLIP: fam = FAM_IMG3D; return 2;
        case LFG_OP_RANDOM_BRIGHTNESS: fam = FAM_IMG3D; return 3;
        case LFG_OP_GAUSSIAN_NOISE: fam = FAM_IMG3D; return 4;
        case LFG_OP_CAST: fam = FAM_IMG3D; return 5;
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
        if (c->oh < 1 || c->ow < 1 || c->ow > 256 || c->oh > 4096)
            fail(LFG_ERR_UNSUPPORTED, "Resize output must be <= 256 wide");
        c->nplanes = 1;
        c->plane_bytes[0] = int64_t(3) * c->oh * c->ow * 4;
    } else {
        fail(LFG_ERR_UNSUPPORTED, "speech chain not available in this build");
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
    chains_.push_back(std::move(c));
    return chains_.back().get();
}

void Context::chain_destroy(Chain* c) {
    for (auto& g : groups)
        if (g.chain == c && !g.complete) fail(LFG_ERR_STATE, "chain has samples in flight");
    for (size_t i = 0; i < chains_.size(); ++i) {
        if (chains_[i].get() == c) {
            open_buf_.erase(c);
            open_group_[0].erase(c);
            open_group_[1].erase(c);
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

int Context::alloc_buf(const Chain* c, bool for_batch) {
    // Slot buffers (samples are written into them) and gather buffers (targets
    // of a collating seal) are bounded separately so stragglers pinning slot
    // buffers can never starve the seal of a destination.
    int count = 0;
    const int64_t need = static_cast<int64_t>(cfg.batch_size) * c->out_bytes;
    for (size_t i = 0; i < bufs_.size(); ++i) {
        SlotBuf& b = bufs_[i];
        if (b.gather_role != for_batch) continue;
        bool alive = b.chain == c;
        if (!alive) {
            bool chain_live = false;
            for (auto& ch : chains_) chain_live |= ch.get() == b.chain;
            if (chain_live) continue;          // belongs to another live chain
            if (b.bytes < need) continue;      // dead chain's buffer, too small to recycle
        }
        ++count;
        if (buf_reusable(b)) {
            b.chain = c;
            b.cap = cfg.batch_size;
            b.assigned = 0;
            b.live = 0;
            b.open = !for_batch;
            b.in_batch = for_batch;
            return static_cast<int>(i);
        }
    }
    if (count >= cfg.max_slot_buffers) {
        fail(LFG_ERR_AGAIN, "all output buffers are in use (consume or release batches)");
    }
    SlotBuf b;
    cuda_check(cudaMalloc(&b.base, static_cast<size_t>(need)), "cudaMalloc(slot buffer)");
    b.cap = cfg.batch_size;
    b.chain = c;
    b.bytes = need;
    b.gather_role = for_batch;
    b.open = !for_batch;
    b.in_batch = for_batch;
    bufs_.push_back(b);
    return static_cast<int>(bufs_.size()) - 1;
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
int64_t Context::get_raw(int64_t bytes) {
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
    r.cap = std::max<int64_t>(bytes, 1 << 20);
    cuda_check(cudaMalloc(&r.ptr, static_cast<size_t>(r.cap)), "cudaMalloc(raw staging)");
    raws_.push_back(r);
    return static_cast<int64_t>(raws_.size()) - 1;
}

static int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

int64_t Context::stage_raw_bytes(const Chain& c, const Ticket& t) const {
    if (c.fam == FAM_IMG3D) {
        int64_t vox = 1;
        for (int a = 0; a < 3; ++a) vox *= std::min<int64_t>(c.crop[a], t.desc.dims[a] - t.p3.off[a]);
        return align256(vox * 4) + align256(vox);
    }
    if (c.fam == FAM_RRC2D) return align256(t.p2.h * t.p2.w * 3);
    return align256(t.desc.dims[0] * 4);
}

// ------------------------------------------------------------------ submit
int64_t Context::submit(Chain* c, const lfg_sample_desc& s) {
    if (c == nullptr) fail(LFG_ERR_INVALID, "null chain");
    if (s.data == nullptr) fail(LFG_ERR_INVALID, "sample has no payload");
    if (s.src_kind != LFG_SRC_DEVICE && s.src_kind != LFG_SRC_HOST_PINNED)
        fail(LFG_ERR_INVALID, "bad src_kind");
    Ticket t;
    t.id = s.id;
    t.desc = s;
    if (c->fam == FAM_IMG3D) {
        if (s.ndim != 3 || s.aux == nullptr) fail(LFG_ERR_INVALID, "img_seg sample needs a D,H,W volume and a label");
        for (int a = 0; a < 3; ++a)
            if (s.dims[a] < 1 || s.dims[a] > (1 << 20)) fail(LFG_ERR_INVALID, "volume dims out of range");
        draw_3d(*c, cfg.seed, s.id, s.dims, t.p3);
    } else if (c->fam == FAM_RRC2D) {
        if (s.ndim != 3 || s.dims[2] != 3 || s.dims[0] < 1 || s.dims[1] < 1)
            fail(LFG_ERR_INVALID, "obj_det sample needs an H,W,3 image");
        draw_2d(*c, cfg.seed, s.id, s.dims[0], s.dims[1], t.p2);
    } else {
        if (s.ndim != 1 || s.dims[0] < 2 || s.dims[0] > c->max_L)
            fail(LFG_ERR_INVALID, "speech sample needs a waveform of length in [2, max_L]");
        draw_sp(*c, cfg.seed, s.id, s.dims[0], t.ps);
    }
    for (int k = 0; k < c->n_spin; ++k)
        if (s.spin_us[k] < 0) fail(LFG_ERR_STATE, "negative transform cost");  // balancer.cpp:16
    assign_slot(t, c);
    auto& og = open_group_[s.src_kind == LFG_SRC_DEVICE ? 0 : 1];
    auto it = og.find(c);
    int64_t gi;
    if (it == og.end()) {
        Group g;
        g.id = static_cast<int64_t>(groups.size());
        g.chain = c;
        g.src_kind = s.src_kind;
        groups.push_back(std::move(g));
        gi = static_cast<int64_t>(groups.size()) - 1;
        og[c] = gi;
    } else {
        gi = it->second;
    }
    const int64_t ti = static_cast<int64_t>(tickets.size());
    t.group = gi;
    t.idx = static_cast<int>(groups[gi].tickets.size());
    tickets.push_back(t);
    Group& g = groups[gi];
    g.tickets.push_back(ti);
    g.refs++;
    counters.submitted++;
    const int cap = c->fam == FAM_IMG3D ? kMax3D : (c->fam == FAM_RRC2D ? kMax2D : kMaxSp);
    if (static_cast<int>(g.tickets.size()) >= std::min(cfg.max_group, cap)) {
        og.erase(c);
        launch_group(g);
    }
    return ti;
}

int64_t Context::open_group_count() const {
    return static_cast<int64_t>(open_group_[0].size() + open_group_[1].size());
}

void Context::flush() {
    for (auto& og : open_group_) {
        for (auto& kv : og) launch_group(groups[kv.second]);
        og.clear();
    }
}

void Context::launch_group(Group& g) {
    const Chain& c = *g.chain;
    g.stream_idx = get_stream();
    g.stream = streams_[g.stream_idx];
    const int nst = static_cast<int>(c.stages.size());
    g.ev.resize(nst + 1);
    for (auto& e : g.ev) e = get_event();
    cudaStream_t st = g.stream;
    cuda_check(cudaEventRecord(g.ev[0], st), "record start");
    const int n = static_cast<int>(g.tickets.size());

    // host-pinned payloads: copy only the bytes the chain reads (crop window /
    // crop box / waveform) into one device staging buffer
    std::vector<const char*> src0(n), src1(n);
    std::vector<int64_t> sdim(3 * n);
    if (g.src_kind == LFG_SRC_HOST_PINNED) {
        int64_t total = 0;
        for (int i = 0; i < n; ++i) total += stage_raw_bytes(c, tickets[g.tickets[i]]);
        g.raw_idx = get_raw(total);
        char* dst = raws_[g.raw_idx].ptr;
        for (int i = 0; i < n; ++i) {
            Ticket& t = tickets[g.tickets[i]];
            if (c.fam == FAM_IMG3D) {
                int64_t wd[3];
                for (int a = 0; a < 3; ++a) wd[a] = std::min<int64_t>(c.crop[a], t.desc.dims[a] - t.p3.off[a]);
                const int64_t vox = wd[0] * wd[1] * wd[2];
                for (int plane = 0; plane < 2; ++plane) {
                    const int64_t esz = plane == 0 ? 4 : 1;
                    cudaMemcpy3DParms p{};
                    p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(plane == 0 ? t.desc.data : t.desc.aux),
                                                   t.desc.dims[2] * esz, t.desc.dims[2], t.desc.dims[1]);
                    p.srcPos = make_cudaPos(t.p3.off[2] * esz, t.p3.off[1], t.p3.off[0]);
                    p.dstPtr = make_cudaPitchedPtr(dst, wd[2] * esz, wd[2], wd[1]);
                    p.extent = make_cudaExtent(wd[2] * esz, wd[1], wd[0]);
                    p.kind = cudaMemcpyHostToDevice;
                    cuda_check(cudaMemcpy3DAsync(&p, st), "H2D crop window");
                    (plane == 0 ? src0 : src1)[i] = dst;
                    dst += align256(vox * esz);
                    counters.h2d_bytes += vox * esz;
                }
                for (int a = 0; a < 3; ++a) sdim[3 * i + a] = wd[a];
            } else if (c.fam == FAM_RRC2D) {
                const int64_t W = t.desc.dims[1];
                const char* s = static_cast<const char*>(t.desc.data) + (t.p2.top * W + t.p2.left) * 3;
                cuda_check(cudaMemcpy2DAsync(dst, t.p2.w * 3, s, W * 3, t.p2.w * 3, t.p2.h,
                                             cudaMemcpyHostToDevice, st),
                           "H2D crop box");
                src0[i] = dst;
                sdim[3 * i] = t.p2.w;
                counters.h2d_bytes += t.p2.h * t.p2.w * 3;
                dst += align256(t.p2.h * t.p2.w * 3);
            } else {
                cuda_check(cudaMemcpyAsync(dst, t.desc.data, t.desc.dims[0] * 4,
                                           cudaMemcpyHostToDevice, st),
                           "H2D waveform");
                src0[i] = dst;
                counters.h2d_bytes += t.desc.dims[0] * 4;
                dst += align256(t.desc.dims[0] * 4);
            }
        }
    } else {
        for (int i = 0; i < n; ++i) {
            Ticket& t = tickets[g.tickets[i]];
            src0[i] = static_cast<const char*>(t.desc.data);
            src1[i] = static_cast<const char*>(t.desc.aux);
            if (c.fam == FAM_IMG3D) for (int a = 0; a < 3; ++a) sdim[3 * i + a] = t.desc.dims[a];
            else if (c.fam == FAM_RRC2D) sdim[3 * i] = t.desc.dims[1];
        }
    }
    const bool staged = g.src_kind == LFG_SRC_HOST_PINNED;

    auto launch_spins = [&](int slot) {
        SpinLaunch L{};
        L.n = n;
        for (int i = 0; i < n; ++i) L.ns[i] = tickets[g.tickets[i]].desc.spin_us[slot] * 1000;
        cuda_check(launch_spin(L, st), "spin launch");
        counters.launches++;
    };

    for (int s = 0; s < nst; ++s) {
        const Stage& S = c.stages[s];
        if (S.kind == ST_SPIN) {
            launch_spins(S.spin_ops[0]);
        } else if (S.kind == ST_IMG3D) {
            Img3dLaunch L{};
            for (int a = 0; a < 3; ++a) L.crop[a] = c.crop[a];
            L.n = n;
            for (int i = 0; i < n; ++i) {
                Ticket& t = tickets[g.tickets[i]];
                Img3dDesc& d = L.d[i];
                d.img = reinterpret_cast<const float*>(src0[i]);
                d.lbl = reinterpret_cast<const uint8_t*>(src1[i]);
                d.out_img = reinterpret_cast<float*>(slot_ptr(t, 0));
                d.out_lbl = reinterpret_cast<uint8_t*>(slot_ptr(t, 1));
                for (int a = 0; a < 3; ++a) {
                    d.sdim[a] = static_cast<int32_t>(sdim[3 * i + a]);
                    d.off[a] = staged ? 0 : static_cast<int32_t>(t.p3.off[a]);
                }
                d.flip = t.p3.flip[0] | (t.p3.flip[1] << 1) | (t.p3.flip[2] << 2);
                d.scale = static_cast<float>(t.p3.scale);
                d.sigma = static_cast<float>(t.p3.sigma);
                d.key0 = t.p3.key[0];
                d.key1 = t.p3.key[1];
                counters.kernel_bytes += c.algo_bytes_per_sample(t.desc);
            }
            cuda_check(launch_img3d(L, st), "img3d launch");
            counters.launches++;
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
            for (int i = 0; i < n; ++i) {
                Ticket& t = tickets[g.tickets[i]];
                RrcDesc& d = L.d[i];
                d.src = reinterpret_cast<const uint8_t*>(src0[i]);
                d.out = reinterpret_cast<float*>(slot_ptr(t, 0));
                d.sw = static_cast<int32_t>(sdim[3 * i]);
                d.top = staged ? 0 : static_cast<int32_t>(t.p2.top);
                d.left = staged ? 0 : static_cast<int32_t>(t.p2.left);
                d.h = static_cast<int32_t>(t.p2.h);
                d.w = static_cast<int32_t>(t.p2.w);
                d.flip = t.p2.flip;
                const int64_t rows = std::min<int64_t>(t.p2.h, 2 * c.oh);
                const int64_t cols = std::min<int64_t>(t.p2.w, 2 * c.ow);
                counters.kernel_bytes += c.out_bytes + rows * cols * 3;
            }
            cuda_check(launch_rrc2d(L, st), "rrc2d launch");
            counters.launches++;
        } else {
            fail(LFG_ERR_UNSUPPORTED, "speech stage not available");
        }
        for (int slot : S.spin_ops) launch_spins(slot);
        cuda_check(cudaEventRecord(g.ev[s + 1], st), "record stage end");
    }
    g.launched = true;
    g.t_launch_us = host_now_us();
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
        cudaError_t q = cudaEventQuery(g.ev[g.stages_done + 1]);
        if (q == cudaErrorNotReady) return false;
        cuda_check(q, "stage event");
        g.stages_done++;
    }
    g.complete = true;
    finalize_group_timing(g);
    counters.completed += static_cast<int64_t>(g.tickets.size());
    if (!serial || g.stream_idx != 0) free_streams_.push_back(g.stream_idx);
    if (g.raw_idx >= 0) {
        free_raws_.push_back(g.raw_idx);
        g.raw_idx = -1;
    }
    return true;
}

void Context::finalize_group_timing(Group& g) {
    const int nst = static_cast<int>(g.chain->stages.size());
    g.stage_ms.assign(nst, 0.0f);
    for (int s = 0; s < nst; ++s) {
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, g.ev[s], g.ev[s + 1]), "stage time");
        g.stage_ms[s] = ms;
    }
    for (auto e : g.ev) put_event(e);
    g.ev.clear();
}

void Context::progress(int64_t t, int* ops_done, int* complete, int64_t* elapsed_us) {
    Group& g = group_of(t);
    poll_group(g);
    const auto& st = g.chain->stages;
    const int od = g.stages_done > 0 ? st[g.stages_done - 1].last_op : 0;
    if (ops_done) *ops_done = g.complete ? static_cast<int>(g.chain->ops.size()) : od;
    if (complete) *complete = g.complete ? 1 : 0;
    if (elapsed_us) *elapsed_us = g.launched ? host_now_us() - g.t_launch_us : 0;
}

void Context::wait(int64_t t) {
    Group& g = group_of(t);
    if (!g.launched) {
        for (auto& og : open_group_)
            for (auto it = og.begin(); it != og.end(); ++it)
                if (it->second == g.id) { og.erase(it); break; }
        launch_group(g);
    }
    if (!g.complete) {
        cuda_check(cudaEventSynchronize(g.ev.back()), "wait");
        poll_group(g);
    }
}

int Context::exec_costs(int64_t t, double* out, int cap) {
    Group& g = group_of(t);
    if (!g.complete) fail(LFG_ERR_STATE, "sample not complete");
    const int nops = static_cast<int>(g.chain->ops.size());
    if (cap < nops) fail(LFG_ERR_INVALID, "cost buffer too small");
    for (int i = 0; i < nops; ++i) out[i] = 0.0;
    for (size_t s = 0; s < g.stage_ms.size(); ++s)
        out[g.chain->stages[s].last_op - 1] = 1000.0 * g.stage_ms[s];
    return nops;
}

void Context::ticket_output(int64_t t, void* dst, size_t bytes) {
    Group& g = group_of(t);
    Ticket& tk = tickets[t];
    if (!g.complete) fail(LFG_ERR_STATE, "sample not complete");
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
        if (!g.complete) fail(LFG_ERR_STATE, "cannot release an in-flight sample");
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
        if (!poll_group(g)) fail(LFG_ERR_STATE, "cannot seal an incomplete sample");
        if (c == nullptr) c = g.chain;
        if (g.chain != c) fail(LFG_ERR_INVALID, "batch mixes chains");
        if (t.buf != tickets[ts[0]].buf) same_buf = false;
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j)
            if (ts[i] == ts[j]) fail(LFG_ERR_INVALID, "duplicate ticket in batch");
    const int b0 = tickets[ts[0]].buf;
    const bool in_place = same_buf && bufs_[b0].assigned == n && !bufs_[b0].in_batch;

    BatchRec br;
    br.chain = c;
    br.n = n;
    br.in_place = in_place;
    // the seal stream waits for every distinct producing group
    std::vector<int64_t> gs;
    for (int i = 0; i < n; ++i) gs.push_back(tickets[ts[i]].group);
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
    (void)gs;  // all producing groups are complete (checked above): no device wait needed

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
        cuda_check(launch_gather(L, seal_stream), "gather launch");
        counters.launches++;
        counters.kernel_bytes += 2 * static_cast<int64_t>(n) * c->out_bytes;
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
    br.ready = get_event();
    cuda_check(cudaEventRecord(br.ready, seal_stream), "record batch ready");
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
    cuda_check(cudaStreamWaitEvent(s, batch(b).ready, 0), "batch wait");
}

void Context::batch_release(int64_t b, cudaStream_t s) {
    BatchRec& br = batch(b);
    SlotBuf& buf = bufs_[br.buf];
    cudaEvent_t e = get_event();
    cuda_check(cudaEventRecord(e, s), "record batch release");
    buf.pending.push_back(e);
    buf.in_batch = false;
    if (br.in_place) buf.live -= br.n;
    br.released = true;
    put_event(br.ready);
    br.ready = nullptr;
}

void Context::trainer_step(int64_t b, cudaStream_t s, int64_t us) {
    batch_wait_stream(b, s);
    if (us > 0) {
        cuda_check(launch_trainer_spin(us * 1000, 1, s), "trainer step");
        counters.launches++;
    }
}

}  // namespace lfg
