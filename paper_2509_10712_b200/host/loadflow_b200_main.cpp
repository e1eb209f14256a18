// loadflow_b200_main.cpp -- `loadflow_b200 run | compare`: the reference CLI's
// experiment entry points (proj/tools/loadflow_main.cpp:34-134) for the GPU
// loaders, SURVEY 8(f) row 4.
//
//   loadflow_b200 run <config.ini> [--loader minato-gpu|sync-gpu] [--seed N] [--out DIR]
//   loadflow_b200 compare <report.json>... [--csv FILE]
//   loadflow_b200 dropin [...]   (lf_dropin.cpp: throughput of the drop-in C++ path)
//
// The config file uses the reference's flat `[section] key = value` format and key
// names (experiment.cpp:64-116): workload.name / n_samples / seed,
// pipeline.loader / batch_size, consumer.compute_ms, scheduler.enabled /
// initial_workers / max_workers / tick_ms, profiler.window / warmup_ms /
// update_interval_ms / initial_timeout_ms, run.out_dir; plus gpu.* extensions:
// gpu.device, gpu.time_scale_us_per_ms (reference milliseconds -> device
// microseconds, default 10), gpu.pool (distinct synthetic payloads), gpu.group
// (samples per launch group, default 1), gpu.src
// (device | pinned | file: payloads written once as sample files under gpu.data_dir and
// read back by gpu.readers threads into gpu.slots pinned buffers, lfgpu_files.h).  The
// sample stream is the reference workload generator's
// (generate(spec): same ids, costs and sizes); every sample runs the workload's
// real transform chain on the GPU plus a synthetic device cost of its reference
// cost x time_scale, and a synthetic trainer step of consumer.compute_ms x
// time_scale per batch.  The report follows MetricsReport's fields
// (metrics.hpp:29-69) with a "gpu" block.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "lfgpu.h"
#include "lfgpu_files.h"
#include "loadflow/api.hpp"

namespace {

using Kv = std::map<std::string, std::string>;

std::string trim(const std::string& s) {
    const auto a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    const auto b = s.find_last_not_of(" \t\r\n");
    return s.substr(a, b - a + 1);
}

// flat `[section]` / `key = value` / `#` or `;` comments -> "section.key" -> value
Kv parse_config(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open config: " + path);
    Kv kv;
    std::string line, section;
    int ln = 0;
    while (std::getline(in, line)) {
        ++ln;
        const auto c = line.find_first_of("#;");
        line = trim(c == std::string::npos ? line : line.substr(0, c));
        if (line.empty()) continue;
        if (line.front() == '[') {
            if (line.back() != ']') throw std::runtime_error(path + ":" + std::to_string(ln) + ": bad section");
            section = trim(line.substr(1, line.size() - 2));
            continue;
        }
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw std::runtime_error(path + ":" + std::to_string(ln) + ": expected key = value");
        kv[(section.empty() ? "" : section + ".") + trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
    }
    return kv;
}

std::string get(const Kv& kv, const std::string& k, const std::string& d) {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
}
double getd(const Kv& kv, const std::string& k, double d) {
    auto it = kv.find(k);
    return it == kv.end() ? d : std::stod(it->second);
}
bool getb(const Kv& kv, const std::string& k, bool d) {
    auto it = kv.find(k);
    if (it == kv.end()) return d;
    return it->second == "true" || it->second == "1" || it->second == "yes";
}

void check(int rc, const char* what) {
    if (rc != LFG_OK) throw std::runtime_error(std::string(what) + ": " + lfg_last_error());
}

lfg_op mk(int kind, const char* name, double f, std::initializer_list<double> p = {}) {
    lfg_op o{};
    o.kind = kind;
    o.size_factor = f;
    int i = 0;
    for (double v : p) o.param[i++] = v;
    std::snprintf(o.name, sizeof(o.name), "%s", name);
    return o;
}

// the workload's reference transform chain (workloads.cpp:103-156) as device ops,
// behind a leading synthetic-cost op carrying the reference per-sample cost
std::vector<lfg_op> chain_ops(loadflow::WorkloadKind k) {
    using loadflow::WorkloadKind;
    std::vector<lfg_op> ops{mk(LFG_OP_SPIN, "SampleCost", 1.0)};
    if (k == WorkloadKind::img_seg) {
        ops.push_back(mk(LFG_OP_RANDOM_CROP, "RandomCrop", 0.0735, {128, 128, 128}));
        ops.push_back(mk(LFG_OP_RANDOM_FLIP, "RandomFlip", 1.0, {1.0 / 3.0}));
        ops.push_back(mk(LFG_OP_RANDOM_BRIGHTNESS, "RandomBrightness", 1.0, {0.1, 0.7, 1.3}));
        ops.push_back(mk(LFG_OP_GAUSSIAN_NOISE, "GaussianNoise", 1.0, {0.1, 0.1}));
        ops.push_back(mk(LFG_OP_CAST, "Cast", 1.0));
    } else if (k == WorkloadKind::obj_det) {
        ops.push_back(mk(LFG_OP_RESIZE, "Resize", 1.2, {224, 224, 0.08, 1.0, 0.75, 4.0 / 3.0}));
        ops.push_back(mk(LFG_OP_RANDOM_HFLIP, "RandomHorizontalFlip", 1.0, {0.5}));
        ops.push_back(mk(LFG_OP_TO_TENSOR, "ToTensor", 8.0));
        ops.push_back(mk(LFG_OP_NORMALIZE, "Normalize", 1.0, {0.485, 0.456, 0.406, 0.229, 0.224, 0.225}));
    } else {
        ops.push_back(mk(LFG_OP_PAD, "Pad", 1.12));
        ops.push_back(mk(LFG_OP_SPEC_AUGMENT, "SpecAugment", 1.0, {2, 27, 10, 0.05}));
        // waveforms as int16 PCM: the reference's speech bytes_in is 2 B per sample (workloads.cpp:115)
        ops.push_back(mk(LFG_OP_FILTER_BANK, "FilterBank", 1.0, {512, 320, 160, 80, 170000, LFG_DT_I16}));
        ops.push_back(mk(LFG_OP_FRAME_SPLICING, "FrameSplicing", 0.9, {3}));
        ops.push_back(mk(LFG_OP_PERMUTE_AUDIO, "PermuteAudio", 1.0));
    }
    return ops;
}

struct Payload {
    void* data = nullptr;
    void* aux = nullptr;
    int ndim = 0;
    int64_t dims[4] = {0, 0, 0, 0};
};

int cmd_run(const std::string& cfg_path, const std::string& loader_arg, int64_t seed_arg,
            const std::string& out_arg) {
    Kv kv = parse_config(cfg_path);
    if (!loader_arg.empty()) kv["pipeline.loader"] = loader_arg;
    if (seed_arg >= 0) kv["workload.seed"] = std::to_string(seed_arg);
    if (!out_arg.empty()) kv["run.out_dir"] = out_arg;
    const std::string loader = get(kv, "pipeline.loader", "minato-gpu");
    if (loader != "minato-gpu" && loader != "sync-gpu")
        throw std::invalid_argument("pipeline.loader must be minato-gpu or sync-gpu (got " + loader + ")");
    const auto kind = loadflow::workload_from_name(get(kv, "workload.name", "img_seg"));
    const int64_t n = static_cast<int64_t>(getd(kv, "workload.n_samples", 1000));
    const uint64_t seed = static_cast<uint64_t>(getd(kv, "workload.seed", 1));
    const int B = static_cast<int>(getd(kv, "pipeline.batch_size", 24));
    const double scale = getd(kv, "gpu.time_scale_us_per_ms", 10.0);
    const int pool = static_cast<int>(getd(kv, "gpu.pool", 16));
    const std::string src_kind = get(kv, "gpu.src", "device");   // device | pinned | file
    if (src_kind != "device" && src_kind != "pinned" && src_kind != "file")
        throw std::invalid_argument("gpu.src must be device, pinned or file");
    const bool from_file = src_kind == "file";
    const bool pinned = src_kind == "pinned" || from_file;   // file payloads are synthesised in pinned memory
    if (static_cast<int>(getd(kv, "pipeline.n_consumers", 1)) != 1)
        throw std::invalid_argument("one consumer per process: run one process per GPU for more");

    loadflow::WorkloadSpec spec = loadflow::default_spec(kind, n, seed);
    loadflow::Stream stream = loadflow::generate(spec);

    lfg_config cfg;
    lfg_config_default(&cfg);
    cfg.device = static_cast<int>(getd(kv, "gpu.device", 0));
    cfg.batch_size = B;
    const int workers = static_cast<int>(getd(kv, "scheduler.initial_workers", 12));
    cfg.n_workers = workers;
    // samples per launch group: 1 = per-sample classification, as the reference's
    // per-sample timeouts (default); larger groups for loader-throughput runs
    cfg.max_group = static_cast<int>(getd(kv, "gpu.group", 1));
    cfg.max_slot_buffers = std::max(8, 2 * workers / std::max(1, B) + 8);
    cfg.seed = seed;
    lfg_ctx* ctx = nullptr;
    check(lfg_open(&cfg, &ctx), "lfg_open");
    const auto ops = chain_ops(kind);
    lfg_chain* chain = nullptr;
    check(lfg_chain_create(ctx, ops.data(), static_cast<int>(ops.size()), &chain), "chain");

    // synthetic payloads shaped by the stream's first `pool` samples' bytes_in
    std::vector<Payload> pay(static_cast<size_t>(std::min<int64_t>(pool, n)));
    for (size_t i = 0; i < pay.size(); ++i) {
        const double bytes = stream.samples[i].bytes_in;
        Payload& p = pay[i];
        auto alloc = [&](size_t b) {
            void* q = nullptr;
            check(pinned ? lfg_host_alloc(ctx, b, &q) : lfg_device_alloc(ctx, b, &q), "alloc");
            return q;
        };
        if (kind == loadflow::WorkloadKind::img_seg) {
            const int64_t D = std::clamp<int64_t>(std::llround(bytes / (5.0 * 384 * 384)), 128, 512);
            p.ndim = 3;
            p.dims[0] = D, p.dims[1] = 384, p.dims[2] = 384;
            p.data = alloc(D * 384 * 384 * 4);
            p.aux = alloc(D * 384 * 384);
            check(lfg_synth_volume(ctx, seed, i, D, 384, 384, p.data, p.aux, pinned ? 0 : 1), "synth volume");
        } else if (kind == loadflow::WorkloadKind::obj_det) {
            const int64_t side = std::clamp<int64_t>(std::llround(std::sqrt(bytes / 3.0)), 256, 512);
            p.ndim = 3;
            p.dims[0] = side, p.dims[1] = side, p.dims[2] = 3;
            p.data = alloc(side * side * 3);
            check(lfg_synth_image(ctx, seed, i, side, side, p.data, pinned ? 0 : 1), "synth image");
        } else {
            const int64_t L = std::clamp<int64_t>(std::llround(bytes / 2.0), 30000, 170000);
            p.ndim = 1;
            p.dims[0] = L;
            p.data = alloc(L * 2);
            std::vector<float> wav(static_cast<size_t>(L));
            check(lfg_synth_waveform(ctx, seed, i, L, wav.data(), 0), "synth waveform");
            std::vector<int16_t> pcm(static_cast<size_t>(L));
            for (size_t v = 0; v < pcm.size(); ++v)
                pcm[v] = static_cast<int16_t>(std::clamp<long>(std::lrint(wav[v] * 20000.0f), -32768, 32767));
            if (pinned) std::memcpy(p.data, pcm.data(), pcm.size() * 2);
            else check(lfg_memcpy_h2d(ctx, p.data, pcm.data(), pcm.size() * 2), "upload waveform");
        }
    }
    check(lfg_synchronize(ctx), "sync");
    std::vector<lfg_sample_desc> descs(static_cast<size_t>(n));
    double bytes_out = 0;
    for (int64_t i = 0; i < n; ++i) {
        const auto& s = stream.samples[static_cast<size_t>(i)];
        const Payload& p = pay[static_cast<size_t>(i) % pay.size()];
        lfg_sample_desc& d = descs[static_cast<size_t>(i)];
        std::memset(&d, 0, sizeof(d));
        d.id = s.id;
        d.src_kind = pinned ? LFG_SRC_HOST_PINNED : LFG_SRC_DEVICE;
        d.ndim = p.ndim;
        for (int a = 0; a < 4; ++a) d.dims[a] = p.dims[a];
        d.data = p.data;
        d.aux = p.aux;
        int64_t cost = 0;
        for (auto c : s.step_costs) cost += c;
        d.spin_us[0] = static_cast<int64_t>(std::llround(static_cast<double>(cost) * scale));
        bytes_out += s.bytes_out;
    }

    lfg_run_config rc{};
    rc.batch_size = B;
    rc.policy = loader == "sync-gpu" ? 3 : 1;
    rc.t_out_us = kv.count("profiler.initial_timeout_ms")
                      ? static_cast<int64_t>(getd(kv, "profiler.initial_timeout_ms", 0) * scale)
                      : 0;
    rc.warmup_us = static_cast<int64_t>(getd(kv, "profiler.warmup_ms", 10000) * scale);
    rc.update_interval_us = static_cast<int64_t>(getd(kv, "profiler.update_interval_ms", 1000) * scale);
    rc.window = static_cast<int32_t>(getd(kv, "profiler.window", 1024));
    rc.n_workers = workers;
    rc.trainer_us = static_cast<int64_t>(getd(kv, "consumer.compute_ms", 200) * scale);
    rc.trainer_priority = 1;
    rc.percentile = 75;
    rc.scheduler = (loader == "minato-gpu" && getb(kv, "scheduler.enabled", true)) ? 1 : 0;
    rc.max_workers = static_cast<int32_t>(getd(kv, "scheduler.max_workers", 2 * workers));
    rc.sched_tick_us = static_cast<int64_t>(getd(kv, "scheduler.tick_ms", 500) * scale);
    rc.prefetch_factor = static_cast<int32_t>(getd(kv, "pipeline.prefetch_factor", 2));   // experiment.cpp:83
    lfg_run_report rep{};
    std::vector<uint64_t> ids(static_cast<size_t>(n));
    std::vector<int32_t> bsz(static_cast<size_t>(n)), cls(static_cast<size_t>(n));
    int64_t file_bytes = 0;
    double file_seconds = 0;
    if (from_file) {
        // raw reads from storage: the pool's payloads become sample
        // files once; reader threads pread them into recycled pinned slots ahead of the shard
        const std::string dir = get(kv, "gpu.data_dir", "/tmp/lfg_data_" + std::string(loadflow::workload_name(kind)));
        mkdir(dir.c_str(), 0755);
        std::vector<std::string> files;
        const int fkind = kind == loadflow::WorkloadKind::img_seg
                              ? LFG_FILE_VOLUME
                              : (kind == loadflow::WorkloadKind::obj_det ? LFG_FILE_IMAGE : LFG_FILE_PCM16);
        for (size_t i = 0; i < pay.size(); ++i) {
            files.push_back(dir + "/sample_" + std::to_string(i) + ".lfgs");
            check(lfg_write_sample_file(files.back().c_str(), fkind, pay[i].ndim, pay[i].dims, pay[i].data, pay[i].aux),
                  "write sample file");
        }
        std::vector<const char*> paths(static_cast<size_t>(n));
        std::vector<uint64_t> fids(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            paths[static_cast<size_t>(i)] = files[static_cast<size_t>(i) % files.size()].c_str();
            fids[static_cast<size_t>(i)] = descs[static_cast<size_t>(i)].id;
        }
        lfg_file_source* fs = nullptr;
        if (lfg_file_source_open(ctx, paths.data(), fids.data(), n, static_cast<int>(getd(kv, "gpu.readers", 8)),
                                 static_cast<int>(getd(kv, "gpu.slots", 64)), &fs) != LFG_OK)
            throw std::runtime_error(std::string("file source: ") + lfg_files_last_error());
        // the per-sample synthetic costs ride on the descriptors the source cannot know:
        // wrap its next() to copy them in
        struct Wrap {
            lfg_source inner;
            const std::vector<lfg_sample_desc>* descs;
            int64_t i = 0;
        } w{};
        check(lfg_file_source_get(fs, &w.inner), "file source");
        w.descs = &descs;
        lfg_source wrapped{&w,
                           [](void* u, lfg_sample_desc* d) {
                               auto* ww = static_cast<Wrap*>(u);
                               const int r = ww->inner.next(ww->inner.user, d);
                               if (r == 1) {
                                   for (int k = 0; k < 4; ++k) d->spin_us[k] = (*ww->descs)[static_cast<size_t>(ww->i)].spin_us[k];
                                   ++ww->i;
                               }
                               return r;
                           },
                           [](void* u, uint64_t id) {
                               auto* ww = static_cast<Wrap*>(u);
                               ww->inner.release(ww->inner.user, id);
                           }};
        const int rc_run = lfg_run_shard_source(ctx, chain, &wrapped, n, &rc, &rep, ids.data(), bsz.data(), cls.data());
        lfg_file_source_stats(fs, &file_bytes, &file_seconds);
        lfg_file_source_close(fs);
        check(rc_run, "run");
    } else {
        check(lfg_run_shard(ctx, chain, descs.data(), n, &rc, &rep, ids.data(), bsz.data(), cls.data()), "run");
    }

    const double completion_ms = rep.elapsed_ms;
    const double slow_rate = rep.samples ? static_cast<double>(rep.slow) / static_cast<double>(rep.samples) : 0;
    std::ostringstream js;
    js.precision(10);
    js << "{\n  \"workload\": \"" << loadflow::workload_name(kind) << "\",\n  \"loader\": \"" << loader
       << "\",\n  \"mode\": \"gpu\",\n  \"n_samples\": " << n << ",\n  \"batch_size\": " << B
       << ",\n  \"completion_ms\": " << completion_ms << ",\n  \"completion_ref_ms\": "
       << (scale > 0 ? std::to_string(completion_ms * 1000.0 / scale) : std::string("null")) << ",\n  \"samples\": " << rep.samples << ",\n  \"batches\": "
       << rep.batches << ",\n  \"short_batches\": " << rep.short_batches << ",\n  \"slow_rate\": " << slow_rate
       << ",\n  \"avg_throughput_mbps\": " << (completion_ms > 0 ? bytes_out / 1e6 / (completion_ms / 1e3) : 0)
       << ",\n  \"exactly_once\": " << (rep.exactly_once ? "true" : "false") << ",\n  \"duplicates\": "
       << rep.duplicates << ",\n  \"consumers\": [{\"busy_ms\": " << rep.consumer_busy_ms
       << ", \"span_ms\": " << rep.consumer_span_ms << ", \"idle_ms\": "
       << rep.consumer_span_ms - rep.consumer_busy_ms << ", \"idle_fraction\": " << rep.consumer_idle_frac
       << "}],\n  \"gpu\": {\"device\": " << cfg.device << ", \"time_scale_us_per_ms\": " << scale
       << ", \"samples_per_s\": " << rep.samples_per_s << ", \"kernel_ms\": " << rep.kernel_ms
       << ", \"h2d_bytes\": " << rep.h2d_bytes << ", \"launches\": " << rep.launches
       << ", \"final_t_out_us\": " << rep.final_t_out_us << ", \"final_percentile\": " << rep.final_percentile
       << ", \"final_workers\": " << rep.final_workers << ", \"mean_workers\": " << rep.mean_workers
       << ", \"src\": \"" << src_kind << "\", \"file_bytes_read\": " << file_bytes
       << ", \"file_read_seconds\": " << file_seconds << "}\n}\n";
    std::cout << "workload=" << loadflow::workload_name(kind) << " loader=" << loader
              << " completion_ms=" << completion_ms << " throughput_mbps="
              << (completion_ms > 0 ? bytes_out / 1e6 / (completion_ms / 1e3) : 0) << " slow_rate=" << slow_rate
              << " idle=" << rep.consumer_idle_frac << " exactly_once=" << (rep.exactly_once ? "yes" : "no")
              << "\n";
    const std::string out_dir = get(kv, "run.out_dir", "");
    if (!out_dir.empty()) {
        mkdir(out_dir.c_str(), 0755);
        std::ofstream(out_dir + "/report.json") << js.str();
        std::ofstream csv(out_dir + "/batches.csv");
        csv << "batch,size\n";
        for (int64_t b = 0; b < rep.batches; ++b) csv << b << "," << bsz[static_cast<size_t>(b)] << "\n";
        std::ofstream sc(out_dir + "/samples.csv");
        sc << "position,id,class,consumed_order_id\n";
        for (int64_t i = 0; i < n; ++i)
            sc << i << "," << descs[static_cast<size_t>(i)].id << "," << (cls[static_cast<size_t>(i)] == 2 ? "slow" : "fast")
               << "," << ids[static_cast<size_t>(i)] << "\n";
        std::cout << "report written to " << out_dir << "/report.json\n";
    }
    for (auto& p : pay) {
        for (void* q : {p.data, p.aux})
            if (q) (pinned ? lfg_host_free(ctx, q) : lfg_device_free(ctx, q));
    }
    lfg_chain_destroy(ctx, chain);
    lfg_close(ctx);
    return rep.exactly_once ? 0 : 3;
}

// minimal reader for the flat fields of our report.json
double json_num(const std::string& js, const std::string& key) {
    const auto k = js.find("\"" + key + "\"");
    if (k == std::string::npos) throw std::runtime_error("report lacks " + key);
    return std::stod(js.substr(js.find(':', k) + 1));
}
std::string json_str(const std::string& js, const std::string& key) {
    const auto k = js.find("\"" + key + "\"");
    if (k == std::string::npos) throw std::runtime_error("report lacks " + key);
    const auto a = js.find('"', js.find(':', k) + 1);
    return js.substr(a + 1, js.find('"', a + 1) - a - 1);
}

// experiment.cpp:439-512 compare(): speedup and idle delta against the first report
int cmd_compare(const std::vector<std::string>& paths, const std::string& csv_out) {
    struct Row { std::string workload, loader; double completion, idle; };
    std::vector<Row> rows;
    for (const auto& p : paths) {
        std::ifstream in(p);
        if (!in) throw std::runtime_error("cannot open report: " + p);
        std::stringstream ss;
        ss << in.rdbuf();
        const std::string js = ss.str();
        rows.push_back({json_str(js, "workload"), json_str(js, "loader"), json_num(js, "completion_ms"),
                        json_num(js, "idle_fraction")});
    }
    std::ostringstream t, c;
    t << "workload      loader        completion_ms  speedup  idle    idle_delta\n";
    c << "workload,loader,completion_ms,speedup,idle_fraction,idle_delta\n";
    for (const auto& r : rows) {
        const double sp = r.completion > 0 ? rows[0].completion / r.completion : 0;
        char line[256];
        std::snprintf(line, sizeof(line), "%-13s %-13s %13.3f %8.3f %7.4f %+10.4f\n", r.workload.c_str(),
                      r.loader.c_str(), r.completion, sp, r.idle, r.idle - rows[0].idle);
        t << line;
        c << r.workload << "," << r.loader << "," << r.completion << "," << sp << "," << r.idle << ","
          << r.idle - rows[0].idle << "\n";
    }
    std::cout << t.str();
    if (!csv_out.empty()) {
        std::ofstream(csv_out) << c.str();
        std::cout << "comparison csv written to " << csv_out << "\n";
    }
    return 0;
}

int usage() {
    std::cerr << "usage: loadflow_b200 run <config.ini> [--loader minato-gpu|sync-gpu] [--seed N] [--out DIR]\n"
                 "       loadflow_b200 compare <report.json>... [--csv FILE]\n"
                 "       loadflow_b200 dropin [--workers N] [--samples N] [--batch B] [--group G]\n"
                 "                            [--coalesce-us U] [--t-out-us T] [--pool P] [--seed S] [--max-seconds M]\n";
    return 1;
}

}  // namespace

int cmd_dropin(int argc, char** argv);   // lf_dropin.cpp

int main(int argc, char** argv) {
    // the application's choice (the library never sets it): one hardware queue per
    // launch-group stream, before the first CUDA call creates the device context
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
    try {
        if (argc >= 2 && std::string(argv[1]) == "dropin") return cmd_dropin(argc, argv);
        if (argc < 3) return usage();
        const std::string cmd = argv[1];
        if (cmd == "run") {
            std::string loader, out;
            int64_t seed = -1;
            for (int i = 3; i + 1 < argc; i += 2) {
                const std::string k = argv[i];
                if (k == "--loader") loader = argv[i + 1];
                else if (k == "--seed") seed = std::atoll(argv[i + 1]);
                else if (k == "--out") out = argv[i + 1];
                else return usage();
            }
            return cmd_run(argv[2], loader, seed, out);
        }
        if (cmd == "compare") {
            std::vector<std::string> paths;
            std::string csv;
            for (int i = 2; i < argc; ++i) {
                if (std::string(argv[i]) == "--csv" && i + 1 < argc) csv = argv[++i];
                else paths.push_back(argv[i]);
            }
            if (paths.empty()) return usage();
            return cmd_compare(paths, csv);
        }
        return usage();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
