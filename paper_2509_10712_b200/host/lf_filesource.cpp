// lf_filesource.cpp -- raw sample files and the reader-thread source of
// lfgpu_files.h.  The reference's feeder (experiment.cpp:
// 221-228) only models a load latency; here the bytes come from storage (page
// cache or disk) through pread into pinned buffers that the shard's K0 / DMA
// staging reads directly.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "lfgpu_files.h"

namespace {

struct Header {
    char magic[4];
    uint32_t version;
    int32_t kind;
    int32_t ndim;
    int64_t dims[4];
};
static_assert(sizeof(Header) == 48, "file header is 48 bytes");

int64_t payload_bytes(int kind, const int64_t dims[4], int64_t* first) {
    if (kind == LFG_FILE_VOLUME) {
        const int64_t v = dims[0] * dims[1] * dims[2];
        *first = 4 * v;
        return 5 * v;
    }
    if (kind == LFG_FILE_IMAGE) return *first = dims[0] * dims[1] * 3;
    if (kind == LFG_FILE_WAVEFORM) return *first = 4 * dims[0];
    if (kind == LFG_FILE_PCM16) return *first = 2 * dims[0];
    return *first = -1;
}

thread_local std::string g_err;
int err(int code, const std::string& m) {
    g_err = m;
    return code;
}

bool read_all(int fd, void* dst, int64_t bytes, int64_t off) {
    char* p = static_cast<char*>(dst);
    while (bytes > 0) {
        const ssize_t r = pread(fd, p, static_cast<size_t>(std::min<int64_t>(bytes, 1 << 30)), off);
        if (r <= 0) return false;
        p += r;
        bytes -= r;
        off += r;
    }
    return true;
}

}  // namespace

struct lfg_file_source {
    lfg_ctx* ctx = nullptr;
    std::vector<std::string> paths;
    std::vector<uint64_t> ids;
    std::vector<Header> hdr;
    int64_t n = 0;
    int64_t slot_bytes = 0;
    std::vector<char*> slots;
    std::vector<int64_t> slot_of;        // sample -> slot (-1 until assigned)
    std::vector<uint8_t> state;          // 0 pending, 1 reading, 2 ready, 3 failed
    std::vector<int> free_slots;
    std::mutex mu;
    std::condition_variable cv;
    int64_t next_read = 0, next_give = 0;
    bool stop = false;
    std::vector<std::thread> readers;
    std::atomic<int64_t> bytes_read{0};
    std::atomic<int64_t> read_ns{0};
    std::vector<std::pair<uint64_t, int64_t>> live;   // (id, sample index) handed to the shard

    void reader() {
        for (;;) {
            int64_t i;
            int s;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || (next_read < n && !free_slots.empty()); });
                if (stop) return;
                i = next_read++;
                s = free_slots.back();
                free_slots.pop_back();
                slot_of[i] = s;
                state[i] = 1;
            }
            const auto t0 = std::chrono::steady_clock::now();
            bool ok = false;
            const int fd = open(paths[i].c_str(), O_RDONLY);
            if (fd >= 0) {
                int64_t first = 0;
                const int64_t pb = payload_bytes(hdr[i].kind, hdr[i].dims, &first);
                ok = pb > 0 && read_all(fd, slots[s], pb, sizeof(Header));
                close(fd);
                if (ok) bytes_read += pb + static_cast<int64_t>(sizeof(Header));
            }
            read_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
                           .count();
            {
                std::lock_guard<std::mutex> lk(mu);
                state[i] = ok ? 2 : 3;
            }
            cv.notify_all();
        }
    }

    int next(lfg_sample_desc* out) {
        std::lock_guard<std::mutex> lk(mu);
        if (next_give >= n) return 0;
        const int64_t i = next_give;
        if (state[i] == 3) return err(-1, "cannot read " + paths[i]);
        if (state[i] != 2) return 2;
        const Header& h = hdr[i];
        std::memset(out, 0, sizeof(*out));
        out->id = ids[i];
        out->src_kind = LFG_SRC_HOST_PINNED;
        out->ndim = (h.kind == LFG_FILE_WAVEFORM || h.kind == LFG_FILE_PCM16) ? 1 : 3;
        for (int a = 0; a < 4; ++a) out->dims[a] = h.dims[a];
        if (h.kind == LFG_FILE_IMAGE) out->dims[2] = 3;
        char* base = slots[slot_of[i]];
        out->data = base;
        if (h.kind == LFG_FILE_VOLUME) {
            int64_t first = 0;
            payload_bytes(h.kind, h.dims, &first);
            out->aux = base + first;
        }
        live.emplace_back(ids[i], i);
        ++next_give;
        return 1;
    }

    void release(uint64_t id) {
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = std::find_if(live.begin(), live.end(), [&](const auto& p) { return p.first == id; });
            if (it == live.end()) return;
            free_slots.push_back(static_cast<int>(slot_of[it->second]));
            *it = live.back();
            live.pop_back();
        }
        cv.notify_all();
    }
};

extern "C" {

int lfg_write_sample_file(const char* path, int kind, int ndim, const int64_t dims[4], const void* data,
                          const void* aux) {
    if (!path || !dims || !data || (kind == LFG_FILE_VOLUME && !aux)) return err(LFG_ERR_INVALID, "null argument");
    Header h{};
    std::memcpy(h.magic, "LFGS", 4);
    h.version = 1;
    h.kind = kind;
    h.ndim = ndim;
    for (int a = 0; a < 4; ++a) h.dims[a] = dims[a];
    int64_t first = 0;
    const int64_t pb = payload_bytes(kind, h.dims, &first);
    if (pb <= 0) return err(LFG_ERR_INVALID, "bad kind / dims");
    const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) return err(LFG_ERR_INVALID, std::string("cannot create ") + path);
    auto wr = [&](const void* p, int64_t b) {
        const char* q = static_cast<const char*>(p);
        while (b > 0) {
            const ssize_t r = write(fd, q, static_cast<size_t>(std::min<int64_t>(b, 1 << 30)));
            if (r <= 0) return false;
            q += r;
            b -= r;
        }
        return true;
    };
    bool ok = wr(&h, sizeof(h)) && wr(data, first) && (pb == first || wr(aux, pb - first));
    ok = (close(fd) == 0) && ok;
    return ok ? LFG_OK : err(LFG_ERR_INVALID, std::string("short write to ") + path);
}

int lfg_file_source_open(lfg_ctx* ctx, const char* const* paths, const uint64_t* ids, int64_t n, int readers,
                         int slots, lfg_file_source** out) {
    if (!ctx || !paths || !ids || !out || n < 1 || readers < 1 || slots < 1)
        return err(LFG_ERR_INVALID, "bad file source arguments");
    auto fs = new lfg_file_source;
    fs->ctx = ctx;
    fs->n = n;
    fs->paths.assign(paths, paths + n);
    fs->ids.assign(ids, ids + n);
    fs->hdr.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {   // headers up front: slot size = the largest payload
        const int fd = open(paths[i], O_RDONLY);
        Header& h = fs->hdr[static_cast<size_t>(i)];
        const bool ok = fd >= 0 && read_all(fd, &h, sizeof(h), 0) && std::memcmp(h.magic, "LFGS", 4) == 0 &&
                        h.version == 1;
        if (fd >= 0) close(fd);
        int64_t first = 0;
        const int64_t pb = ok ? payload_bytes(h.kind, h.dims, &first) : -1;
        if (pb <= 0) {
            delete fs;
            return err(LFG_ERR_INVALID, std::string("not a sample file: ") + paths[i]);
        }
        fs->slot_bytes = std::max(fs->slot_bytes, (pb + 255) / 256 * 256);
    }
    for (int s = 0; s < slots; ++s) {
        void* p = nullptr;
        if (lfg_host_alloc(ctx, static_cast<size_t>(fs->slot_bytes), &p) != LFG_OK) {
            for (char* q : fs->slots) lfg_host_free(ctx, q);
            delete fs;
            return err(LFG_ERR_NOMEM, "pinned slot allocation failed");
        }
        fs->slots.push_back(static_cast<char*>(p));
        fs->free_slots.push_back(s);
    }
    fs->slot_of.assign(static_cast<size_t>(n), -1);
    fs->state.assign(static_cast<size_t>(n), 0);
    for (int r = 0; r < readers; ++r) fs->readers.emplace_back([fs] { fs->reader(); });
    *out = fs;
    return LFG_OK;
}

int lfg_file_source_get(lfg_file_source* fs, lfg_source* out) {
    if (!fs || !out) return err(LFG_ERR_INVALID, "null argument");
    out->user = fs;
    out->next = [](void* u, lfg_sample_desc* d) { return static_cast<lfg_file_source*>(u)->next(d); };
    out->release = [](void* u, uint64_t id) { static_cast<lfg_file_source*>(u)->release(id); };
    return LFG_OK;
}

int lfg_file_source_stats(lfg_file_source* fs, int64_t* bytes_read, double* read_seconds) {
    if (!fs) return err(LFG_ERR_INVALID, "null argument");
    if (bytes_read) *bytes_read = fs->bytes_read.load();
    if (read_seconds) *read_seconds = static_cast<double>(fs->read_ns.load()) * 1e-9;
    return LFG_OK;
}

int lfg_file_source_close(lfg_file_source* fs) {
    if (!fs) return LFG_OK;
    {
        std::lock_guard<std::mutex> lk(fs->mu);
        fs->stop = true;
    }
    fs->cv.notify_all();
    for (auto& t : fs->readers) t.join();
    for (char* q : fs->slots) lfg_host_free(fs->ctx, q);
    delete fs;
    return LFG_OK;
}

const char* lfg_files_last_error(void) { return g_err.c_str(); }

}  // extern "C"
