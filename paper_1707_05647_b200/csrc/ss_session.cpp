// ss_session.cpp -- the native host runtime of screen() (screening.py:474-539):
// one C call runs the whole screen of one (image, template) pair -- template
// features (f2) on their own stream, the image upload through pinned staging
// filled by host worker threads, the table build (K1/K2), the key sets on the
// host while the build runs, the fused ladder (K3), the survivor list (K4)
// beside the region (K5) and every result's D2H into the caller's host
// buffers -- with one host synchronisation at the end.  A session owns its
// device and pinned buffers (grown on demand, reused across calls) and its
// streams; it replaces the Python orchestration of engine.py for one screen
// (same kernels, same results), cutting the per-call host cost from about
// half a millisecond of interpreter work to tens of microseconds.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "ss_common.cuh"

namespace {

// ── host worker threads (parallel pageable -> pinned copies) ────────────────
class Workers {
   public:
    static Workers& get() {
        static Workers* w = new Workers();  // never destroyed: its threads sleep until exit
        return *w;
    }
    // fn(i) for every i in [0, n), on the pool and the calling thread
    void run(int n, const std::function<void(int)>& fn) {
        if (n <= 1 || threads_.empty()) {
            for (int i = 0; i < n; ++i) fn(i);
            return;
        }
        Job j;
        j.fn = &fn;
        j.n = n;
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(&j);
            gen_.fetch_add(1, std::memory_order_release);
        }
        if (sleepers_.load() > 0) cv_.notify_all();
        work(&j);
        std::unique_lock<std::mutex> lk(mu_);
        auto it = std::find(q_.begin(), q_.end(), &j);
        if (it != q_.end()) q_.erase(it);
        done_.wait(lk, [&] { return j.done.load() == n && j.users == 0; });
    }
    // get the sleeping workers spinning (they take the next job without a
    // futex wake-up; a sleeping thread's wake-up costs tens of microseconds)
    void wake() {
        if (sleepers_.load() > 0) {
            {
                std::lock_guard<std::mutex> lk(mu_);
                gen_.fetch_add(1, std::memory_order_release);
            }
            cv_.notify_all();
        }
    }
    int size() const { return (int)threads_.size() + 1; }

   private:
    struct Job {
        const std::function<void(int)>* fn = nullptr;
        int n = 0;
        std::atomic<int> next{0}, done{0};
        int users = 0;  // workers inside work(), guarded by mu_
    };
    Workers() {
        const unsigned hw = std::thread::hardware_concurrency();
        const int n = (int)std::min(7u, hw > 1 ? hw - 1 : 0u);
        for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
    }
    static void work(Job* j) {
        int i;
        while ((i = j->next.fetch_add(1)) < j->n) {
            (*j->fn)(i);
            j->done.fetch_add(1);
        }
    }
    void loop() {
        using clock = std::chrono::steady_clock;
        uint64_t seen = gen_.load();
        for (;;) {
            // spin up to 1 ms for new work, then sleep until notified
            const auto until = clock::now() + std::chrono::microseconds(1000);
            while (gen_.load(std::memory_order_acquire) == seen && clock::now() < until) {
#if defined(__x86_64__)
                __builtin_ia32_pause();
#endif
            }
            std::unique_lock<std::mutex> lk(mu_);
            if (gen_.load() == seen && q_.empty()) {
                ++sleepers_;
                cv_.wait(lk, [&] { return gen_.load() != seen || !q_.empty(); });
                --sleepers_;
            }
            seen = gen_.load();
            while (!q_.empty()) {
                Job* j = q_.front();
                if (j->next.load() >= j->n) {
                    q_.pop_front();
                    continue;
                }
                ++j->users;
                lk.unlock();
                work(j);
                lk.lock();
                --j->users;
                if (!q_.empty() && q_.front() == j) q_.pop_front();
                done_.notify_all();
            }
        }
    }
    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::deque<Job*> q_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> sleepers_{0};
    std::vector<std::thread> threads_;
};

void parallel_copy(void* dst, const void* src, size_t bytes) {
    constexpr size_t PART = 128 << 10;
    Workers& w = Workers::get();
    const int parts = (int)std::min<size_t>((size_t)w.size(), (bytes + PART - 1) / PART);
    if (parts <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t per = ((bytes + parts - 1) / parts + 63) & ~(size_t)63;
    w.run(parts, [&](int i) {
        const size_t a = std::min(bytes, (size_t)i * per), b = std::min(bytes, a + per);
        if (b > a) std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
}

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
};
struct HostBuf {
    void* p = nullptr;
    size_t n = 0;
};

int ensure(DevBuf& b, size_t bytes, const char* what) {
    bytes = std::max<size_t>(bytes, 256);
    if (b.n >= bytes) return SS_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.n = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        ss::set_error("session: out of device memory for %s (%zu bytes)", what, bytes);
        return SS_ECUDA;
    }
    b.n = bytes;
    return SS_OK;
}

int ensure(HostBuf& b, size_t bytes, const char* what) {
    bytes = std::max<size_t>(bytes, 256);
    if (b.n >= bytes) return SS_OK;
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.n = 0;
    if (cudaHostAlloc(&b.p, bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        ss::set_error("session: out of pinned host memory for %s (%zu bytes)", what, bytes);
        return SS_ECUDA;
    }
    b.n = bytes;
    return SS_OK;
}

int cuda_ok(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SS_OK;
    cudaGetLastError();
    ss::set_error("session: %s: %s", what, cudaGetErrorString(e));
    return SS_ECUDA;
}

#define SS_TRY(x)                    \
    do {                             \
        if (int e_ = (x)) return e_; \
    } while (0)

// grid_count (config.py; screening.py:433-437): stride-grid coordinates in [lo, limit-1-hi]
int64_t grid_count(int64_t limit, int64_t lo, int64_t hi, int64_t stride) {
    const int64_t top = limit - 1 - hi;
    if (top < lo) return 0;
    const int64_t first = ((lo + stride - 1) / stride) * stride;
    return first > top ? 0 : (top - first) / stride + 1;
}

constexpr int MIN_PATCH_SIDE = 8;  // screening.py:50

// restores the calling thread's current device (a session call switches to the session's)
struct DeviceGuard {
    int dev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&dev) != cudaSuccess) {
            cudaGetLastError();
            dev = -1;
        }
    }
    ~DeviceGuard() {
        if (dev >= 0) cudaSetDevice(dev);
    }
};

// SS_SESSION_TRACE=1: per-phase host times and main-stream GPU times to stderr (experiments)
struct Trace {
    bool on = false;
    std::vector<std::pair<const char*, std::chrono::steady_clock::time_point>> host;
    std::vector<std::pair<const char*, cudaEvent_t>> dev;
    cudaStream_t s = nullptr;
    explicit Trace(cudaStream_t st) : s(st) {
        const char* e = std::getenv("SS_SESSION_TRACE");
        on = e && e[0] == '1';
        mark("start");
    }
    // a host time stamp and an event on `st` (default: the main stream)
    void mark(const char* what, cudaStream_t st = nullptr) {
        if (!on) return;
        host.emplace_back(what, std::chrono::steady_clock::now());
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st ? st : s);
        dev.emplace_back(what, ev);
    }
    ~Trace() {
        if (!on) return;
        cudaDeviceSynchronize();
        std::fprintf(stderr, "[session] (ms since start: host / gpu)");
        for (size_t i = 1; i < host.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, dev[0].second, dev[i].second);
            std::fprintf(stderr, " %s %.3f/%.3f", host[i].first,
                         std::chrono::duration<double, std::milli>(host[i].second - host[0].second).count(), ms);
        }
        std::fprintf(stderr, "\n");
        for (auto& d : dev) cudaEventDestroy(d.second);
    }
};
}  // namespace

struct ss_session {
    int device = 0;
    int64_t W = 0, H = 0, pitch = 0, words = 0;
    cudaStream_t s_main = nullptr, s_tpl = nullptr, s_region = nullptr, s_copy = nullptr;
    cudaEvent_t e_feat = nullptr, e_k3 = nullptr;
    DevBuf img, planes32, planes64, hi16, coarse, build_ws, ladder_ws, masks, row_counts, counts, compact_ws, region,
        region_ws, xy, blobs, tpl, feats, desc;
    HostBuf stage, feats_h, counts_h, blobs_h;
    std::vector<int32_t> desc_last;
    std::vector<int64_t> keys, key_off, boff, blob_off;
    int64_t capacity = 0, last_kept = -1;
    std::mutex mu;
};

namespace {

// the plane decisions of engine.py (needs_int64, wide_as_hi16, coarse_shifts_for)
struct Decisions {
    bool int64 = false, hi16 = false;
    std::vector<int32_t> shifts;
};

Decisions decide(const ss_session& s, const ss_ladder_plan& p) {
    Decisions d;
    bool wide = false;
    std::vector<int> wide_sizes;
    for (int k = 0; k < p.n_sizes; ++k) {
        const int nr = p.n_rings[k];
        if (nr < 1) continue;
        if (!ss_screen_fits32(nr, p.ring_n + (size_t)k * SS_MAX_RINGS, p.ring_d + (size_t)k * SS_MAX_RINGS)) {
            wide = true;
            wide_sizes.push_back(k);
        }
    }
    if (wide) {
        // engine.py wide_as_hi16: the fused rings read 32-bit + hi16 cells (mod 2^48)
        bool ok = s.H < (1 << 24) && s.W <= (1LL << 30) && wide_sizes.size() <= 64;
        int total_rings = 0;
        const __int128 span = std::max(s.W, s.H) + 1;
        for (int k : wide_sizes) {
            const int nr = p.n_rings[k];
            total_rings += nr;
            if (nr > 8) ok = false;
            for (int r = 0; r < nr && ok; ++r) {
                const __int128 n = p.ring_n[(size_t)k * SS_MAX_RINGS + r], dd = p.ring_d[(size_t)k * SS_MAX_RINGS + r];
                const __int128 c = std::max(4 * n * n, 2 * dd * dd + 2 * dd + 1);
                if (255 * c * span >= ((__int128)1 << 48)) ok = false;
                if (r == 0 && 255 * c >= ((__int128)1 << 32)) ok = false;
            }
        }
        if (total_rings > 104) ok = false;
        d.hi16 = ok;
        d.int64 = !ok;
    }
    const char* env = std::getenv("SS_COARSE");
    if (!(env && std::strcmp(env, "0") == 0)) {
        std::set<int32_t> need;
        bool ok = true;
        for (int k = 0; k < p.n_sizes && ok; ++k) {
            if (p.n_rings[k] < 1) continue;
            const int64_t n = p.ring_n[(size_t)k * SS_MAX_RINGS], dd = p.ring_d[(size_t)k * SS_MAX_RINGS];
            for (int64_t count : {4 * n * n, 2 * dd * dd + 2 * dd + 1}) {
                const int32_t sh = ss_coarse_shift(count);
                if (sh < 0) {
                    ok = false;
                    break;
                }
                need.insert(sh);
            }
        }
        if (ok && (int)need.size() <= SS_MAX_COARSE) d.shifts.assign(need.begin(), need.end());
    }
    return d;
}

int screen_locked(ss_session& s, const uint8_t* h_img, const uint8_t* h_tpl, int32_t n, const ss_ladder_plan& p,
                  ss_screen_out& out) {
    const int L = p.n_sizes;
    const int64_t W = s.W, H = s.H, words = s.words;
    SS_TRY(cuda_ok(cudaSetDevice(s.device), "set device"));
    Trace tr(s.s_main);
    const Decisions dec = decide(s, p);

    // patches_tested (screening.py:446, 513) and the first survivor capacity
    int64_t tested = 0;
    for (int k = 0; k < L; ++k) {
        const int m = p.m[k];
        if (m < MIN_PATCH_SIDE) continue;
        const int64_t lo = (m - 1) / 2, hi = m / 2;
        tested += grid_count(W, lo, hi, p.stride) * grid_count(H, lo, hi, p.stride);
    }
    out.tested = tested;

    // buffers (grown on demand; cudaFree / cudaMalloc only when a shape or ladder grows)
    const size_t mask_bytes = (size_t)L * H * words * 4;
    SS_TRY(ensure(s.img, (size_t)W * H, "image"));
    SS_TRY(ensure(s.stage, (size_t)W * H, "image staging"));
    SS_TRY(ensure(s.planes32, ss_tables32_bytes(W, H), "32-bit planes"));
    if (dec.int64) SS_TRY(ensure(s.planes64, ss_tables_bytes(W, H), "int64 planes"));
    if (dec.hi16) SS_TRY(ensure(s.hi16, ss_tables_hi16_bytes(W, H), "hi16 planes"));
    if (!dec.shifts.empty()) SS_TRY(ensure(s.coarse, ss_coarse_bytes(W, H, (int32_t)dec.shifts.size()), "coarse"));
    SS_TRY(ensure(s.build_ws, ss_build_workspace_bytes(W, H), "build workspace"));
    SS_TRY(ensure(s.ladder_ws, ss_ladder_workspace_bytes(W, H, L), "ladder workspace"));
    SS_TRY(ensure(s.masks, mask_bytes, "masks"));
    SS_TRY(ensure(s.row_counts, (size_t)L * H * 4, "row counts"));
    SS_TRY(ensure(s.counts, (size_t)(2 + L) * 8, "counts"));
    SS_TRY(ensure(s.counts_h, (size_t)(2 + L) * 8, "counts"));
    SS_TRY(ensure(s.compact_ws, ss_compact_ladder_workspace_bytes(H, L), "compaction workspace"));
    SS_TRY(ensure(s.region, (size_t)H * words * 4, "region"));
    SS_TRY(ensure(s.region_ws, ss_region_ladder_workspace_bytes(W, H, L), "region workspace"));
    if (s.capacity < 1) s.capacity = std::max<int64_t>(1 << 16, tested / 50);
    SS_TRY(ensure(s.xy, (size_t)s.capacity * 12, "survivor rows"));

    tr.mark("buffers");
    // f2: the template's ring features on their own stream, round trip to pinned memory
    int n_eval = 0;
    for (int k = 0; k < L; ++k) n_eval += p.n_rings[k] > 0;
    if (p.n_inst > 0) {
        const size_t db = (size_t)p.n_inst * p.desc_stride;
        if (s.desc_last.size() != db || std::memcmp(s.desc_last.data(), p.desc, db * 4) != 0) {
            SS_TRY(ensure(s.desc, db * 4, "descriptors"));
            SS_TRY(cuda_ok(cudaMemcpy(s.desc.p, p.desc, db * 4, cudaMemcpyHostToDevice), "descriptor upload"));
            s.desc_last.assign(p.desc, p.desc + db);
        }
        const size_t fb = (size_t)p.n_inst * SS_MAX_RINGS * 3 * sizeof(double);
        SS_TRY(ensure(s.tpl, (size_t)n * n, "template"));
        SS_TRY(ensure(s.feats, fb, "template features"));
        SS_TRY(ensure(s.feats_h, fb, "template features"));
        SS_TRY(ss_template_features_async(h_tpl, n, p.n_inst, static_cast<const int32_t*>(s.desc.p), p.desc_stride,
                                          static_cast<uint8_t*>(s.tpl.p), static_cast<double*>(s.feats.p),
                                          static_cast<double*>(s.feats_h.p), s.s_tpl, s.e_feat));
    }

    tr.mark("f2");
    // the image: straight from the caller's buffer when it is pinned (one DMA
    // per row chunk); else row chunks through pinned staging (worker threads),
    // each chunk's DMA overlapping the next chunk's host copy
    {
        const size_t total = (size_t)W * H;
        cudaPointerAttributes attr{};
        const bool pinned = cudaPointerGetAttributes(&attr, h_img) == cudaSuccess && attr.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (pinned) {
            SS_TRY(cuda_ok(cudaMemcpyAsync(s.img.p, h_img, total, cudaMemcpyHostToDevice, s.s_main), "image upload"));
        } else {
            Workers::get().wake();
            const size_t chunk = std::max<size_t>(total / 4, 1 << 20);
            for (size_t a = 0; a < total; a += chunk) {
                const size_t b = std::min(total, a + chunk);
                parallel_copy(static_cast<uint8_t*>(s.stage.p) + a, h_img + a, b - a);
                SS_TRY(cuda_ok(cudaMemcpyAsync(static_cast<uint8_t*>(s.img.p) + a,
                                               static_cast<uint8_t*>(s.stage.p) + a, b - a, cudaMemcpyHostToDevice,
                                               s.s_main),
                               "image upload"));
            }
        }
    }

    tr.mark("upload");
    // K1/K2
    SS_TRY(ss_build_tables3(static_cast<const uint8_t*>(s.img.p), W, H, W,
                            dec.int64 ? static_cast<int64_t*>(s.planes64.p) : nullptr,
                            static_cast<uint32_t*>(s.planes32.p), dec.hi16 ? static_cast<uint16_t*>(s.hi16.p) : nullptr,
                            s.pitch, dec.shifts.empty() ? nullptr : static_cast<uint16_t*>(s.coarse.p),
                            (int32_t)dec.shifts.size(), dec.shifts.empty() ? nullptr : dec.shifts.data(), s.build_ws.p,
                            s.build_ws.n, s.s_main));

    tr.mark("build");
    // key sets (host, while the GPU builds the tables), blobs to the device
    s.blob_off.assign((size_t)L + 1, 0);
    size_t blob_slots = 1;
    if (n_eval > 0) {
        std::vector<int32_t> nk(p.nk, p.nk + n_eval), nr;
        nr.reserve(n_eval);
        int64_t keys_cap = 0, blobs_cap = 0;
        for (int k = 0; k < L; ++k)
            if (p.n_rings[k] > 0) nr.push_back(p.n_rings[k]);
        for (int i = 0; i < n_eval; ++i) {
            keys_cap += 27LL * nk[i] * nr[i];
            blobs_cap += 1 + 16LL * nr[i] + (int64_t)nr[i] * (81LL * nk[i] + SS_BLOB_MAX_BITMAP_WORDS / 2 + 2);
        }
        s.keys.resize((size_t)std::max<int64_t>(keys_cap, 1));
        s.key_off.resize((size_t)n_eval * (SS_MAX_RINGS + 1) + 1);
        s.boff.resize((size_t)n_eval + 1);
        SS_TRY(ensure(s.blobs_h, (size_t)std::max<int64_t>(blobs_cap, 1) * 8, "key blobs"));
        SS_TRY(cuda_ok(cudaEventSynchronize(s.e_feat), "template features"));
        SS_TRY(ss_ladder_keysets(static_cast<const double*>(s.feats_h.p), SS_MAX_RINGS, n_eval, nk.data(), nr.data(),
                                 p.q_mean, p.q_std, p.q_grad, s.keys.data(), (int64_t)s.keys.size(), s.key_off.data(),
                                 static_cast<int64_t*>(s.blobs_h.p), blobs_cap, s.boff.data()));
        int i = 0;
        for (int k = 0; k < L; ++k) {
            if (p.n_rings[k] > 0) ++i;
            s.blob_off[(size_t)k + 1] = s.boff[(size_t)i];
        }
        blob_slots = std::max<size_t>(1, (size_t)s.boff[(size_t)n_eval]);
    } else {
        SS_TRY(ensure(s.blobs_h, 8, "key blobs"));
        static_cast<int64_t*>(s.blobs_h.p)[0] = 0;
    }
    SS_TRY(ensure(s.blobs, blob_slots * 8, "key blobs"));
    SS_TRY(cuda_ok(cudaMemcpyAsync(s.blobs.p, s.blobs_h.p, blob_slots * 8, cudaMemcpyHostToDevice, s.s_main),
                   "key blob upload"));

    tr.mark("keysets");
    // K3: the fused ladder over the whole image
    void* streams[1] = {s.s_main};
    void* wss[1] = {s.ladder_ws.p};
    SS_TRY(ss_screen_ladder2(dec.int64 ? static_cast<const int64_t*>(s.planes64.p) : nullptr,
                             static_cast<const uint32_t*>(s.planes32.p), W, H, s.pitch, W, H, 0, 0, H, p.stride, L,
                             p.m, p.n_rings, p.ring_n, p.ring_d, static_cast<const int64_t*>(s.blobs.p),
                             static_cast<const int64_t*>(s.blobs_h.p), s.blob_off.data(), p.q_mean, p.q_std, p.q_grad,
                             static_cast<uint32_t*>(s.masks.p), words, H * words,
                             static_cast<uint32_t*>(s.row_counts.p), H, nullptr, 2, 1, streams, wss, s.ladder_ws.n,
                             dec.shifts.empty() ? nullptr : static_cast<const uint16_t*>(s.coarse.p),
                             (int32_t)dec.shifts.size(), dec.shifts.empty() ? nullptr : dec.shifts.data(),
                             dec.hi16 ? static_cast<const uint16_t*>(s.hi16.p) : nullptr));
    SS_TRY(cuda_ok(cudaEventRecord(s.e_k3, s.s_main), "event"));

    tr.mark("K3");
    // the masks' D2H (the largest result) beside K4 / K5
    if (out.masks) {
        SS_TRY(cuda_ok(cudaStreamWaitEvent(s.s_copy, s.e_k3, 0), "event wait"));
        SS_TRY(cuda_ok(cudaMemcpyAsync(out.masks, s.masks.p, mask_bytes, cudaMemcpyDeviceToHost, s.s_copy),
                       "mask readback"));
        tr.mark("masks_d2h", s.s_copy);
    }
    // K5 + popcount + the region's D2H on the region stream
    unsigned long long* d_counts = static_cast<unsigned long long*>(s.counts.p);
    SS_TRY(cuda_ok(cudaStreamWaitEvent(s.s_region, s.e_k3, 0), "event wait"));
    SS_TRY(ss_region_ladder2(static_cast<const uint32_t*>(s.masks.p), words, H * words, W, H, L, p.m, p.stride,
                             static_cast<const uint32_t*>(s.row_counts.p), H, static_cast<uint32_t*>(s.region.p),
                             s.region_ws.p, s.region_ws.n, s.s_region));
    tr.mark("k5_kernels", s.s_region);
    SS_TRY(ss_popcount(static_cast<const uint32_t*>(s.region.p), words, W, H, d_counts + 1, s.s_region));
    unsigned long long* h_counts = static_cast<unsigned long long*>(s.counts_h.p);
    SS_TRY(cuda_ok(cudaMemcpyAsync(h_counts + 1, d_counts + 1, 8, cudaMemcpyDeviceToHost, s.s_region),
                   "count readback"));
    if (out.region)
        SS_TRY(cuda_ok(cudaMemcpyAsync(out.region, s.region.p, (size_t)H * words * 4, cudaMemcpyDeviceToHost,
                                       s.s_region),
                       "region readback"));
    tr.mark("region_d2h", s.s_region);
    // K4 on the main stream, then its counts and (a guess of) the survivor rows
    SS_TRY(ss_compact_ladder(static_cast<const uint32_t*>(s.masks.p), words, H * words, W, H, 0, H, L, p.m, p.stride,
                             static_cast<const uint32_t*>(s.row_counts.p), static_cast<int32_t*>(s.xy.p), 3,
                             s.capacity, d_counts, d_counts + 2, s.compact_ws.p, s.compact_ws.n, s.s_main));
    SS_TRY(cuda_ok(cudaMemcpyAsync(h_counts, d_counts, 8, cudaMemcpyDeviceToHost, s.s_main), "count readback"));
    SS_TRY(cuda_ok(cudaMemcpyAsync(h_counts + 2, d_counts + 2, (size_t)L * 8, cudaMemcpyDeviceToHost, s.s_main),
                   "count readback"));
    tr.mark("K4+counts");
    int64_t guess = s.last_kept < 0 ? 0 : s.last_kept + s.last_kept / 4 + 4096;
    guess = std::min(guess, std::min(s.capacity, out.rows ? out.rows_cap : 0));
    if (guess > 0)
        SS_TRY(cuda_ok(cudaMemcpyAsync(out.rows, s.xy.p, (size_t)guess * 12, cudaMemcpyDeviceToHost, s.s_main),
                       "row readback"));
    tr.mark("rows_d2h");
    SS_TRY(cuda_ok(cudaStreamSynchronize(s.s_region), "region"));
    SS_TRY(cuda_ok(cudaStreamSynchronize(s.s_main), "screen"));
    SS_TRY(cuda_ok(cudaStreamSynchronize(s.s_copy), "mask readback"));

    tr.mark("sync");
    const unsigned long long* hc = static_cast<const unsigned long long*>(s.counts_h.p);
    const int64_t kept = (int64_t)hc[0];
    out.kept = kept;
    out.region_pixels = (int64_t)hc[1];
    if (out.size_counts)
        for (int k = 0; k < L; ++k) out.size_counts[k] = (int64_t)hc[2 + k];
    s.last_kept = kept;
    if (kept > s.capacity) {  // the survivor buffer overflowed: grow it and redo K4
        s.capacity = kept + kept / 4;
        SS_TRY(ensure(s.xy, (size_t)s.capacity * 12, "survivor rows"));
        SS_TRY(ss_compact_ladder(static_cast<const uint32_t*>(s.masks.p), words, H * words, W, H, 0, H, L, p.m,
                                 p.stride, static_cast<const uint32_t*>(s.row_counts.p),
                                 static_cast<int32_t*>(s.xy.p), 3, s.capacity, d_counts, d_counts + 2,
                                 s.compact_ws.p, s.compact_ws.n, s.s_main));
        guess = 0;
    }
    if (kept > (out.rows ? out.rows_cap : 0)) {
        ss::set_error("session: %lld survivor rows, the output holds %lld (ss_session_rows)", (long long)kept,
                      (long long)(out.rows ? out.rows_cap : 0));
        return SS_ECAPACITY;
    }
    if (kept > guess)
        SS_TRY(cuda_ok(cudaMemcpyAsync(static_cast<int32_t*>(out.rows) + guess * 3,
                                       static_cast<const int32_t*>(s.xy.p) + guess * 3, (size_t)(kept - guess) * 12,
                                       cudaMemcpyDeviceToHost, s.s_main),
                       "row readback"));
    SS_TRY(cuda_ok(cudaStreamSynchronize(s.s_main), "row readback"));
    return SS_OK;
}

void destroy(ss_session* s) {
    if (!s) return;
    DeviceGuard guard;
    cudaSetDevice(s->device);
    for (DevBuf* b : {&s->img, &s->planes32, &s->planes64, &s->hi16, &s->coarse, &s->build_ws, &s->ladder_ws,
                      &s->masks, &s->row_counts, &s->counts, &s->compact_ws, &s->region, &s->region_ws, &s->xy,
                      &s->blobs, &s->tpl, &s->feats, &s->desc})
        if (b->p) cudaFree(b->p);
    for (HostBuf* b : {&s->stage, &s->feats_h, &s->counts_h, &s->blobs_h})
        if (b->p) cudaFreeHost(b->p);
    for (cudaStream_t st : {s->s_main, s->s_tpl, s->s_region, s->s_copy})
        if (st) cudaStreamDestroy(st);
    for (cudaEvent_t e : {s->e_feat, s->e_k3})
        if (e) cudaEventDestroy(e);
    delete s;
}

}  // namespace

extern "C" int ss_session_create(int32_t device, int64_t W, int64_t H, ss_session** out) {
    if (!out || W < 1 || H < 1 || W > (1LL << 31) || H > (1LL << 31)) {
        ss::set_error("bad session arguments");
        return SS_EINVAL;
    }
    *out = nullptr;
    DeviceGuard guard;
    ss_session* s = new ss_session();
    s->device = device;
    s->W = W;
    s->H = H;
    s->pitch = ss_plane_pitch(W);
    s->words = (W + 31) / 32;
    int e = cuda_ok(cudaSetDevice(device), "set device");
    for (cudaStream_t* st : {&s->s_main, &s->s_tpl, &s->s_region, &s->s_copy})
        if (!e) e = cuda_ok(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t* ev : {&s->e_feat, &s->e_k3})
        if (!e) e = cuda_ok(cudaEventCreateWithFlags(ev, cudaEventDisableTiming), "event");
    if (e) {
        destroy(s);
        return e;
    }
    *out = s;
    return SS_OK;
}

extern "C" void ss_session_destroy(ss_session* s) { destroy(s); }

extern "C" int ss_session_screen(ss_session* s, const uint8_t* h_img, const uint8_t* h_template, int32_t n,
                                 const ss_ladder_plan* plan, ss_screen_out* out) {
    if (!s || !h_img || !h_template || !plan || !out || n < MIN_PATCH_SIDE || plan->n_sizes < 1 ||
        plan->n_sizes > SS_MAX_SIZES || !plan->m || !plan->n_rings || !plan->ring_n || !plan->ring_d ||
        plan->stride < 1 || plan->n_inst < 0 || (plan->n_inst > 0 && (!plan->desc || !plan->nk)) ||
        plan->desc_stride < 4 + 2 * SS_MAX_RINGS || (out->rows_cap > 0 && !out->rows)) {
        ss::set_error("bad session screen arguments");
        return SS_EINVAL;
    }
    std::lock_guard<std::mutex> lk(s->mu);
    out->kept = out->region_pixels = out->tested = 0;
    DeviceGuard guard;  // the caller's current device is restored on return
    return screen_locked(*s, h_img, h_template, n, *plan, *out);
}

extern "C" int ss_session_rows(ss_session* s, int32_t* h_rows, int64_t first, int64_t count) {
    if (!s || (count > 0 && !h_rows) || first < 0 || count < 0) {
        ss::set_error("bad session row arguments");
        return SS_EINVAL;
    }
    std::lock_guard<std::mutex> lk(s->mu);
    if (first + count > std::min(s->capacity, std::max<int64_t>(s->last_kept, 0))) {
        ss::set_error("session rows [%lld, %lld) beyond the last screen's %lld survivors", (long long)first,
                      (long long)(first + count), (long long)s->last_kept);
        return SS_EINVAL;
    }
    if (count == 0) return SS_OK;
    DeviceGuard guard;
    SS_TRY(cuda_ok(cudaSetDevice(s->device), "set device"));
    return cuda_ok(cudaMemcpy(h_rows, static_cast<const int32_t*>(s->xy.p) + first * 3, (size_t)count * 12,
                              cudaMemcpyDeviceToHost),
                   "row readback");
}
