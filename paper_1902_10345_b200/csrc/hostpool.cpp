// hostpool.cpp -- persistent host worker threads and the staging
// conversions of the drop-in entries (see hostpool.h).
#include "hostpool.h"

#include <immintrin.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#define SDFGB_SIMD __attribute__((target_clones("avx512f", "avx2", "default")))

namespace sdfgb {
namespace host {
namespace {

class Pool {
 public:
    explicit Pool(int n) {
        for (int i = 1; i < n; ++i) workers_.emplace_back([this] { work(); });
        for (auto& t : workers_) t.detach();  // the pool is never destroyed (see get())
    }
    int size() const { return (int)workers_.size() + 1; }

    void run(int64_t ntasks, const std::function<void(int64_t)>& fn) {
        if (ntasks <= 0) return;
        std::lock_guard<std::mutex> job(job_mu_);
        if (ntasks == 1 || workers_.empty()) {
            for (int64_t t = 0; t < ntasks; ++t) fn(t);
            return;
        }
        {
            std::unique_lock<std::mutex> lk(mu_);
            // a worker that picked up the previous job may still be about to
            // take (and find no) task from it: reset only once it has left
            while (active_.load(std::memory_order_acquire) > 0) {
                lk.unlock();
                std::this_thread::yield();
                lk.lock();
            }
            fn_ = &fn;
            ntasks_ = ntasks;
            next_.store(0, std::memory_order_relaxed);
            done_.store(0, std::memory_order_relaxed);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        drain(&fn, ntasks);
        while (done_.load(std::memory_order_acquire) < ntasks) std::this_thread::yield();
    }

 private:
    void drain(const std::function<void(int64_t)>* fn, int64_t nt) {
        for (int64_t t; (t = next_.fetch_add(1, std::memory_order_acq_rel)) < nt;) {
            (*fn)(t);
            done_.fetch_add(1, std::memory_order_acq_rel);
        }
    }
    void work() {
        uint64_t seen = 0;
        for (;;) {
            // the host entries issue jobs back to back (one per staged chunk):
            // poll for the next one for a while before sleeping, so a job
            // does not pay a futex wake-up per worker
            const auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; gen_.load(std::memory_order_acquire) == seen; ++i) {
                spin_pause();
                if ((i & 255) == 255 && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(kSpinUs))
                    break;
            }
            const std::function<void(int64_t)>* fn;
            int64_t nt;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_relaxed) != seen; });
                seen = gen_.load(std::memory_order_relaxed);
                fn = fn_;
                nt = ntasks_;
                active_.fetch_add(1, std::memory_order_acq_rel);
            }
            drain(fn, nt);
            active_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    static void spin_pause() {
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    static inline const int kSpinUs = [] {
        const char* e = getenv("SDFGB_HOST_SPIN_US");
        return e ? atoi(e) : 200;
    }();

    std::mutex job_mu_, mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    const std::function<void(int64_t)>* fn_ = nullptr;
    int64_t ntasks_ = 0;
    std::atomic<int64_t> next_{0}, done_{0};
    std::atomic<int> active_{0};
    std::vector<std::thread> workers_;
};

std::mutex g_mu;
Pool* g_pool = nullptr;
pid_t g_pid = 0;

Pool& get() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_pool || g_pid != getpid()) {  // first use, or a forked child (no workers)
        int n = (int)std::thread::hardware_concurrency();
        if (const char* e = getenv("SDFGB_HOST_THREADS")) n = atoi(e);
        g_pool = new Pool(std::max(1, std::min(n, 64)));  // leaked: workers never outlive it
        g_pid = getpid();
    }
    return *g_pool;
}

// elements per task (default 2^15: 256 KB of float64, so even a small
// staging chunk spreads over every thread); SDFGB_HOST_GRAIN overrides
const int64_t kGrain = [] {
    const char* e = getenv("SDFGB_HOST_GRAIN");
    const long g = e ? atol(e) : (1L << 15);
    return (int64_t)std::max<long>(g, 1024);
}();

template <typename F>
void blocks(int64_t n, F&& f) {
    if (n <= 0) return;
    const int64_t nt = (n + kGrain - 1) / kGrain;
    parallel_for(nt, [&](int64_t t) {
        const int64_t b = t * kGrain;
        f(b, std::min(n, b + kGrain));
    });
}

SDFGB_SIMD void k_narrow_rn(const double* __restrict s, float* __restrict d, int64_t n) {
    for (int64_t i = 0; i < n; ++i) d[i] = (float)s[i];
}

SDFGB_SIMD void k_narrow_rd(const double* __restrict s, float* __restrict d, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const double v = s[i];
        const float f = (float)v;
        uint32_t b;
        memcpy(&b, &f, 4);
        // rounded up: step one ulp towards -inf (+1 on the magnitude when
        // negative; -0.0 -> the negative subnormal; +inf -> FLT_MAX)
        b += ((double)f > v) ? ((b >> 31) ? 1u : 0xffffffffu) : 0u;
        memcpy(d + i, &b, 4);
    }
}

SDFGB_SIMD int k_narrow_exact(const double* __restrict s, float* __restrict d, int64_t n) {
    int ok = 1;
    for (int64_t i = 0; i < n; ++i) {
        const float f = (float)s[i];
        d[i] = f;
        ok &= ((double)f == s[i]);
    }
    return ok;
}

SDFGB_SIMD void k_widen(const float* __restrict s, double* __restrict d, int64_t n) {
    for (int64_t i = 0; i < n; ++i) d[i] = (double)s[i];
}

// Widening into the caller's (large, cold) buffer: streaming stores skip
// the read-for-ownership of every destination line -- a third less DRAM
// traffic on a host whose memory bandwidth, not PCIe, bounds the drain.
__attribute__((target("avx512f"))) void k_widen_nt512(const float* __restrict s, double* __restrict d,
                                                      int64_t n) {
    int64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 63); ++i) d[i] = (double)s[i];
    for (; i + 8 <= n; i += 8) _mm512_stream_pd(d + i, _mm512_cvtps_pd(_mm256_loadu_ps(s + i)));
    for (; i < n; ++i) d[i] = (double)s[i];
    _mm_sfence();
}
__attribute__((target("avx2"))) void k_widen_nt256(const float* __restrict s, double* __restrict d, int64_t n) {
    int64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = (double)s[i];
    for (; i + 4 <= n; i += 4) _mm256_stream_pd(d + i, _mm256_cvtps_pd(_mm_loadu_ps(s + i)));
    for (; i < n; ++i) d[i] = (double)s[i];
    _mm_sfence();
}
__attribute__((target("avx2"))) void k_copy_nt256(const uint8_t* __restrict s, uint8_t* __restrict d, int64_t n) {
    int64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    for (; i < n; ++i) d[i] = s[i];
    _mm_sfence();
}
const bool g_avx512 = __builtin_cpu_supports("avx512f");
const bool g_avx2 = __builtin_cpu_supports("avx2");

SDFGB_SIMD int64_t k_narrow_index(const int64_t* __restrict s, int32_t* __restrict d, int64_t n, int64_t lo,
                                  int64_t hi) {
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t v = s[i];
        d[i] = (int32_t)v;
        bad += (v < lo) | (v >= hi);
    }
    return bad;
}

}  // namespace

void parallel_for(int64_t ntasks, const std::function<void(int64_t)>& fn) { get().run(ntasks, fn); }
int threads() { return get().size(); }

void narrow_rn(const double* s, float* d, int64_t n) {
    blocks(n, [&](int64_t b, int64_t e) { k_narrow_rn(s + b, d + b, e - b); });
}
void narrow_rd(const double* s, float* d, int64_t n) {
    blocks(n, [&](int64_t b, int64_t e) { k_narrow_rd(s + b, d + b, e - b); });
}
bool narrow_exact(const double* s, float* d, int64_t n) {
    std::atomic<int> ok{1};
    blocks(n, [&](int64_t b, int64_t e) {
        if (!k_narrow_exact(s + b, d + b, e - b)) ok.store(0, std::memory_order_relaxed);
    });
    return ok.load() != 0;
}
void widen(const float* s, double* d, int64_t n) {
    blocks(n, [&](int64_t b, int64_t e) {
        if (g_avx512) k_widen_nt512(s + b, d + b, e - b);
        else if (g_avx2) k_widen_nt256(s + b, d + b, e - b);
        else k_widen(s + b, d + b, e - b);
    });
}
void copy_out(void* dst, const void* src, size_t bytes) {
    if (!g_avx2) return copy(dst, src, bytes);
    const int64_t grain = kGrain * 8;
    const int64_t n = (int64_t)bytes, nt = (n + grain - 1) / grain;
    parallel_for(nt, [&](int64_t t) {
        const int64_t b = t * grain, e = std::min(n, b + grain);
        k_copy_nt256(static_cast<const uint8_t*>(src) + b, static_cast<uint8_t*>(dst) + b, e - b);
    });
}
int64_t narrow_index(const int64_t* s, int32_t* d, int64_t n, int64_t lo, int64_t hi) {
    std::atomic<int64_t> bad{0};
    blocks(n, [&](int64_t b, int64_t e) {
        const int64_t k = k_narrow_index(s + b, d + b, e - b, lo, hi);
        if (k) bad.fetch_add(k, std::memory_order_relaxed);
    });
    return bad.load();
}
bool non_decreasing(const int64_t* s, int64_t n) {
    std::atomic<int> ok{1};
    blocks(n, [&](int64_t b, int64_t e) {
        // each block also compares its first element with its predecessor
        for (int64_t i = std::max<int64_t>(b, 1); i < e; ++i)
            if (s[i] < s[i - 1]) {
                ok.store(0, std::memory_order_relaxed);
                return;
            }
    });
    return ok.load() != 0;
}
void copy(void* dst, const void* src, size_t bytes) {
    const int64_t n = (int64_t)(bytes / 8), tail = (int64_t)(bytes % 8);
    blocks(n, [&](int64_t b, int64_t e) {
        memcpy(static_cast<char*>(dst) + b * 8, static_cast<const char*>(src) + b * 8, (size_t)(e - b) * 8);
    });
    if (tail) memcpy(static_cast<char*>(dst) + n * 8, static_cast<const char*>(src) + n * 8, (size_t)tail);
}
void narrow_rows_rn(const double* s, float* d, int64_t rows, int64_t cols, int64_t dcols) {
    if (cols == dcols) return narrow_rn(s, d, rows * cols);
    const int64_t per = std::max<int64_t>(1, kGrain / std::max<int64_t>(cols, 1));
    parallel_for((rows + per - 1) / per, [&](int64_t t) {
        for (int64_t r = t * per; r < std::min(rows, (t + 1) * per); ++r) {
            k_narrow_rn(s + r * cols, d + r * dcols, cols);
            for (int64_t c = cols; c < dcols; ++c) d[r * dcols + c] = 0.0f;
        }
    });
}

}  // namespace host
}  // namespace sdfgb
