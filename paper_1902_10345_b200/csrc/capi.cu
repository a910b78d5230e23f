// capi.cu -- error state, device queries and the host drop-in entries.
//
// The host entries are what the reference's ctypes binding would call in
// place of the generated C function (CompiledSdfg.run -> self._fn(*ptrs,
// *syms), codegen.py:875-887): they take the reference's host buffers
// (double*, int64_t*) in its argument order, stage them to HBM, run the
// sm_100a kernel(s) and copy the non-transient containers back.
//
// Staging.  Every transfer goes through a ring of pinned slots: host
// threads (hostpool.cpp) convert the next chunk of the caller's buffer into
// a slot while the copy engine drains the previous one, so pageable caller
// memory costs nothing extra (the driver's own pageable path measured
// 11 GB/s against 53 GB/s pinned, profiles/r2_host_narrow.txt).  For the
// fp32 kernels the conversion is the narrowing itself, so PCIe carries 4 B
// per element instead of the reference's 8:
//   * fp32 precision: round to nearest (declared semantics);
//   * native histogram with power-of-two binning: round toward -inf, which
//     keeps floor(v * 2^k) exactly (hostpool.h);
//   * native query: per chunk, narrowed only if every value round-trips,
//     otherwise that chunk runs the float64 kernel -- results are the
//     reference's either way.
// Every entry is synchronous, and its Session drains all three streams on
// every return path, so no copy still reads a caller buffer afterwards.
#include <algorithm>
#include <cmath>
#include <functional>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "hostpool.h"

namespace sdfgb {

static thread_local char g_err[1024] = "";
static thread_local int g_status = SDFGB_OK;

int set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SDFGB_OK;
    return set_error(SDFGB_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

int num_sms() {
    int dev = 0, n = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : kNumSMs;
}

namespace {

// ------------------------------------------------------------ device pool
// Per device: growable scratch buffers, a compute stream and two copy
// streams, the pinned staging ring (kSlots upload + kSlots download slots).
// Host entries are serialised per device (the reference entry is
// synchronous).
constexpr int kSlots = 3;

size_t slot_bytes() {
    static const size_t b = [] {
        const char* e = getenv("SDFGB_STAGE_MB");
        const long mb = e ? atol(e) : 16;
        return (size_t)std::max<long>(mb, 1) << 20;
    }();
    return b;
}

struct DevicePool {
    std::mutex mu;
    void* buf[8] = {};
    size_t cap[8] = {};
    cudaStream_t stream = nullptr;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    int64_t* pinned = nullptr;  // small pinned scratch (counts, flags)
    size_t pinned_n = 0;
    uint8_t* stage = nullptr;  // 2 * kSlots * slot_bytes() pinned
    cudaEvent_t slot_ev[2 * kSlots] = {};
    int next_slot[2] = {0, 0};
    cudaEvent_t mark = nullptr;
    const void* qws_clean = nullptr;  // query workspace known to be all-zero
    size_t qws_bytes = 0;
};
DevicePool g_pools[32];

// ------------------------------------------------------------ conversions
__global__ void widen_kernel(const float* __restrict__ s, double* __restrict__ d, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = (double)s[i];
}

int widen_on_device(const float* s, double* d, int64_t n, cudaStream_t st) {
    if (n <= 0) return SDFGB_OK;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    widen_kernel<<<blocks, 256, 0, st>>>(s, d, n);
    SDFGB_LAUNCHED("widen_kernel");
    return SDFGB_OK;
}

// Page-locked caller memory is DMA'd directly (no host thread touches it);
// pageable memory goes through the staging ring.
bool is_pinned(const void* p, size_t bytes) {
    if (!p || !bytes) return false;
    for (const void* q : {p, static_cast<const void*>(static_cast<const char*>(p) + bytes - 1)}) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (a.type != cudaMemoryTypeHost) return false;
    }
    return true;
}

struct Slot {
    uint8_t* p;
    cudaEvent_t ev;  // recorded after the copy that last used the slot
};

enum { kUp = 0, kDown = 1 };

struct Session {
    DevicePool* pool = nullptr;
    std::unique_lock<std::mutex> lock;

    ~Session() {
        // whatever path the entry returns by (errors included), nothing it
        // queued may still touch the caller's buffers or the pool afterwards
        if (!pool) return;
        if (pool->h2d) cudaStreamSynchronize(pool->h2d);
        if (pool->stream) cudaStreamSynchronize(pool->stream);
        if (pool->d2h) cudaStreamSynchronize(pool->d2h);
    }
    int open() {
        int dev = 0;
        SDFGB_CUDA(cudaGetDevice(&dev));
        DevicePool* p = &g_pools[dev & 31];
        lock = std::unique_lock<std::mutex>(p->mu);
        pool = p;
        if (!p->stream) SDFGB_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
        if (!p->h2d) SDFGB_CUDA(cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking));
        if (!p->d2h) SDFGB_CUDA(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking));
        if (!p->mark) SDFGB_CUDA(cudaEventCreateWithFlags(&p->mark, cudaEventDisableTiming));
        if (!p->stage) {
            SDFGB_CUDA(cudaHostAlloc(&p->stage, 2 * kSlots * slot_bytes(), cudaHostAllocPortable));
            for (auto& e : p->slot_ev) SDFGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        return SDFGB_OK;
    }
    int pinned(size_t n, int64_t** out) {
        if (pool->pinned_n < n) {
            if (pool->pinned) SDFGB_CUDA(cudaFreeHost(pool->pinned));
            pool->pinned = nullptr;
            pool->pinned_n = 0;
            SDFGB_CUDA(cudaHostAlloc(&pool->pinned, n * sizeof(int64_t), cudaHostAllocPortable));
            pool->pinned_n = n;
        }
        *out = pool->pinned;
        return SDFGB_OK;
    }
    template <typename T>
    int get(int slot, int64_t count, T** out) {
        size_t bytes = (size_t)std::max<int64_t>(count, 1) * sizeof(T);
        bytes = (bytes + 255) / 256 * 256;
        if (pool->cap[slot] < bytes) {
            if (pool->buf[slot]) SDFGB_CUDA(cudaFree(pool->buf[slot]));
            pool->buf[slot] = nullptr;
            pool->cap[slot] = 0;
            SDFGB_CUDA(cudaMalloc(&pool->buf[slot], bytes));
            pool->cap[slot] = bytes;
        }
        *out = static_cast<T*>(pool->buf[slot]);
        return SDFGB_OK;
    }
    // the next staging slot of a direction, once its previous copy is done
    int slot(int dir, Slot* out) {
        const int k = dir * kSlots + pool->next_slot[dir];
        pool->next_slot[dir] = (pool->next_slot[dir] + 1) % kSlots;
        SDFGB_CUDA(cudaEventSynchronize(pool->slot_ev[k]));
        out->p = pool->stage + (size_t)k * slot_bytes();
        out->ev = pool->slot_ev[k];
        return SDFGB_OK;
    }
    cudaStream_t s() const { return pool->stream; }
    cudaStream_t up() const { return pool->h2d; }
    cudaStream_t down() const { return pool->d2h; }
};

// Upload n elements of D into dst: for each chunk, fill(off, slot, len) runs
// on the host (it converts the caller's data into the pinned slot; a
// non-zero return aborts), the slot goes H2D on the copy stream, the compute
// stream waits for it, and then(off, len) queues the chunk's compute.
// Elements per staged chunk: about 16 chunks per transfer (fewer leave the
// pipeline's fill and drain exposed, more pay the per-chunk overhead), 2 MB
// at least, one slot at most (tools/stage_grid.sh, profiles/r2_stage_grid.txt)
int64_t chunk_elems(int64_t n, size_t elem, size_t per_elem_bytes = 0) {
    const size_t total = (size_t)std::max<int64_t>(n, 1) * (per_elem_bytes ? per_elem_bytes : elem);
    const size_t bytes = std::min(slot_bytes(), std::max<size_t>(total / 16, (size_t)2 << 20));
    return std::max<int64_t>(1, (int64_t)(bytes / std::max(elem, per_elem_bytes)));
}

template <typename D, typename Fill, typename Then>
int upload(Session& ss, D* dst, int64_t n, Fill&& fill, Then&& then, int64_t chunk = 0) {
    if (chunk <= 0) chunk = chunk_elems(n, sizeof(D));
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t len = std::min(chunk, n - off);
        Slot sl;
        SDFGB_TRY(ss.slot(kUp, &sl));
        SDFGB_TRY(fill(off, reinterpret_cast<D*>(sl.p), len));
        SDFGB_CUDA(cudaMemcpyAsync(dst + off, sl.p, (size_t)len * sizeof(D), cudaMemcpyHostToDevice, ss.up()));
        SDFGB_CUDA(cudaEventRecord(sl.ev, ss.up()));
        SDFGB_CUDA(cudaStreamWaitEvent(ss.s(), sl.ev, 0));
        SDFGB_TRY(then(off, len));
    }
    return SDFGB_OK;
}
constexpr auto kNoCompute = [](int64_t, int64_t) { return SDFGB_OK; };

template <typename T>
int upload_copy(Session& ss, T* dst, const T* src, int64_t n) {
    if (is_pinned(src, (size_t)n * sizeof(T))) {
        SDFGB_CUDA(cudaMemcpyAsync(dst, src, (size_t)n * sizeof(T), cudaMemcpyHostToDevice, ss.up()));
        SDFGB_CUDA(cudaEventRecord(ss.pool->mark, ss.up()));
        return check_cuda(cudaStreamWaitEvent(ss.s(), ss.pool->mark, 0), "wait");
    }
    return upload(ss, dst, n, [&](int64_t off, T* p, int64_t len) {
        host::copy(p, src + off, (size_t)len * sizeof(T));
        return SDFGB_OK;
    }, kNoCompute);
}

// Device -> host through the download slots: each copy lands in a slot on
// the D2H stream, and finish(slot) runs on the host once it has arrived --
// one copy stays in flight while the previous slot is finished.
class DownQueue {
 public:
    explicit DownQueue(Session& ss) : ss_(ss) {}
    // the next copies wait for everything queued on the compute stream so far
    int after_compute() {
        SDFGB_CUDA(cudaEventRecord(ss_.pool->mark, ss_.s()));
        return check_cuda(cudaStreamWaitEvent(ss_.down(), ss_.pool->mark, 0), "wait");
    }
    int push(const void* dev, size_t bytes, std::function<void(const uint8_t*)> finish) {
        while ((int)q_.size() >= kSlots - 1) SDFGB_TRY(pop());
        Slot sl;
        SDFGB_TRY(ss_.slot(kDown, &sl));
        if (bytes) SDFGB_CUDA(cudaMemcpyAsync(sl.p, dev, bytes, cudaMemcpyDeviceToHost, ss_.down()));
        SDFGB_CUDA(cudaEventRecord(sl.ev, ss_.down()));
        q_.push_back({sl, std::move(finish)});
        return SDFGB_OK;
    }
    int drain() {
        while (!q_.empty()) SDFGB_TRY(pop());
        return SDFGB_OK;
    }
    // finish the copies that have already landed, without waiting
    int poll() {
        while (!q_.empty()) {
            const cudaError_t e = cudaEventQuery(q_.front().sl.ev);
            if (e == cudaErrorNotReady) return SDFGB_OK;
            SDFGB_CUDA(e);
            SDFGB_TRY(pop());
        }
        return SDFGB_OK;
    }

 private:
    int pop() {
        Item it = std::move(q_.front());
        q_.erase(q_.begin());
        SDFGB_CUDA(cudaEventSynchronize(it.sl.ev));
        it.finish(it.sl.p);
        return SDFGB_OK;
    }
    struct Item {
        Slot sl;
        std::function<void(const uint8_t*)> finish;
    };
    Session& ss_;
    std::vector<Item> q_;
};

// n elements of S on the device -> host, finish(off, slot, len) per chunk
template <typename S, typename Finish>
int download(Session& ss, const S* src, int64_t n, Finish&& finish) {
    DownQueue dq(ss);
    SDFGB_TRY(dq.after_compute());
    const int64_t chunk = chunk_elems(n, sizeof(S));
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t len = std::min(chunk, n - off);
        SDFGB_TRY(dq.push(src + off, (size_t)len * sizeof(S), [&finish, off, len](const uint8_t* p) {
            finish(off, reinterpret_cast<const S*>(p), len);
        }));
    }
    return dq.drain();
}

template <typename T>
int download_copy(Session& ss, T* dst, const T* src, int64_t n) {
    if (is_pinned(dst, (size_t)n * sizeof(T))) {
        SDFGB_CUDA(cudaEventRecord(ss.pool->mark, ss.s()));
        SDFGB_CUDA(cudaStreamWaitEvent(ss.down(), ss.pool->mark, 0));
        SDFGB_CUDA(cudaMemcpyAsync(dst, src, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost, ss.down()));
        return check_cuda(cudaStreamSynchronize(ss.down()), "D2H");
    }
    return download(ss, src, n, [&](int64_t off, const T* p, int64_t len) {
        host::copy_out(dst + off, p, (size_t)len * sizeof(T));
    });
}
// fp32 results into the caller's float64 container, widened by host threads
// out of the staging slots (half the PCIe bytes; widening on the device and
// DMA'ing float64 into a page-locked container measured slower for the
// large outputs: Jacobi 55.8 vs 46.1 ms, profiles/r2_stage_grid.txt)
int download_widen(Session& ss, double* dst, const float* src, int64_t n) {
    return download(ss, src, n, [&](int64_t off, const float* p, int64_t len) { host::widen(p, dst + off, len); });
}

bool pow2(double x) {
    int e;
    return x > 0 && std::isfinite(x) && std::frexp(x, &e) == 0.5;
}

int remember(int rc) {
    g_status = rc;
    return rc;
}

// ----------------------------------------------------------------- histogram
int host_histogram(const double* img, int64_t* hist, int64_t H, int64_t W, int64_t bins, double scale,
                   double div, int precision) {
    if (H < 0 || W < 0 || bins <= 0 || !hist || (H * W > 0 && !img))
        return set_error(SDFGB_ERR_INVALID, "histogram: bad arguments");
    Session ss;
    SDFGB_TRY(ss.open());
    const int64_t n = H * W;
    cudaStream_t s = ss.s();
    int64_t* dhist;
    SDFGB_TRY(ss.get(1, bins + 1, &dhist));
    uint64_t* doob = reinterpret_cast<uint64_t*>(dhist + bins);
    SDFGB_TRY(upload_copy(ss, dhist, hist, bins));
    SDFGB_CUDA(cudaMemsetAsync(doob, 0, 8, s));
    // floor(v * 2^a / 2^b) of the float64 value survives rounding v toward
    // -inf to fp32 (hostpool.h), so native power-of-two binning ships 4 B
    const bool rd = precision == SDFGB_PREC_NATIVE && pow2(scale) && pow2(div) && bins <= (1 << 24);
    if (rd || precision == SDFGB_PREC_FP32) {
        float* d;
        SDFGB_TRY(ss.get(0, n, &d));
        SDFGB_TRY(upload(ss, d, n, [&](int64_t off, float* p, int64_t len) {
            if (rd) host::narrow_rd(img + off, p, len);
            else host::narrow_rn(img + off, p, len);
            return SDFGB_OK;
        }, [&](int64_t off, int64_t len) { return sdfgb_hist_f32(d + off, len, scale, div, dhist, bins, doob, s); }));
    } else {
        double* d;
        SDFGB_TRY(ss.get(0, n, &d));
        SDFGB_TRY(upload(ss, d, n, [&](int64_t off, double* p, int64_t len) {
            host::copy(p, img + off, (size_t)len * 8);
            return SDFGB_OK;
        }, [&](int64_t off, int64_t len) { return sdfgb_hist_f64(d + off, len, scale, div, dhist, bins, doob, s); }));
    }
    int64_t* h;
    SDFGB_TRY(ss.pinned(1, &h));
    SDFGB_CUDA(cudaMemcpyAsync(h, doob, 8, cudaMemcpyDeviceToHost, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    if (h[0])
        return set_error(SDFGB_ERR_OOB, "histogram: %llu bin indices out of bounds for 'hist' (size %lld)",
                         (unsigned long long)h[0], (long long)bins);
    return download_copy(ss, hist, dhist, bins);
}

int host_histogram_i64(const int64_t* img, int64_t* hist, int64_t H, int64_t W, int64_t bins) {
    if (H < 0 || W < 0 || bins <= 0 || !hist || (H * W > 0 && !img))
        return set_error(SDFGB_ERR_INVALID, "histogram: bad arguments");
    Session ss;
    SDFGB_TRY(ss.open());
    const int64_t n = H * W;
    cudaStream_t s = ss.s();
    int64_t *dimg, *dhist;
    SDFGB_TRY(ss.get(0, n, &dimg));
    SDFGB_TRY(ss.get(1, bins + 1, &dhist));
    uint64_t* doob = reinterpret_cast<uint64_t*>(dhist + bins);
    SDFGB_TRY(upload_copy(ss, dhist, hist, bins));
    SDFGB_CUDA(cudaMemsetAsync(doob, 0, 8, s));
    SDFGB_TRY(upload(ss, dimg, n, [&](int64_t off, int64_t* p, int64_t len) {
        host::copy(p, img + off, (size_t)len * 8);
        return SDFGB_OK;
    }, [&](int64_t off, int64_t len) { return sdfgb_hist_i64(dimg + off, len, dhist, bins, doob, s); }));
    int64_t* h;
    SDFGB_TRY(ss.pinned(1, &h));
    SDFGB_CUDA(cudaMemcpyAsync(h, doob, 8, cudaMemcpyDeviceToHost, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    if (h[0])
        return set_error(SDFGB_ERR_OOB, "histogram: %llu bin indices out of bounds for 'hist' (size %lld)",
                         (unsigned long long)h[0], (long long)bins);
    return download_copy(ss, hist, dhist, bins);
}

// --------------------------------------------------------------------- query
int host_query(const double* col, const double* thr, double* out_vals, int64_t* count, int64_t N, int op,
               int precision) {
    // Pipelined per chunk: host threads narrow the column into a pinned slot
    // (fp32 precision: rounded; native: only if the whole chunk round-trips,
    // else the chunk is copied as float64), the copy engine ships it, the
    // chunk is compacted into its own slice of the device output, and its
    // survivors come back behind it and are widened into out_vals at the
    // running count.  Chunks keep their order, so with SDFGB_QUERY_ORDERED
    // the output is the reference's FIFO order.
    if (N < 0 || !thr || !count || (N > 0 && (!col || !out_vals)))
        return set_error(SDFGB_ERR_INVALID, "query: bad arguments");
    if (N == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    const bool rn = precision == SDFGB_PREC_FP32;
    const int64_t chunk = chunk_elems(N, 8);  // a chunk may fall back to float64
    const int64_t nch = (N + chunk - 1) / chunk;
    uint8_t *dcol, *dout;
    SDFGB_TRY(ss.get(0, nch * chunk * 8, &dcol));
    SDFGB_TRY(ss.get(1, nch * chunk * 8, &dout));
    int64_t* dcnt;
    SDFGB_TRY(ss.get(3, nch, &dcnt));
    const size_t wsb = std::max(sdfgb_query_workspace_bytes(chunk, 4), sdfgb_query_workspace_bytes(chunk, 8));
    uint8_t* wsp;
    SDFGB_TRY(ss.get(4, (int64_t)wsb, &wsp));
    // the workspace resets itself at the end of every launch; after a failed
    // call (or on a new buffer) it is cleared again
    if (ss.pool->qws_clean != wsp || ss.pool->qws_bytes < wsb) SDFGB_CUDA(cudaMemsetAsync(wsp, 0, wsb, s));
    ss.pool->qws_clean = nullptr;
    int64_t* hcnt;
    SDFGB_TRY(ss.pinned((size_t)nch, &hcnt));
    SDFGB_CUDA(cudaMemsetAsync(dcnt, 0, (size_t)nch * 8, s));
    std::vector<char> is32(nch);
    std::vector<cudaEvent_t> ev(nch, nullptr);
    struct Events {  // destroyed on every return path
        std::vector<cudaEvent_t>& v;
        ~Events() {
            for (auto e : v)
                if (e) cudaEventDestroy(e);
        }
    } guard{ev};
    for (auto& e : ev) SDFGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    DownQueue dq(ss);
    int64_t running = count[0];
    // page-locked out_vals: survivors are widened on the device (on the D2H
    // stream, beside the next chunk's compaction) and DMA'd straight in
    const bool direct = is_pinned(out_vals, (size_t)N * 8);
    double* dwide = nullptr;
    if (direct) SDFGB_TRY(ss.get(5, nch * chunk, &dwide));
    auto drain_chunk = [&](int64_t i) -> int {
        SDFGB_CUDA(cudaEventSynchronize(ev[i]));
        const int64_t k = hcnt[i];
        if (k <= 0) return SDFGB_OK;
        SDFGB_CUDA(cudaStreamWaitEvent(ss.down(), ev[i], 0));
        double* dst = out_vals + (running - count[0]);
        running += k;
        const uint8_t* src = dout + (size_t)i * chunk * 8;
        if (direct) {
            const double* from = reinterpret_cast<const double*>(src);
            if (is32[i]) {
                SDFGB_TRY(widen_on_device(reinterpret_cast<const float*>(src), dwide + i * chunk, k, ss.down()));
                from = dwide + i * chunk;
            }
            return check_cuda(cudaMemcpyAsync(dst, from, (size_t)k * 8, cudaMemcpyDeviceToHost, ss.down()), "D2H");
        }
        if (is32[i]) return dq.push(src, (size_t)k * 4, [dst, k](const uint8_t* p) {
            host::widen(reinterpret_cast<const float*>(p), dst, k);
        });
        return dq.push(src, (size_t)k * 8, [dst, k](const uint8_t* p) { host::copy_out(dst, p, (size_t)k * 8); });
    };
    int64_t next_drain = 0;  // chunks before it have their survivors issued
    auto drain_ready = [&](bool block, int64_t upto) -> int {
        for (; next_drain < upto; ++next_drain) {
            if (!block) {
                const cudaError_t e = cudaEventQuery(ev[next_drain]);
                if (e == cudaErrorNotReady) return SDFGB_OK;
                SDFGB_CUDA(e);
            }
            SDFGB_TRY(drain_chunk(next_drain));
        }
        return SDFGB_OK;
    };
    for (int64_t i = 0; i < nch; ++i) {
        const int64_t off = i * chunk, len = std::min(chunk, N - off);
        Slot sl;
        SDFGB_TRY(ss.slot(kUp, &sl));
        float* pf = reinterpret_cast<float*>(sl.p);
        bool f32 = true;
        if (rn) host::narrow_rn(col + off, pf, len);
        else f32 = host::narrow_exact(col + off, pf, len);
        if (!f32) host::copy(sl.p, col + off, (size_t)len * 8);
        is32[i] = f32;
        uint8_t* dc = dcol + (size_t)i * chunk * 8;
        uint8_t* dd = dout + (size_t)i * chunk * 8;
        SDFGB_CUDA(cudaMemcpyAsync(dc, sl.p, (size_t)len * (f32 ? 4 : 8), cudaMemcpyHostToDevice, ss.up()));
        SDFGB_CUDA(cudaEventRecord(sl.ev, ss.up()));
        SDFGB_CUDA(cudaStreamWaitEvent(s, sl.ev, 0));
        if (f32)
            SDFGB_TRY(sdfgb_query_f32(reinterpret_cast<float*>(dc), len, op, thr[0], reinterpret_cast<float*>(dd),
                                      dcnt + i, wsp, wsb, s));
        else
            SDFGB_TRY(sdfgb_query_f64(reinterpret_cast<double*>(dc), len, op, thr[0],
                                      reinterpret_cast<double*>(dd), dcnt + i, wsp, wsb, s));
        SDFGB_CUDA(cudaMemcpyAsync(hcnt + i, dcnt + i, 8, cudaMemcpyDeviceToHost, s));
        SDFGB_CUDA(cudaEventRecord(ev[i], s));
        // survivors of every chunk already compacted go out behind it; the
        // host threads never wait for the GPU here (only for a free slot)
        SDFGB_TRY(drain_ready(false, i + 1));
        SDFGB_TRY(dq.poll());
    }
    SDFGB_TRY(drain_ready(true, nch));
    SDFGB_TRY(dq.drain());
    SDFGB_CUDA(cudaStreamSynchronize(ss.down()));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    ss.pool->qws_clean = wsp;
    ss.pool->qws_bytes = wsb;
    count[0] = running;
    return SDFGB_OK;
}

// ---------------------------------------------------------------------- spmv
int host_spmv(const int64_t* A_row, const int64_t* A_col, const double* A_val, const double* x, double* b,
              int64_t H, int64_t W, int64_t nnz, int precision) {
    if (H < 0 || W < 0 || nnz < 0 || !A_row || (H > 0 && !b) || (nnz > 0 && (!A_col || !A_val || !x)))
        return set_error(SDFGB_ERR_INVALID, "spmv: bad arguments");
    if (H == 0) return SDFGB_OK;
    // the data-dependent ranges must stay inside the containers (the
    // interpreter's bounds checks, interpreter.py:216-233)
    if (A_row[0] < 0 || A_row[H] > nnz || !host::non_decreasing(A_row, H + 1))
        return set_error(SDFGB_ERR_INVALID, "spmv: row pointers out of bounds for the column/value containers");
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    const bool idx32 = nnz <= INT32_MAX && W <= INT32_MAX;
    const bool f32 = precision == SDFGB_PREC_FP32 && idx32;
    int64_t bad = 0;
    auto cols32 = [&](int64_t j0) {
        return [&, j0](int64_t off, int32_t* p, int64_t len) {
            bad += host::narrow_index(A_col + j0 + off, p, len, 0, W);
            return bad ? set_error(SDFGB_ERR_OOB, "spmv: column index out of bounds for 'x' (size %lld)",
                                   (long long)W)
                       : SDFGB_OK;
        };
    };
    // rows go in chunks of about one slot of nonzeros: a chunk's kernel runs
    // while the next chunk's columns and values are converted and shipped
    auto row_chunks = [&](int64_t target, auto&& per_chunk) -> int {
        for (int64_t r0 = 0; r0 < H;) {
            const int64_t* e = std::upper_bound(A_row + r0 + 1, A_row + H + 1, A_row[r0] + target);
            int64_t r1 = std::max<int64_t>(r0 + 1, (int64_t)(e - A_row) - 1);
            SDFGB_TRY(per_chunk(r0, r1, A_row[r0], A_row[r1]));
            r0 = r1;
        }
        return SDFGB_OK;
    };
    if (idx32) {
        int32_t *rp, *ci;
        SDFGB_TRY(ss.get(0, H + 1, &rp));
        SDFGB_TRY(ss.get(1, nnz, &ci));
        SDFGB_TRY(upload(ss, rp, H + 1, [&](int64_t off, int32_t* p, int64_t len) {
            host::narrow_index(A_row + off, p, len, 0, nnz + 1);  // range checked above
            return SDFGB_OK;
        }, kNoCompute));
        if (f32) {
            float *v, *xv, *bv;
            SDFGB_TRY(ss.get(2, nnz, &v));
            SDFGB_TRY(ss.get(5, W + H, &xv));
            bv = xv + W;
            auto rn = [](const double* src) {
                return [src](int64_t off, float* p, int64_t len) {
                    host::narrow_rn(src + off, p, len);
                    return SDFGB_OK;
                };
            };
            SDFGB_TRY(upload(ss, xv, W, rn(x), kNoCompute));
            SDFGB_TRY(upload(ss, bv, H, rn(b), kNoCompute));
            SDFGB_TRY(row_chunks((int64_t)(slot_bytes() / 4), [&](int64_t r0, int64_t r1, int64_t j0, int64_t j1) -> int {
                SDFGB_TRY(upload(ss, ci + j0, j1 - j0, cols32(j0), kNoCompute));
                SDFGB_TRY(upload(ss, v + j0, j1 - j0, rn(A_val + j0), kNoCompute));
                return sdfgb_spmv_csr_f32(rp + r0, ci, v, xv, bv + r0, r1 - r0, s);
            }));
            return download_widen(ss, b, bv, H);
        }
        double *v, *xv, *bv;
        SDFGB_TRY(ss.get(2, nnz, &v));
        SDFGB_TRY(ss.get(5, W + H, &xv));
        bv = xv + W;
        SDFGB_TRY(upload_copy(ss, xv, x, W));
        SDFGB_TRY(upload_copy(ss, bv, b, H));
        SDFGB_TRY(row_chunks((int64_t)(slot_bytes() / 8), [&](int64_t r0, int64_t r1, int64_t j0, int64_t j1) -> int {
            SDFGB_TRY(upload(ss, ci + j0, j1 - j0, cols32(j0), kNoCompute));
            SDFGB_TRY(upload_copy(ss, v + j0, A_val + j0, j1 - j0));
            return spmv_csr_f64_i32(rp + r0, ci, v, xv, bv + r0, r1 - r0, s);
        }));
        return download_copy(ss, b, bv, H);
    }
    // beyond int32 indices: float64 with the int64 containers as they are
    int64_t *rp, *ci;
    double *v, *xv, *bv;
    SDFGB_TRY(ss.get(0, H + 1, &rp));
    SDFGB_TRY(ss.get(1, nnz, &ci));
    SDFGB_TRY(ss.get(2, nnz, &v));
    SDFGB_TRY(ss.get(5, W + H, &xv));
    bv = xv + W;
    SDFGB_TRY(upload_copy(ss, rp, A_row, H + 1));
    SDFGB_TRY(upload(ss, ci, nnz, [&](int64_t off, int64_t* p, int64_t len) {
        host::copy(p, A_col + off, (size_t)len * 8);
        for (int64_t j = 0; j < len; ++j)
            if (p[j] < 0 || p[j] >= W)
                return set_error(SDFGB_ERR_OOB, "spmv: column index out of bounds for 'x' (size %lld)", (long long)W);
        return SDFGB_OK;
    }, kNoCompute));
    SDFGB_TRY(upload_copy(ss, v, A_val, nnz));
    SDFGB_TRY(upload_copy(ss, xv, x, W));
    SDFGB_TRY(upload_copy(ss, bv, b, H));
    SDFGB_TRY(sdfgb_spmv_csr_f64(rp, ci, v, xv, bv, H, s));
    return download_copy(ss, b, bv, H);
}

// ------------------------------------------------------------------- jacobi2d
template <typename T>
int host_jacobi2d_t(double* A, int64_t N, int64_t T_, double coef, const int32_t* di, const int32_t* dj,
                    int nterms) {
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    const int64_t NN = N * N;
    T* dA;
    SDFGB_TRY(ss.get(0, 2 * NN, &dA));
    auto conv = [](const double* src) {
        return [src](int64_t off, T* p, int64_t len) {
            if constexpr (sizeof(T) == 4) host::narrow_rn(src + off, p, len);
            else host::copy(p, src + off, (size_t)len * 8);
            return SDFGB_OK;
        };
    };
    if (T_ >= 1 && N > 2) {
        // step 0 overwrites the interior of plane 1 before anything reads it
        // (the map covers [1, N-2]^2): only plane 0 and plane 1's border
        // lines are inputs
        SDFGB_TRY(upload(ss, dA, NN, conv(A), kNoCompute));
        SDFGB_TRY(upload(ss, dA + NN, N, conv(A + NN), kNoCompute));
        SDFGB_TRY(upload(ss, dA + NN + (N - 1) * N, N, conv(A + NN + (N - 1) * N), kNoCompute));
        // the two border columns, gathered on the host, scattered by 2-D copies
        Slot sl;
        SDFGB_TRY(ss.slot(kUp, &sl));
        T* p = reinterpret_cast<T*>(sl.p);
        const int64_t rows = N - 2;
        if ((size_t)(2 * rows) * sizeof(T) > slot_bytes())
            return set_error(SDFGB_ERR_INVALID, "jacobi2d: N too large for the staging slot");
        for (int64_t r = 0; r < rows; ++r) {
            p[r] = (T)A[NN + (r + 1) * N];
            p[rows + r] = (T)A[NN + (r + 1) * N + N - 1];
        }
        for (int c = 0; c < 2; ++c)
            SDFGB_CUDA(cudaMemcpy2DAsync(dA + NN + N + (c ? N - 1 : 0), (size_t)N * sizeof(T), p + c * rows,
                                         sizeof(T), sizeof(T), (size_t)rows, cudaMemcpyHostToDevice, ss.up()));
        SDFGB_CUDA(cudaEventRecord(sl.ev, ss.up()));
        SDFGB_CUDA(cudaStreamWaitEvent(s, sl.ev, 0));
    } else {
        SDFGB_TRY(upload(ss, dA, 2 * NN, conv(A), kNoCompute));
    }
    if constexpr (sizeof(T) == 4) {
        SDFGB_TRY(sdfgb_jacobi2d_f32(dA, N, T_, coef, di, dj, nterms, s));
        return download_widen(ss, A, dA, 2 * NN);
    } else {
        SDFGB_TRY(sdfgb_jacobi2d_f64(dA, N, T_, coef, di, dj, nterms, s));
        return download_copy(ss, A, dA, 2 * NN);
    }
}

int host_jacobi2d(double* A, int64_t N, int64_t T, double coef, const int32_t* di, const int32_t* dj, int nterms,
                  int precision) {
    if (N < 0 || T < 0 || (N > 0 && !A)) return set_error(SDFGB_ERR_INVALID, "jacobi2d: bad arguments");
    if (N == 0) return SDFGB_OK;
    if (precision == SDFGB_PREC_FP32) return host_jacobi2d_t<float>(A, N, T, coef, di, dj, nterms);
    return host_jacobi2d_t<double>(A, N, T, coef, di, dj, nterms);
}

// --------------------------------------------------------------------- matmul
int host_matmul_f64(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
    // native precision: float64 end to end, k-ordered IEEE multiply + add
    if (M < 0 || N < 0 || K < 0 || (M * N > 0 && !C) || (M * K > 0 && !A) || (K * N > 0 && !B))
        return set_error(SDFGB_ERR_INVALID, "matmul: bad arguments");
    if (M == 0 || N == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    double* dd;
    SDFGB_TRY(ss.get(0, M * K + K * N + M * N, &dd));
    double *dA = dd, *dB = dd + M * K, *dC = dB + K * N;
    SDFGB_TRY(upload_copy(ss, dA, A, M * K));
    SDFGB_TRY(upload_copy(ss, dB, B, K * N));
    SDFGB_TRY(sdfgb_gemm_f64(dA, dB, dC, M, N, K, ss.s()));
    return download_copy(ss, C, dC, M * N);
}

int host_matmul(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
    if (M < 0 || N < 0 || K < 0 || (M * N > 0 && !C) || (M * K > 0 && !A) || (K * N > 0 && !B))
        return set_error(SDFGB_ERR_INVALID, "matmul: bad arguments");
    if (M == 0 || N == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    // K padded to a multiple of 4 with zero columns/rows (TMA row stride)
    const int64_t Kp = (K + 3) / 4 * 4;
    if ((size_t)Kp * 4 > slot_bytes()) return set_error(SDFGB_ERR_INVALID, "matmul: K too large for the staging slot");
    // row panels of A and C: each panel's GEMM runs while the next panel of A
    // is narrowed and shipped and the previous panel of C comes back (every C
    // element sees the same k loop, so the panel split does not change results)
    const int64_t prow = std::min<int64_t>(M, std::max<int64_t>(128, (M / 8 + 127) / 128 * 128));
    auto r256 = [](int64_t n) { return (n + 63) / 64 * 64; };  // floats, 256-byte aligned
    float* f;
    SDFGB_TRY(ss.get(1, r256(M * Kp) + r256(Kp * N) + r256(M * N) + 2 * r256(N * Kp) + 2 * r256(prow * Kp), &f));
    float *fA = f, *fB = fA + r256(M * Kp), *fC = fB + r256(Kp * N);
    float *Bhi = fC + r256(M * N), *Blo = Bhi + r256(N * Kp);
    float *Ahi = Blo + r256(N * Kp), *Alo = Ahi + r256(prow * Kp);
    if (K == 0) {
        SDFGB_CUDA(cudaMemsetAsync(fC, 0, (size_t)M * N * 4, s));  // init_C only (library.py:541-554)
        return download_widen(ss, C, fC, M * N);
    }
    if (Kp != K) SDFGB_CUDA(cudaMemsetAsync(fB + K * N, 0, (size_t)(Kp - K) * N * 4, s));
    SDFGB_TRY(upload(ss, fB, K * N, [&](int64_t off, float* p, int64_t len) {
        host::narrow_rn(B + off, p, len);
        return SDFGB_OK;
    }, kNoCompute));
    GemmB bops;
    SDFGB_TRY(gemm_split_b(fB, Bhi, Blo, Kp, N, s, &bops));  // once for all panels
    DownQueue dq(ss);
    const int64_t rows_per_slot = std::max<int64_t>(1, (int64_t)(slot_bytes() / ((size_t)Kp * 4)));

    for (int64_t r0 = 0; r0 < M; r0 += prow) {
        const int64_t rows = std::min(prow, M - r0);
        SDFGB_TRY(upload(ss, fA + r0 * Kp, rows * Kp, [&](int64_t off, float* p, int64_t len) {
            host::narrow_rows_rn(A + (r0 + off / Kp) * K, p, len / Kp, K, Kp);
            return SDFGB_OK;
        }, kNoCompute, rows_per_slot * Kp));
        SDFGB_TRY(gemm_f32_presplit(fA + r0 * Kp, bops, fC + r0 * N, rows, N, Kp, Ahi, Alo, s));
        SDFGB_TRY(dq.after_compute());
        const int64_t per = (int64_t)(slot_bytes() / 4);
        for (int64_t o = 0; o < rows * N; o += per) {
            const int64_t len = std::min(per, rows * N - o);
            double* dst = C + r0 * N + o;
            SDFGB_TRY(dq.push(fC + r0 * N + o, (size_t)len * 4, [dst, len](const uint8_t* p) {
                host::widen(reinterpret_cast<const float*>(p), dst, len);
            }));
        }
    }
    SDFGB_TRY(dq.drain());
    return check_cuda(cudaStreamSynchronize(ss.down()), "D2H");
}

}  // namespace
}  // namespace sdfgb

using namespace sdfgb;

extern "C" int sdfgb_abi_version(void) { return SDFGB_ABI_VERSION; }
extern "C" const char* sdfgb_last_error(void) { return g_err; }
extern "C" int sdfgb_last_status(void) { return g_status; }
extern "C" int sdfgb_host_threads(void) { return host::threads(); }

extern "C" int sdfgb_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (count) *count = e == cudaSuccess ? n : 0;
    return check_cuda(e, "cudaGetDeviceCount");
}
// Let kernels on the current device reach memory that lives on `peer` (the
// IPC mappings of the P2P entries are made in the owning device's context)
extern "C" int sdfgb_enable_peer_access(int peer) {
    int dev = 0;
    SDFGB_CUDA(cudaGetDevice(&dev));
    if (peer == dev) return SDFGB_OK;
    int can = 0;
    SDFGB_CUDA(cudaDeviceCanAccessPeer(&can, dev, peer));
    if (!can) return set_error(SDFGB_ERR_COMM, "device %d cannot access device %d (no peer path)", dev, peer);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return SDFGB_OK;
    }
    return check_cuda(e, "cudaDeviceEnablePeerAccess");
}

// Cross-rank ordering for kernels that write peer memory: signal stores
// `value` into a flag (usually a peer rank's, over NVLink) once everything
// queued before it on the stream is done and visible system-wide; wait
// holds the stream until a (local) flag reaches `value`.  Flags only grow.
__global__ void flag_signal_kernel(int* flag, int value) {
    __threadfence_system();
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}
__global__ void flag_wait_kernel(const int* flag, int value) {
    int v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v >= value) break;
        __nanosleep(256);
    }
}
extern "C" int sdfgb_flag_signal(int* flag, int value, void* stream) {
    if (!flag) return set_error(SDFGB_ERR_INVALID, "flag_signal: null flag");
    flag_signal_kernel<<<1, 1, 0, as_stream(stream)>>>(flag, value);
    SDFGB_LAUNCHED("flag_signal_kernel");
    return SDFGB_OK;
}
extern "C" int sdfgb_flag_wait(const int* flag, int value, void* stream) {
    if (!flag) return set_error(SDFGB_ERR_INVALID, "flag_wait: null flag");
    flag_wait_kernel<<<1, 1, 0, as_stream(stream)>>>(flag, value);
    SDFGB_LAUNCHED("flag_wait_kernel");
    return SDFGB_OK;
}

extern "C" int sdfgb_host_alloc(void** ptr, size_t bytes) {
    return check_cuda(cudaHostAlloc(ptr, std::max<size_t>(bytes, 1), cudaHostAllocPortable), "cudaHostAlloc");
}
extern "C" int sdfgb_host_free(void* ptr) { return check_cuda(cudaFreeHost(ptr), "cudaFreeHost"); }

// ---------------------------------------------------------- host entries
// Each records its status for sdfgb_last_status(): the per-graph shims that
// carry the reference's exact `void <name>(...)` signature (dispatch.py)
// return nothing, so their callers read the status afterwards.
extern "C" int sdfgb_host_histogram(const double* img, int64_t* hist, int64_t H, int64_t W, int64_t bins,
                                    double scale, double div, int precision) {
    return remember(host_histogram(img, hist, H, W, bins, scale, div, precision));
}
extern "C" int sdfgb_host_histogram_i64(const int64_t* img, int64_t* hist, int64_t H, int64_t W, int64_t bins) {
    return remember(host_histogram_i64(img, hist, H, W, bins));
}
extern "C" int sdfgb_host_query(const double* col, const double* thr, double* out_vals, int64_t* count,
                                int64_t N, int op, int precision) {
    return remember(host_query(col, thr, out_vals, count, N, op, precision));
}
extern "C" int sdfgb_host_spmv(const int64_t* A_row, const int64_t* A_col, const double* A_val, const double* x,
                               double* b, int64_t H, int64_t W, int64_t nnz, int precision) {
    return remember(host_spmv(A_row, A_col, A_val, x, b, H, W, nnz, precision));
}
extern "C" int sdfgb_host_jacobi2d(double* A, int64_t N, int64_t T, double coef, const int32_t* di,
                                   const int32_t* dj, int nterms, int precision) {
    return remember(host_jacobi2d(A, N, T, coef, di, dj, nterms, precision));
}
extern "C" int sdfgb_host_matmul_f64(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
    return remember(host_matmul_f64(A, B, C, M, N, K));
}
extern "C" int sdfgb_host_matmul(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
    return remember(host_matmul(A, B, C, M, N, K));
}

// The host-side conversions of the staging ring, exposed for CPU tests
// (no device needed).  kind: 0 round-to-nearest, 1 toward -inf, 2 exact
// (returns 1 iff every element round-trips), 3 widen, 4 int64 -> int32 with
// the count of elements outside [lo, hi) returned, 5 non-decreasing check.
extern "C" int64_t sdfgb_host_convert(int kind, const void* src, void* dst, int64_t n, int64_t lo, int64_t hi) {
    switch (kind) {
    case 0: host::narrow_rn(static_cast<const double*>(src), static_cast<float*>(dst), n); return 0;
    case 1: host::narrow_rd(static_cast<const double*>(src), static_cast<float*>(dst), n); return 0;
    case 2: return host::narrow_exact(static_cast<const double*>(src), static_cast<float*>(dst), n) ? 1 : 0;
    case 3: host::widen(static_cast<const float*>(src), static_cast<double*>(dst), n); return 0;
    case 4: return host::narrow_index(static_cast<const int64_t*>(src), static_cast<int32_t*>(dst), n, lo, hi);
    case 5: return host::non_decreasing(static_cast<const int64_t*>(src), n) ? 1 : 0;
    default: return -1;
    }
}
