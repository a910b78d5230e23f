// capi.cu -- error state, device queries and the host drop-in entries.
//
// The host entries are what the reference's ctypes binding would call in
// place of the generated C function (CompiledSdfg.run -> self._fn(*ptrs,
// *syms), codegen.py:875-887): they take the reference's host buffers
// (double*, int64_t*) in its argument order, stage them to HBM, run the
// sm_100a kernel(s) and copy the non-transient containers back.
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace sdfgb {

static thread_local char g_err[1024] = "";

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

// ------------------------------------------------------------ conversions
template <typename S, typename D>
__global__ void convert_kernel(const S* __restrict__ s, D* __restrict__ d, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        d[i] = (D)s[i];
}

template <typename S, typename D>
int convert(const S* s, D* d, int64_t n, cudaStream_t st) {
    if (n <= 0) return SDFGB_OK;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
    convert_kernel<S, D><<<blocks, 256, 0, st>>>(s, d, n);
    SDFGB_LAUNCHED("convert_kernel");
    return SDFGB_OK;
}

// row-strided widening copy: dst[r * dcols + c] = src[r * cols + c]
__global__ void convert_rows_kernel(const double* __restrict__ s, float* __restrict__ d, int64_t rows,
                                    int64_t cols, int64_t dcols) {
    const int64_t n = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        d[(i / cols) * dcols + (i % cols)] = (float)s[i];
}

int convert_rows(const double* s, float* d, int64_t rows, int64_t cols, int64_t dcols, cudaStream_t st) {
    const int64_t n = rows * cols;
    if (n <= 0) return SDFGB_OK;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
    convert_rows_kernel<<<blocks, 256, 0, st>>>(s, d, rows, cols, dcols);
    SDFGB_LAUNCHED("convert_rows_kernel");
    return SDFGB_OK;
}

// ------------------------------------------------------------ device pool
// One growable scratch buffer per slot per device, plus one stream.  Host
// entries are serialised per device (the reference entry is synchronous).
struct DevicePool {
    std::mutex mu;
    void* buf[8] = {};
    size_t cap[8] = {};
    cudaStream_t stream = nullptr;
    cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams for the pipelined entries
    int64_t* pinned = nullptr;                  // small pinned scratch (per-chunk counts)
    size_t pinned_n = 0;
};
DevicePool g_pools[32];

struct Session {
    DevicePool* pool = nullptr;
    std::unique_lock<std::mutex> lock;
    int open() {
        int dev = 0;
        SDFGB_CUDA(cudaGetDevice(&dev));
        pool = &g_pools[dev & 31];
        lock = std::unique_lock<std::mutex>(pool->mu);
        if (!pool->stream) SDFGB_CUDA(cudaStreamCreateWithFlags(&pool->stream, cudaStreamNonBlocking));
        if (!pool->h2d) SDFGB_CUDA(cudaStreamCreateWithFlags(&pool->h2d, cudaStreamNonBlocking));
        if (!pool->d2h) SDFGB_CUDA(cudaStreamCreateWithFlags(&pool->d2h, cudaStreamNonBlocking));
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
    cudaStream_t s() const { return pool->stream; }
};

template <typename T>
int h2d(T* d, const T* h, int64_t n, cudaStream_t s) {
    if (n <= 0) return SDFGB_OK;
    return check_cuda(cudaMemcpyAsync(d, h, (size_t)n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
}
template <typename T>
int d2h(T* h, const T* d, int64_t n, cudaStream_t s) {
    if (n <= 0) return SDFGB_OK;
    return check_cuda(cudaMemcpyAsync(h, d, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
}

}  // namespace
}  // namespace sdfgb

using namespace sdfgb;

extern "C" int sdfgb_abi_version(void) { return SDFGB_ABI_VERSION; }
extern "C" const char* sdfgb_last_error(void) { return g_err; }

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

extern "C" int sdfgb_host_alloc(void** ptr, size_t bytes) {
    return check_cuda(cudaHostAlloc(ptr, std::max<size_t>(bytes, 1), cudaHostAllocPortable), "cudaHostAlloc");
}
extern "C" int sdfgb_host_free(void* ptr) { return check_cuda(cudaFreeHost(ptr), "cudaFreeHost"); }

// ----------------------------------------------------------------- histogram
extern "C" int sdfgb_host_histogram(const double* img, int64_t* hist, int64_t H, int64_t W, int64_t bins,
                                    double scale, double div, int precision) {
    if (H < 0 || W < 0 || bins <= 0 || !hist || (H * W > 0 && !img))
        return set_error(SDFGB_ERR_INVALID, "histogram: bad arguments");
    Session ss;
    SDFGB_TRY(ss.open());
    const int64_t n = H * W;
    double* dimg;
    int64_t* dhist;
    uint64_t* doob;
    SDFGB_TRY(ss.get(0, n, &dimg));
    SDFGB_TRY(ss.get(1, bins + 1, &dhist));
    doob = reinterpret_cast<uint64_t*>(dhist + bins);
    cudaStream_t s = ss.s(), hs = ss.pool->h2d;
    SDFGB_TRY(h2d(dhist, hist, bins, s));
    SDFGB_CUDA(cudaMemsetAsync(doob, 0, 8, s));
    float* dimgf = nullptr;
    if (precision == SDFGB_PREC_FP32) SDFGB_TRY(ss.get(2, n, &dimgf));
    // pipelined: the image streams in on the copy stream while earlier
    // chunks are binned (WCR sum: chunk launches accumulate into `hist`)
    const int64_t chunk = std::max<int64_t>(std::min<int64_t>(n, (int64_t)1 << 21), 1);
    const int64_t nch = (n + chunk - 1) / chunk;
    std::vector<cudaEvent_t> ev(nch);
    int rc = SDFGB_OK;
    for (int64_t i = 0; i < nch; ++i)
        if (rc == SDFGB_OK) rc = check_cuda(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
    for (int64_t i = 0; i < nch && rc == SDFGB_OK; ++i) {
        const int64_t off = i * chunk, len = std::min(chunk, n - off);
        rc = h2d(dimg + off, img + off, len, hs);
        if (rc == SDFGB_OK) rc = check_cuda(cudaEventRecord(ev[i], hs), "event");
        if (rc == SDFGB_OK) rc = check_cuda(cudaStreamWaitEvent(s, ev[i], 0), "wait");
        if (rc != SDFGB_OK) break;
        if (precision == SDFGB_PREC_FP32) {
            rc = convert(dimg + off, dimgf + off, len, s);
            if (rc == SDFGB_OK) rc = sdfgb_hist_f32(dimgf + off, len, scale, div, dhist, bins, doob, s);
        } else {
            rc = sdfgb_hist_f64(dimg + off, len, scale, div, dhist, bins, doob, s);
        }
    }
    if (rc != SDFGB_OK) cudaStreamSynchronize(hs);
    for (int64_t i = 0; i < nch; ++i)
        if (ev[i]) cudaEventDestroy(ev[i]);
    if (rc != SDFGB_OK) return rc;
    uint64_t oob = 0;
    SDFGB_TRY(d2h(&oob, doob, 1, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    if (oob) return set_error(SDFGB_ERR_OOB, "histogram: %llu bin indices out of bounds for 'hist' (size %lld)",
                              (unsigned long long)oob, (long long)bins);
    SDFGB_TRY(d2h(hist, dhist, bins, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    return SDFGB_OK;
}

extern "C" int sdfgb_host_histogram_i64(const int64_t* img, int64_t* hist, int64_t H, int64_t W, int64_t bins) {
    if (H < 0 || W < 0 || bins <= 0 || !hist || (H * W > 0 && !img))
        return set_error(SDFGB_ERR_INVALID, "histogram: bad arguments");
    Session ss;
    SDFGB_TRY(ss.open());
    const int64_t n = H * W;
    int64_t *dimg, *dhist;
    SDFGB_TRY(ss.get(0, n, &dimg));
    SDFGB_TRY(ss.get(1, bins + 1, &dhist));
    uint64_t* doob = reinterpret_cast<uint64_t*>(dhist + bins);
    cudaStream_t s = ss.s();
    SDFGB_TRY(h2d(dimg, img, n, s));
    SDFGB_TRY(h2d(dhist, hist, bins, s));
    SDFGB_CUDA(cudaMemsetAsync(doob, 0, 8, s));
    SDFGB_TRY(sdfgb_hist_i64(dimg, n, dhist, bins, doob, s));
    uint64_t oob = 0;
    SDFGB_TRY(d2h(&oob, doob, 1, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    if (oob) return set_error(SDFGB_ERR_OOB, "histogram: %llu bin indices out of bounds for 'hist' (size %lld)",
                              (unsigned long long)oob, (long long)bins);
    SDFGB_TRY(d2h(hist, dhist, bins, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    return SDFGB_OK;
}

// --------------------------------------------------------------------- query
extern "C" int sdfgb_host_query(const double* col, const double* thr, double* out_vals, int64_t* count,
                                int64_t N, int op, int precision) {
    // Pipelined: the column streams in chunks on a copy stream, each chunk is
    // compacted (into its own slice of the device output) on the compute
    // stream, and each chunk's survivors stream back on a second copy stream
    // to their final offset (the running count) -- H2D, compute and D2H of
    // different chunks overlap.  Order is the input order, as in the
    // reference's FIFO drain.
    if (N < 0 || !thr || !count || (N > 0 && (!col || !out_vals)))
        return set_error(SDFGB_ERR_INVALID, "query: bad arguments");
    if (N == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t cs = ss.s(), hs = ss.pool->h2d, ds = ss.pool->d2h;
    const bool f32 = precision == SDFGB_PREC_FP32;
    const int64_t chunk = std::min<int64_t>(N, (int64_t)1 << 23);
    const int64_t nch = (N + chunk - 1) / chunk;
    double *dcol, *dout;
    SDFGB_TRY(ss.get(0, N, &dcol));
    SDFGB_TRY(ss.get(1, N, &dout));
    float* df = nullptr;
    if (f32) SDFGB_TRY(ss.get(2, 2 * N, &df));
    int64_t* dcnt;
    SDFGB_TRY(ss.get(3, nch, &dcnt));
    const size_t wsb = sdfgb_query_workspace_bytes(chunk, f32 ? 4 : 8);
    uint8_t* wsp;
    SDFGB_TRY(ss.get(4, (int64_t)wsb, &wsp));
    static thread_local void* cleared = nullptr;
    static thread_local size_t cleared_bytes = 0;
    if (cleared != wsp || cleared_bytes < wsb) {
        SDFGB_CUDA(cudaMemsetAsync(wsp, 0, wsb, cs));
        cleared = wsp;
        cleared_bytes = wsb;
    }
    int64_t* hcnt;
    SDFGB_TRY(ss.pinned((size_t)nch, &hcnt));
    SDFGB_CUDA(cudaMemsetAsync(dcnt, 0, (size_t)nch * 8, cs));
    std::vector<cudaEvent_t> ev_in(nch), ev_cnt(nch);
    for (int64_t i = 0; i < nch; ++i) {
        SDFGB_CUDA(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming));
        SDFGB_CUDA(cudaEventCreateWithFlags(&ev_cnt[i], cudaEventDisableTiming));
    }
    cudaEvent_t start;
    SDFGB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    SDFGB_CUDA(cudaEventRecord(start, cs));
    SDFGB_CUDA(cudaStreamWaitEvent(hs, start, 0));  // after the workspace/count clears
    for (int64_t i = 0; i < nch; ++i) {
        const int64_t off = i * chunk, len = std::min(chunk, N - off);
        SDFGB_TRY(h2d(dcol + off, col + off, len, hs));
        SDFGB_CUDA(cudaEventRecord(ev_in[i], hs));
        SDFGB_CUDA(cudaStreamWaitEvent(cs, ev_in[i], 0));
        if (f32) {
            SDFGB_TRY(convert(dcol + off, df + off, len, cs));
            SDFGB_TRY(sdfgb_query_f32(df + off, len, op, thr[0], df + N + off, dcnt + i, wsp, wsb, cs));
        } else {
            SDFGB_TRY(sdfgb_query_f64(dcol + off, len, op, thr[0], dout + off, dcnt + i, wsp, wsb, cs));
        }
        SDFGB_CUDA(cudaMemcpyAsync(hcnt + i, dcnt + i, 8, cudaMemcpyDeviceToHost, cs));
        SDFGB_CUDA(cudaEventRecord(ev_cnt[i], cs));
    }
    int64_t running = count[0];
    int rc = SDFGB_OK;
    for (int64_t i = 0; i < nch && rc == SDFGB_OK; ++i) {
        rc = check_cuda(cudaEventSynchronize(ev_cnt[i]), "query chunk");
        if (rc != SDFGB_OK) break;
        const int64_t off = i * chunk, k = hcnt[i];
        if (k > 0) {
            rc = check_cuda(cudaStreamWaitEvent(ds, ev_cnt[i], 0), "wait");
            // widen this chunk's survivors on the D2H stream (not behind the
            // remaining chunks' kernels), then ship them
            if (f32 && rc == SDFGB_OK) rc = convert(df + N + off, dout + off, k, ds);
            if (rc == SDFGB_OK) rc = d2h(out_vals + (running - count[0]), dout + off, k, ds);
        }
        running += k;
    }
    if (rc == SDFGB_OK) rc = check_cuda(cudaStreamSynchronize(ds), "D2H");
    if (rc == SDFGB_OK) rc = check_cuda(cudaStreamSynchronize(cs), "query");
    for (int64_t i = 0; i < nch; ++i) {
        cudaEventDestroy(ev_in[i]);
        cudaEventDestroy(ev_cnt[i]);
    }
    cudaEventDestroy(start);
    if (rc != SDFGB_OK) return rc;
    count[0] = running;
    return SDFGB_OK;
}

// ---------------------------------------------------------------------- spmv
extern "C" int sdfgb_host_spmv(const int64_t* A_row, const int64_t* A_col, const double* A_val, const double* x,
                               double* b, int64_t H, int64_t W, int64_t nnz, int precision) {
    if (H < 0 || W < 0 || nnz < 0 || !A_row || (H > 0 && !b) || (nnz > 0 && (!A_col || !A_val || !x)))
        return set_error(SDFGB_ERR_INVALID, "spmv: bad arguments");
    if (H == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    int64_t *drow, *dcol;
    double *dval, *dx, *db;
    SDFGB_TRY(ss.get(0, H + 1, &drow));
    SDFGB_TRY(ss.get(1, nnz, &dcol));
    SDFGB_TRY(ss.get(2, nnz, &dval));
    SDFGB_TRY(ss.get(3, W + H, &dx));
    db = dx + W;
    SDFGB_TRY(h2d(drow, A_row, H + 1, s));
    SDFGB_TRY(h2d(dcol, A_col, nnz, s));
    SDFGB_TRY(h2d(dval, A_val, nnz, s));
    SDFGB_TRY(h2d(dx, x, W, s));
    SDFGB_TRY(h2d(db, b, H, s));
    const bool fits32 = nnz < INT32_MAX && W < INT32_MAX;
    if (precision == SDFGB_PREC_FP32 && fits32) {
        int32_t *r32, *c32;
        float *v32, *x32, *b32;
        SDFGB_TRY(ss.get(4, H + 1 + nnz, &r32));
        c32 = r32 + H + 1;
        SDFGB_TRY(ss.get(5, nnz + W + H, &v32));
        x32 = v32 + nnz;
        b32 = x32 + W;
        SDFGB_TRY(convert(drow, r32, H + 1, s));
        SDFGB_TRY(convert(dcol, c32, nnz, s));
        SDFGB_TRY(convert(dval, v32, nnz, s));
        SDFGB_TRY(convert(dx, x32, W, s));
        SDFGB_TRY(convert(db, b32, H, s));
        SDFGB_TRY(sdfgb_spmv_csr_f32(r32, c32, v32, x32, b32, H, s));
        SDFGB_TRY(convert(b32, db, H, s));
    } else {
        SDFGB_TRY(sdfgb_spmv_csr_f64(drow, dcol, dval, dx, db, H, s));
    }
    SDFGB_TRY(d2h(b, db, H, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    return SDFGB_OK;
}

// ------------------------------------------------------------------- jacobi2d
extern "C" int sdfgb_host_jacobi2d(double* A, int64_t N, int64_t T, double coef, const int32_t* di,
                                   const int32_t* dj, int nterms, int precision) {
    if (N < 0 || T < 0 || (N > 0 && !A)) return set_error(SDFGB_ERR_INVALID, "jacobi2d: bad arguments");
    if (N == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    const int64_t n = 2 * N * N;
    double* dA;
    SDFGB_TRY(ss.get(0, n, &dA));
    if (T >= 1 && N > 2) {
        // step 0 overwrites the interior of plane 1 before anything reads it
        // (the map covers [1, N-2]^2): only plane 0 and plane 1's border
        // lines are inputs, a quarter less PCIe traffic than both planes
        const int64_t NN = N * N;
        SDFGB_TRY(h2d(dA, A, NN, s));
        SDFGB_TRY(h2d(dA + NN, A + NN, N, s));
        SDFGB_TRY(h2d(dA + NN + (N - 1) * N, A + NN + (N - 1) * N, N, s));
        for (int64_t c : {(int64_t)0, N - 1})
            SDFGB_CUDA(cudaMemcpy2DAsync(dA + NN + N + c, (size_t)N * 8, A + NN + N + c, (size_t)N * 8, 8,
                                         (size_t)(N - 2), cudaMemcpyHostToDevice, s));
    } else {
        SDFGB_TRY(h2d(dA, A, n, s));
    }
    if (precision == SDFGB_PREC_FP32) {
        float* fA;
        SDFGB_TRY(ss.get(1, n, &fA));
        SDFGB_TRY(convert(dA, fA, n, s));
        SDFGB_TRY(sdfgb_jacobi2d_f32(fA, N, T, coef, di, dj, nterms, s));
        SDFGB_TRY(convert(fA, dA, n, s));
    } else {
        SDFGB_TRY(sdfgb_jacobi2d_f64(dA, N, T, coef, di, dj, nterms, s));
    }
    SDFGB_TRY(d2h(A, dA, n, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    return SDFGB_OK;
}

// --------------------------------------------------------------------- matmul
extern "C" int sdfgb_host_matmul_f64(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
    // native precision: float64 end to end, k-ordered IEEE multiply + add
    if (M < 0 || N < 0 || K < 0 || (M * N > 0 && !C) || (M * K > 0 && !A) || (K * N > 0 && !B))
        return set_error(SDFGB_ERR_INVALID, "matmul: bad arguments");
    if (M == 0 || N == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    double* dd;
    SDFGB_TRY(ss.get(0, M * K + K * N + M * N, &dd));
    double *dA = dd, *dB = dd + M * K, *dC = dB + K * N;
    SDFGB_TRY(h2d(dA, A, M * K, s));
    SDFGB_TRY(h2d(dB, B, K * N, s));
    SDFGB_TRY(sdfgb_gemm_f64(dA, dB, dC, M, N, K, s));
    SDFGB_TRY(d2h(C, dC, M * N, s));
    SDFGB_CUDA(cudaStreamSynchronize(s));
    return SDFGB_OK;
}

extern "C" int sdfgb_host_matmul(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
    if (M < 0 || N < 0 || K < 0 || (M * N > 0 && !C) || (M * K > 0 && !A) || (K * N > 0 && !B))
        return set_error(SDFGB_ERR_INVALID, "matmul: bad arguments");
    if (M == 0 || N == 0) return SDFGB_OK;
    Session ss;
    SDFGB_TRY(ss.open());
    cudaStream_t s = ss.s();
    // K padded to a multiple of 4 with zero columns/rows (TMA row-stride rule)
    const int64_t Kp = (K + 3) / 4 * 4;
    double* dd;
    SDFGB_TRY(ss.get(0, M * K + K * N + M * N, &dd));
    double *dA = dd, *dB = dd + M * K, *dC = dB + K * N;
    float* f;
    SDFGB_TRY(ss.get(1, M * Kp + Kp * N + M * N, &f));
    float *fA = f, *fB = f + M * Kp, *fC = fB + Kp * N;
    cudaStream_t hs = ss.pool->h2d, ds = ss.pool->d2h;
    // Pipelined over row panels of A and C: B comes in first, then each A
    // panel streams in while the previous panel multiplies and the one
    // before ships C back (every C element sees the same k loop, so the
    // panel split does not change results)
    const int64_t prow = std::min<int64_t>(M, std::max<int64_t>(128, (M / 8 + 127) / 128 * 128));
    const int64_t np = (M + prow - 1) / prow;
    void* ws;
    const size_t wsb = sdfgb_gemm_workspace_bytes(prow, N, Kp);
    uint8_t* w8;
    SDFGB_TRY(ss.get(2, (int64_t)wsb, &w8));
    ws = w8;
    std::vector<cudaEvent_t> ev(2 * np + 1);
    int rc = SDFGB_OK;
    for (auto& e : ev)
        if (rc == SDFGB_OK) rc = check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    if (rc == SDFGB_OK) rc = check_cuda(cudaEventRecord(ev[2 * np], s), "event");  // after earlier work on s
    if (rc == SDFGB_OK) rc = check_cuda(cudaStreamWaitEvent(hs, ev[2 * np], 0), "wait");
    if (rc == SDFGB_OK) rc = h2d(dB, B, K * N, hs);
    for (int64_t p = 0; p < np && rc == SDFGB_OK; ++p) {
        const int64_t r0 = p * prow, rows = std::min(prow, M - r0);
        rc = h2d(dA + r0 * K, A + r0 * K, rows * K, hs);
        if (rc == SDFGB_OK) rc = check_cuda(cudaEventRecord(ev[p], hs), "event");
        if (rc == SDFGB_OK) rc = check_cuda(cudaStreamWaitEvent(s, ev[p], 0), "wait");
        if (rc != SDFGB_OK) break;
        if (p == 0) {
            // zero-padded K columns of A / rows of B contribute nothing
            if (Kp != K) rc = check_cuda(cudaMemsetAsync(fA, 0, (size_t)(M * Kp + Kp * N) * 4, s), "memset");
            if (rc == SDFGB_OK) rc = convert(dB, fB, K * N, s);
        }
        if (rc == SDFGB_OK && Kp != K) rc = convert_rows(dA + r0 * K, fA + r0 * Kp, rows, K, Kp, s);
        if (rc == SDFGB_OK && Kp == K) rc = convert(dA + r0 * K, fA + r0 * K, rows * K, s);
        if (rc == SDFGB_OK) rc = sdfgb_gemm_f32(fA + r0 * Kp, fB, fC + r0 * N, rows, N, Kp, ws, wsb, s);
        if (rc == SDFGB_OK) rc = convert(fC + r0 * N, dC + r0 * N, rows * N, s);
        if (rc == SDFGB_OK) rc = check_cuda(cudaEventRecord(ev[np + p], s), "event");
        if (rc == SDFGB_OK) rc = check_cuda(cudaStreamWaitEvent(ds, ev[np + p], 0), "wait");
        if (rc == SDFGB_OK) rc = d2h(C + r0 * N, dC + r0 * N, rows * N, ds);
    }
    const int sync_rc = check_cuda(cudaStreamSynchronize(ds), "D2H");
    cudaStreamSynchronize(hs);
    cudaStreamSynchronize(s);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    if (rc != SDFGB_OK) return rc;
    return sync_rc;
}
