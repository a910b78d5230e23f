// mgpu.cu -- the multi-GPU (one process per GPU) entries of the C ABI: each
// is one rank's share of a motif plus the exchange step SURVEY.md §8e names,
// done with NCCL on the caller's communicator and stream.  They restate
// paper_1902_10345_b200/multigpu.py (the torch.distributed version) for hosts
// that are not Python:
//
//   histogram  local partial bins -> ncclAllReduce(sum) -> hist += partial
//   query      local compaction -> ncclAllGather(counts) -> global offsets
//   spmv       ncclAllGather(x shards) -> local row block
//   jacobi     row slabs with GHOST-row ghost zones, one grouped
//              ncclSend/ncclRecv per temporal block of up to GHOST steps,
//              issued on a side stream as soon as the edge bands are done
//              and overlapped with the interior band
//   gemm       P x Q grid: ncclAllGather of the B column panel in the grid
//              column, then the A row panel's pieces broadcast in the grid
//              row on a side stream, each piece's C rows computed as soon
//              as it lands
//
// Every decomposition keeps each element's operation order, so results are
// bit-identical to the one-GPU entries (SpMV rows and GEMM's K stay whole).
//
// NCCL is opened at run time (dlopen of libnccl.so.2): the library has no
// link-time NCCL dependency, and inside a PyTorch process it shares the NCCL
// torch already loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

extern "C" {
int sdfgb_hist_f32(const float* img, int64_t n, double scale, double div, int64_t* hist, int64_t bins,
                   uint64_t* oob, void* stream);
int sdfgb_query_f32(const float* col, int64_t n, int op, double thr, float* out_vals, int64_t* count, void* ws,
                    size_t ws_bytes, void* stream);
int sdfgb_spmv_csr_f32(const int32_t* rowptr, const int32_t* col, const float* val, const float* x, float* b,
                       int64_t H, void* stream);
int sdfgb_jacobi2d_block_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k, double coef,
                             void* stream);
int sdfgb_jacobi2d_band_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k, int64_t r0, int64_t r1,
                            double coef, void* stream);
int sdfgb_gemm_f32_ex(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K, void* ws,
                      size_t ws_bytes, int flags, void* stream);
int sdfgb_gemm_f32(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K, void* ws,
                   size_t ws_bytes, void* stream);
}

namespace sdfgb {
namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclCommCount) commCount = nullptr;
    decltype(&ncclCommUserRank) commUserRank = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    bool ok = false;
    char why[256] = "";
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(api.why, sizeof(api.why), "libnccl.so.2 not found: %s", dlerror());
            return;
        }
#define SDFGB_NCCL_SYM(field, name)                                                  \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));               \
    if (!api.field) {                                                                \
        snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks %s", name);           \
        return;                                                                      \
    }
        SDFGB_NCCL_SYM(getUniqueId, "ncclGetUniqueId")
        SDFGB_NCCL_SYM(commInitRank, "ncclCommInitRank")
        SDFGB_NCCL_SYM(commDestroy, "ncclCommDestroy")
        SDFGB_NCCL_SYM(commCount, "ncclCommCount")
        SDFGB_NCCL_SYM(commUserRank, "ncclCommUserRank")
        SDFGB_NCCL_SYM(allReduce, "ncclAllReduce")
        SDFGB_NCCL_SYM(allGather, "ncclAllGather")
        SDFGB_NCCL_SYM(broadcast, "ncclBroadcast")
        SDFGB_NCCL_SYM(send, "ncclSend")
        SDFGB_NCCL_SYM(recv, "ncclRecv")
        SDFGB_NCCL_SYM(groupStart, "ncclGroupStart")
        SDFGB_NCCL_SYM(groupEnd, "ncclGroupEnd")
        SDFGB_NCCL_SYM(errorString, "ncclGetErrorString")
#undef SDFGB_NCCL_SYM
        api.ok = true;
    });
    return api;
}

int nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return SDFGB_OK;
    return set_error(SDFGB_ERR_COMM, "%s: %s", what, nccl().errorString(r));
}
#define SDFGB_NCCL(expr) SDFGB_TRY(::sdfgb::nccl_check((expr), #expr))
#define SDFGB_NEED_NCCL()                                                                    \
    do {                                                                                     \
        if (!::sdfgb::nccl().ok) return set_error(SDFGB_ERR_COMM, "%s", ::sdfgb::nccl().why); \
    } while (0)

// A side stream plus events for overlapping exchanges with compute; every
// return path waits for the side stream's work on the caller's stream and
// frees both (RAII), so nothing is left in flight on error.
struct SideStream {
    cudaStream_t main = nullptr, side = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int rc = SDFGB_OK;
    explicit SideStream(cudaStream_t m) : main(m) {
        rc = check_cuda(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "cudaStreamCreate");
        for (int i = 0; i < 2 && rc == SDFGB_OK; ++i)
            rc = check_cuda(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    // side waits for everything queued on main so far
    int fork() {
        SDFGB_CUDA(cudaEventRecord(ev[0], main));
        return check_cuda(cudaStreamWaitEvent(side, ev[0], 0), "cudaStreamWaitEvent");
    }
    // main waits for everything queued on side so far
    int join() {
        SDFGB_CUDA(cudaEventRecord(ev[1], side));
        return check_cuda(cudaStreamWaitEvent(main, ev[1], 0), "cudaStreamWaitEvent");
    }
    ~SideStream() {
        if (side) {
            join();
            cudaStreamDestroy(side);
        }
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

int comm_shape(ncclComm_t c, int* rank, int* world) {
    SDFGB_NCCL(nccl().commUserRank(c, rank));
    SDFGB_NCCL(nccl().commCount(c, world));
    return SDFGB_OK;
}

__global__ void hist_fold_kernel(int64_t* __restrict__ hist, uint64_t* __restrict__ oob,
                                 const int64_t* __restrict__ part, int64_t bins) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= bins; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < bins)
            hist[i] += part[i];
        else
            *oob += (uint64_t)part[bins];
    }
}

// counts[world] (all ranks' survivor counts) -> count[0] += total;
// offset[0] = survivors on lower ranks (this rank's global output offset)
__global__ void query_fold_kernel(const int64_t* __restrict__ counts, int world, int rank, int64_t* count,
                                  int64_t* offset) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t total = 0, below = 0;
    for (int r = 0; r < world; ++r) {
        if (r < rank) below += counts[r];
        total += counts[r];
    }
    count[0] += total;
    offset[0] = below;
}

}  // namespace
}  // namespace sdfgb

using namespace sdfgb;

extern "C" int sdfgb_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int sdfgb_nccl_unique_id(void* id_out) {
    SDFGB_NEED_NCCL();
    if (!id_out) return set_error(SDFGB_ERR_INVALID, "nccl_unique_id: null output");
    ncclUniqueId id;
    SDFGB_NCCL(nccl().getUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return SDFGB_OK;
}

extern "C" int sdfgb_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank) {
    SDFGB_NEED_NCCL();
    if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(SDFGB_ERR_INVALID, "nccl_comm_init: bad arguments");
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    SDFGB_NCCL(nccl().commInitRank(&c, nranks, uid, rank));
    *comm_out = c;
    return SDFGB_OK;
}

extern "C" int sdfgb_nccl_comm_destroy(void* comm) {
    SDFGB_NEED_NCCL();
    if (comm) SDFGB_NCCL(nccl().commDestroy(static_cast<ncclComm_t>(comm)));
    return SDFGB_OK;
}

// ------------------------------------------------------------------ histogram
extern "C" size_t sdfgb_hist_mgpu_workspace_bytes(int64_t bins) { return (size_t)(bins + 1) * 8; }

extern "C" int sdfgb_hist_f32_mgpu(const float* img, int64_t n, double scale, double div, int64_t* hist,
                                   int64_t bins, uint64_t* oob, void* ws, size_t ws_bytes, void* comm,
                                   void* stream) {
    SDFGB_NEED_NCCL();
    if (bins <= 0 || !hist || !oob || !comm || (n > 0 && !img))
        return set_error(SDFGB_ERR_INVALID, "hist_mgpu: bad arguments");
    if (!ws || ws_bytes < sdfgb_hist_mgpu_workspace_bytes(bins))
        return set_error(SDFGB_ERR_WORKSPACE, "hist_mgpu: workspace too small");
    cudaStream_t s = as_stream(stream);
    int64_t* part = static_cast<int64_t*>(ws);  // bins, then the out-of-range count
    SDFGB_CUDA(cudaMemsetAsync(part, 0, (size_t)(bins + 1) * 8, s));
    SDFGB_TRY(sdfgb_hist_f32(img, n, scale, div, part, bins, reinterpret_cast<uint64_t*>(part + bins), stream));
    SDFGB_NCCL(nccl().allReduce(part, part, (size_t)(bins + 1), ncclInt64, ncclSum, static_cast<ncclComm_t>(comm), s));
    hist_fold_kernel<<<std::max<int64_t>(1, std::min<int64_t>((bins + 256) / 256, 64)), 256, 0, s>>>(hist, oob, part,
                                                                                                     bins);
    SDFGB_LAUNCHED("hist_fold_kernel");
    return SDFGB_OK;
}

// ---------------------------------------------------------------------- query
extern "C" int sdfgb_query_f32_mgpu(const float* col, int64_t n, int op, double thr, float* out_vals,
                                    int64_t* count, int64_t* offset, int64_t* counts, void* ws, size_t ws_bytes,
                                    void* comm, void* stream) {
    SDFGB_NEED_NCCL();
    if (!count || !offset || !counts || !comm) return set_error(SDFGB_ERR_INVALID, "query_mgpu: bad arguments");
    int rank = 0, world = 1;
    SDFGB_TRY(comm_shape(static_cast<ncclComm_t>(comm), &rank, &world));
    cudaStream_t s = as_stream(stream);
    // this rank's survivors -> out_vals[0:k); k lands in counts[rank]
    SDFGB_CUDA(cudaMemsetAsync(counts + rank, 0, 8, s));
    SDFGB_TRY(sdfgb_query_f32(col, n, op, thr, out_vals, counts + rank, ws, ws_bytes, stream));
    SDFGB_NCCL(nccl().allGather(counts + rank, counts, 1, ncclInt64, static_cast<ncclComm_t>(comm), s));
    query_fold_kernel<<<1, 32, 0, s>>>(counts, world, rank, count, offset);
    SDFGB_LAUNCHED("query_fold_kernel");
    return SDFGB_OK;
}

// ----------------------------------------------------------------------- spmv
extern "C" int sdfgb_spmv_csr_f32_mgpu(const int32_t* rowptr, const int32_t* col, const float* val,
                                       const float* x_shard, int64_t w_shard, float* x_full, float* b,
                                       int64_t H_local, void* comm, void* stream) {
    SDFGB_NEED_NCCL();
    if (!comm || w_shard < 0 || (w_shard > 0 && (!x_shard || !x_full)))
        return set_error(SDFGB_ERR_INVALID, "spmv_mgpu: bad arguments");
    cudaStream_t s = as_stream(stream);
    if (w_shard > 0)
        SDFGB_NCCL(nccl().allGather(x_shard, x_full, (size_t)w_shard, ncclFloat32, static_cast<ncclComm_t>(comm), s));
    return sdfgb_spmv_csr_f32(rowptr, col, val, x_full, b, H_local, stream);
}

// --------------------------------------------------------------------- jacobi
namespace sdfgb {
namespace {
// owned edge rows -> the neighbours' ghost rows of one plane ([M, N] fp32)
int ghost_exchange(float* plane, int64_t N, int64_t top, int64_t rows, int64_t bot, int rank, int world,
                   ncclComm_t c, cudaStream_t s) {
    SDFGB_NCCL(nccl().groupStart());
    int rc = SDFGB_OK;
    if (rank > 0 && top) {
        rc = nccl_check(nccl().send(plane + top * N, (size_t)(top * N), ncclFloat32, rank - 1, c, s), "ncclSend");
        if (rc == SDFGB_OK) rc = nccl_check(nccl().recv(plane, (size_t)(top * N), ncclFloat32, rank - 1, c, s), "ncclRecv");
    }
    if (rc == SDFGB_OK && rank < world - 1 && bot) {
        rc = nccl_check(nccl().send(plane + (top + rows - bot) * N, (size_t)(bot * N), ncclFloat32, rank + 1, c, s),
                        "ncclSend");
        if (rc == SDFGB_OK)
            rc = nccl_check(nccl().recv(plane + (top + rows) * N, (size_t)(bot * N), ncclFloat32, rank + 1, c, s),
                            "ncclRecv");
    }
    const int rc2 = nccl_check(nccl().groupEnd(), "ncclGroupEnd");
    return rc != SDFGB_OK ? rc : rc2;
}
}  // namespace
}  // namespace sdfgb

extern "C" int sdfgb_jacobi2d_f32_mgpu(float* A, int64_t top, int64_t rows, int64_t bot, int64_t N, int64_t T,
                                       double coef, void* comm, void* stream) {
    SDFGB_NEED_NCCL();
    if (!A || !comm || top < 0 || bot < 0 || rows < 1 || T < 0 || N % 4 != 0)
        return set_error(SDFGB_ERR_INVALID, "jacobi_mgpu: bad arguments (N must be a multiple of 4)");
    constexpr int64_t GHOST = 7;  // the deepest temporal block
    if ((top && top != GHOST) || (bot && bot != GHOST) || ((top || bot) && rows < GHOST))
        return set_error(SDFGB_ERR_INVALID, "jacobi_mgpu: ghost zones are 7 rows, slabs at least 7 rows");
    int rank = 0, world = 1;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    SDFGB_TRY(comm_shape(c, &rank, &world));
    cudaStream_t s = as_stream(stream);
    const int64_t M = top + rows + bot, plane = M * N;
    // both planes' ghost rows once: their border columns are read by
    // intermediate states of the other parity and never exchanged again
    SDFGB_TRY(ghost_exchange(A + plane, N, top, rows, bot, rank, world, c, s));
    SDFGB_TRY(ghost_exchange(A, N, top, rows, bot, rank, world, c, s));
    // overlapped schedule (multigpu.jacobi): edge bands, exchange of the new
    // edge rows on the side stream, interior band; the next block waits
    constexpr int64_t EDGE = 16;
    const bool band = N >= 128 && (top || bot) && rows >= 3 * EDGE;
    SideStream ss(s);
    SDFGB_TRY(ss.rc);
    for (int64_t t = 0; t < T;) {
        int64_t k = 1;
        if (T - t > 1) {
            k = std::min<int64_t>(GHOST, T - 1 - t);
            k -= (k % 2 == 0);
        }
        const float* src = A + (t % 2) * plane;
        float* dst = A + ((t + 1) % 2) * plane;
        SDFGB_TRY(ss.join());  // src's ghost rows have landed
        if (band) {
            const int64_t lo = top, hi = top + rows;
            const int64_t e0 = top ? lo + EDGE : lo, e1 = bot ? hi - EDGE : hi;
            if (top) SDFGB_TRY(sdfgb_jacobi2d_band_f32(src, dst, M, N, k, lo, e0, coef, stream));
            if (bot) SDFGB_TRY(sdfgb_jacobi2d_band_f32(src, dst, M, N, k, e1, hi, coef, stream));
            SDFGB_TRY(ss.fork());
            SDFGB_TRY(ghost_exchange(dst, N, top, rows, bot, rank, world, c, ss.side));
            SDFGB_TRY(sdfgb_jacobi2d_band_f32(src, dst, M, N, k, e0, e1, coef, stream));
        } else {
            SDFGB_TRY(sdfgb_jacobi2d_block_f32(src, dst, M, N, k, coef, stream));
            SDFGB_TRY(ghost_exchange(dst, N, top, rows, bot, rank, world, c, s));
        }
        t += k;
    }
    return ss.join();
}

// ----------------------------------------------------------------------- gemm
extern "C" int sdfgb_gemm_f32_mgpu(const float* A_piece, int64_t a_rows, const float* B_piece, int64_t b_rows,
                                   int64_t K, int64_t nq, float* A_panel, float* B_panel, float* C_block, void* ws,
                                   size_t ws_bytes, void* row_comm, void* col_comm, void* stream) {
    SDFGB_NEED_NCCL();
    if (!row_comm || !col_comm || !A_panel || !B_panel || !C_block || a_rows < 0 || b_rows < 0 || K < 0 || nq < 0)
        return set_error(SDFGB_ERR_INVALID, "gemm_mgpu: bad arguments");
    int qi = 0, Q = 1, pi = 0, P = 1;
    SDFGB_TRY(comm_shape(static_cast<ncclComm_t>(row_comm), &qi, &Q));
    SDFGB_TRY(comm_shape(static_cast<ncclComm_t>(col_comm), &pi, &P));
    if (b_rows * P != K) return set_error(SDFGB_ERR_INVALID, "gemm_mgpu: the B pieces must tile K");
    cudaStream_t s = as_stream(stream);
    SDFGB_NCCL(nccl().allGather(B_piece, B_panel, (size_t)(b_rows * nq), ncclFloat32,
                                static_cast<ncclComm_t>(col_comm), s));
    if (Q == 1) {
        if (A_panel != A_piece)
            SDFGB_CUDA(cudaMemcpyAsync(A_panel, A_piece, (size_t)(a_rows * K) * 4, cudaMemcpyDeviceToDevice, s));
        return sdfgb_gemm_f32(A_panel, B_panel, C_block, a_rows, nq, K, ws, ws_bytes, stream);
    }
    // the A panel's Q pieces: this rank's first (no wait), the others
    // broadcast on the side stream and consumed as they land; K stays whole
    // so each C row keeps the one-GPU summation
    SideStream ss(s);
    SDFGB_TRY(ss.rc);
    SDFGB_CUDA(cudaMemcpyAsync(A_panel + qi * a_rows * K, A_piece, (size_t)(a_rows * K) * 4,
                               cudaMemcpyDeviceToDevice, s));
    SDFGB_TRY(ss.fork());
    std::vector<cudaEvent_t> landed(Q, nullptr);
    struct Events {
        std::vector<cudaEvent_t>& v;
        ~Events() {
            for (auto e : v)
                if (e) cudaEventDestroy(e);
        }
    } guard{landed};
    for (int q = 0; q < Q; ++q) {
        SDFGB_CUDA(cudaEventCreateWithFlags(&landed[q], cudaEventDisableTiming));
        SDFGB_NCCL(nccl().broadcast(A_panel + q * a_rows * K, A_panel + q * a_rows * K, (size_t)(a_rows * K),
                                    ncclFloat32, q, static_cast<ncclComm_t>(row_comm), ss.side));
        SDFGB_CUDA(cudaEventRecord(landed[q], ss.side));
    }
    for (int i = 0; i < Q; ++i) {
        const int q = (qi + i) % Q;
        if (q != qi) SDFGB_CUDA(cudaStreamWaitEvent(s, landed[q], 0));
        // B is split once (first piece); the later pieces reuse it from ws
        SDFGB_TRY(sdfgb_gemm_f32_ex(A_panel + q * a_rows * K, B_panel, C_block + q * a_rows * nq, a_rows, nq, K, ws,
                                    ws_bytes, i ? SDFGB_GEMM_B_SPLIT : 0, stream));
    }
    return ss.join();
}
