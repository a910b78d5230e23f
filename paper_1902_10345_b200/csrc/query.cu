// query.cu -- K2: predicated stream push + drain as one order-preserving
// stream compaction.
//
// Reference semantics (query motif, gallery.py:300-347):
//   map i in [0:N-1]:  if col[i] OP limit: push col[i] to stream S; count += 1
//   then S is drained FIFO into out_vals[0:n)           (codegen.py:363-376)
// The CPU stream is a realloc-doubling queue with one memcpy per push
// (codegen.py:123-143, :462-471); the FIFO order is the map's iteration order.
//
// B200 design: single pass, HBM-bound (read 4N, write 4n).  Each CTA owns a
// tile of 16 elements x 512 threads (32 KB); predicate bits -> per-thread
// counts -> one 64-bit packed block scan (4 chunk counters in 16-bit lanes)
// -> survivors staged in smem at their tile-local rank -> the tile's global
// offset from a per-round all-gather of tile counts between co-resident CTAs
// (see query_kernel) -> one contiguous, coalesced store of the survivors.  The
// output is therefore IDENTICAL to the CPU FIFO order, not just the same set.
//
// Status words carry a 20-bit launch epoch, so the workspace never needs
// clearing between launches.
#include <algorithm>
#include <atomic>

#include "common.cuh"

namespace sdfgb {
namespace {

constexpr int kQBlock = 512;
constexpr int kQVecPerThread = 4;

constexpr uint64_t kFlagAgg = 1ull;
constexpr uint64_t kFlagPrefix = 2ull;
constexpr int kValueBits = 42;
constexpr uint64_t kValueMask = (1ull << kValueBits) - 1;

struct QueryWs {
    unsigned long long ticket;
    unsigned long long done;
    unsigned long long pad[14];
    unsigned long long status[1];  // num_tiles words
};

__device__ __forceinline__ uint64_t ld_relaxed(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint64_t flag, uint64_t value) {
    return ((uint64_t)epoch << 44) | (flag << kValueBits) | (value & kValueMask);
}

template <typename T, bool VEC, int K, int VN>
__device__ __forceinline__ void q_load(const T* __restrict__ col, int64_t n, int64_t base, int tid,
                                       T (&v)[K][VN]) {
    using V = typename Vec16<T>::type;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int64_t e0 = base + (int64_t)k * kQBlock * VN + (int64_t)tid * VN;
        if (VEC && e0 + VN <= n) {
            V x = ldg_stream(reinterpret_cast<const V*>(col + e0));
#pragma unroll
            for (int c = 0; c < VN; ++c) v[k][c] = vget<V, T>(x, c);
        } else {
#pragma unroll
            for (int c = 0; c < VN; ++c) v[k][c] = (e0 + c < n) ? col[e0 + c] : T(0);
        }
    }
}

// Persistent, co-resident CTAs (cooperative launch) in lock-step rounds: in
// round r CTA c owns tile r*G + c.  Every CTA publishes its tile's survivor
// count, prefetches its next tile, then reads the round's G counts at once
// (one block-wide load) -> its exclusive offset inside the round and the
// round total, which every CTA adds to a private running base.  There is no
// ticket counter and no prefix chain: a round costs one all-gather of counts
// through L2 while the next tile's loads are already in flight.
template <typename T, bool VEC>
__global__ void __launch_bounds__(kQBlock)
query_kernel(const T* __restrict__ col, int64_t n, int op, double thr, T* __restrict__ out,
             unsigned long long* __restrict__ count, QueryWs* __restrict__ ws,
             int64_t num_tiles, uint32_t epoch) {
    constexpr int VN = Vec16<T>::n;
    constexpr int K = kQVecPerThread;
    constexpr int TILE = kQBlock * K * VN;
    constexpr int NW = kQBlock / 32;

    __shared__ T s_stage[TILE];
    __shared__ uint64_t s_warp[NW];
    __shared__ int64_t s_red[NW], s_tot[NW];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t rounds = (num_tiles + G - 1) / G;
    int64_t base_off = 0;
    T v[K][VN];
    if (c < num_tiles) q_load<T, VEC, K, VN>(col, n, c * TILE, tid, v);

    for (int64_t r = 0; r < rounds; ++r) {
        const int64_t tile = r * G + c;
        const int64_t base = tile * TILE;
        uint32_t agg = 0;
        if (tile < num_tiles) {  // CTA-uniform
            uint32_t bits = 0;  // bit k*VN+c
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int64_t e0 = base + (int64_t)k * kQBlock * VN + (int64_t)tid * VN;
#pragma unroll
                for (int cc = 0; cc < VN; ++cc)
                    bits |= (uint32_t)((e0 + cc < n) && cmp_apply((double)v[k][cc], op, thr)) << (k * VN + cc);
            }
            // packed block scan: 16-bit field k = this thread's count in chunk k
            uint64_t mine = 0;
#pragma unroll
            for (int k = 0; k < K; ++k)
                mine |= (uint64_t)__popc((bits >> (k * VN)) & ((1u << VN) - 1)) << (16 * k);
            uint64_t incl = mine;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint64_t o = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += o;
            }
            if (lane == 31) s_warp[warp] = incl;
            __syncthreads();
            uint64_t wpre = 0, total = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                uint64_t t = s_warp[w];
                if (w < warp) wpre += t;
                total += t;
            }
            const uint64_t excl = wpre + incl - mine;
            // stage survivors in smem at their tile-local input-order rank
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t rr = agg + (uint32_t)((excl >> (16 * k)) & 0xffff);
#pragma unroll
                for (int cc = 0; cc < VN; ++cc)
                    if (bits & (1u << (k * VN + cc))) s_stage[rr++] = v[k][cc];
                agg += (uint32_t)((total >> (16 * k)) & 0xffff);
            }
            if (tid == 0) st_relaxed(&ws->status[tile], pack_status(epoch, kFlagAgg, agg));
        }
        // prefetch the next round's tile while this round's counts gather
        if (tile + G < num_tiles) q_load<T, VEC, K, VN>(col, n, (tile + G) * TILE, tid, v);

        // all-gather of the round's counts (thread q reads CTA q's word)
        int64_t val = 0;
        const int64_t q = r * G + tid;
        if (tid < G && q < num_tiles) {
            uint64_t w;
            while (true) {
                w = ld_relaxed(&ws->status[q]);
                if ((uint32_t)(w >> 44) == epoch && ((w >> kValueBits) & 3ull)) break;
                __nanosleep(16);
            }
            val = (int64_t)(w & kValueMask);
        }
        int64_t lower = tid < c ? val : 0;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            lower += __shfl_xor_sync(0xffffffffu, lower, d);
            val += __shfl_xor_sync(0xffffffffu, val, d);
        }
        if (lane == 0) {
            s_red[warp] = lower;
            s_tot[warp] = val;
        }
        __syncthreads();
        int64_t my_off = base_off, round_total = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            my_off += s_red[w];
            round_total += s_tot[w];
        }
        // drain: contiguous, coalesced stores of the staged survivors
        for (uint32_t rr = tid; rr < agg; rr += kQBlock) out[my_off + rr] = s_stage[rr];
        base_off += round_total;
        __syncthreads();  // s_stage / s_red reuse
    }
    if (c == 0 && tid == 0) atomicAdd(count, (unsigned long long)base_off);
}

std::atomic<uint32_t> g_epoch{0};

uint32_t next_epoch() {
    uint32_t e;
    do {
        e = (g_epoch.fetch_add(1) + 1) & 0xFFFFF;
    } while (e == 0);
    return e;
}

template <typename T>
int64_t tiles_for(int64_t n) {
    const int64_t tile = (int64_t)kQBlock * kQVecPerThread * Vec16<T>::n;
    return (n + tile - 1) / tile;
}

template <typename T>
int launch_query(const T* col, int64_t n, int op, double thr, T* out, int64_t* count, void* ws,
                 size_t ws_bytes, void* stream) {
    if (n < 0 || op < 0 || op > 5 || !count || (n > 0 && (!col || !out || !ws)))
        return set_error(SDFGB_ERR_INVALID, "query: bad arguments");
    if (n == 0) return SDFGB_OK;
    if ((uint64_t)n > kValueMask) return set_error(SDFGB_ERR_INVALID, "query: n too large");
    const int64_t tiles = tiles_for<T>(n);
    if (ws_bytes < sdfgb_query_workspace_bytes(n, sizeof(T)))
        return set_error(SDFGB_ERR_WORKSPACE, "query: workspace %zu < %zu bytes", ws_bytes,
                         sdfgb_query_workspace_bytes(n, sizeof(T)));
    if ((reinterpret_cast<uintptr_t>(ws) & 7) != 0)
        return set_error(SDFGB_ERR_INVALID, "query: workspace must be 8-byte aligned");
    const bool vec = (reinterpret_cast<uintptr_t>(col) & 15) == 0;
    auto* W = reinterpret_cast<QueryWs*>(ws);
    auto* C = reinterpret_cast<unsigned long long*>(count);
    const uint32_t epoch = next_epoch();
    cudaStream_t s = as_stream(stream);
    auto kern = vec ? query_kernel<T, true> : query_kernel<T, false>;
    static int occ[2][2] = {};  // [f64][vec] resident CTAs per SM
    int& o = occ[sizeof(T) == 8][vec];
    if (o == 0) SDFGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kQBlock, 0));
    // every CTA must be resident (rounds wait on all of them): cooperative launch
    int64_t grid = std::min<int64_t>({tiles, (int64_t)std::max(o, 1) * num_sms(), (int64_t)kQBlock});
    grid = std::max<int64_t>(grid, 1);
    void* args[] = {(void*)&col, (void*)&n, (void*)&op, (void*)&thr, (void*)&out, (void*)&C, (void*)&W,
                    (void*)&tiles, (void*)&epoch};
    SDFGB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(kQBlock), args, 0, s));
    SDFGB_LAUNCHED("query_kernel");
    return SDFGB_OK;
}

}  // namespace
}  // namespace sdfgb

extern "C" size_t sdfgb_query_workspace_bytes(int64_t n, int elem_bytes) {
    int64_t tiles = elem_bytes == 8 ? sdfgb::tiles_for<double>(n) : sdfgb::tiles_for<float>(n);
    return offsetof(sdfgb::QueryWs, status) + (size_t)std::max<int64_t>(tiles, 1) * 8;
}
extern "C" int sdfgb_query_f32(const float* col, int64_t n, int op, double thr, float* out_vals,
                               int64_t* count, void* ws, size_t ws_bytes, void* stream) {
    return sdfgb::launch_query<float>(col, n, op, thr, out_vals, count, ws, ws_bytes, stream);
}
extern "C" int sdfgb_query_f64(const double* col, int64_t n, int op, double thr, double* out_vals,
                               int64_t* count, void* ws, size_t ws_bytes, void* stream) {
    return sdfgb::launch_query<double>(col, n, op, thr, out_vals, count, ws, ws_bytes, stream);
}
