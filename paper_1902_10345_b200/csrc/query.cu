// query.cu -- K2: predicated stream push + drain as one stream compaction.
// Default: query_push_kernel (unordered, single pass; see its comment).
// SDFGB_QUERY_ORDERED: query_piece_kernel (input order, L2-resident second
// pass); misaligned inputs: query_kernel.  The header below describes the
// ordered kernels.
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
#include <cmath>

#include <cstdlib>

#include "tma.cuh"


namespace sdfgb {
namespace {

constexpr int kQBlock = 512;
constexpr int kQVecPerThread = 4;
constexpr int kQSubs = 2;  // sub-tiles per CTA segment per round

constexpr uint64_t kFlagAgg = 1ull;
[[maybe_unused]] constexpr uint64_t kFlagPrefix = 2ull;
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

__device__ __forceinline__ uint64_t make_policy(bool keep) {
    uint64_t p;
    if (keep)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float4 ldg_pol(const float4* p, uint64_t pol) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double2 ldg_pol(const double2* p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}

// predicate in the element type; OP 6/7 = constant false/true (see fold_threshold)
template <int OP, typename T>
__device__ __forceinline__ bool pred(T v, T t) {
    if constexpr (OP == SDFGB_CMP_LT) return v < t;
    else if constexpr (OP == SDFGB_CMP_LE) return v <= t;
    else if constexpr (OP == SDFGB_CMP_GT) return v > t;
    else if constexpr (OP == SDFGB_CMP_GE) return v >= t;
    else if constexpr (OP == SDFGB_CMP_EQ) return v == t;
    else if constexpr (OP == SDFGB_CMP_NE) return v != t;
    else if constexpr (OP == 6) return false;
    else return true;
}

// Load one sub-tile: element e = base + k*kQBlock*VN + tid*VN + c.  FULL
// (CTA-uniform: the whole sub-tile lies inside [0, n)) drops every bounds test.
template <typename T, bool VEC, bool FULL, int K, int VN>
__device__ __forceinline__ void q_load(const T* __restrict__ col, int64_t n, int64_t base, int tid,
                                       uint64_t pol, T (&v)[K][VN]) {
    using V = typename Vec16<T>::type;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int64_t e0 = base + (int64_t)k * kQBlock * VN + (int64_t)tid * VN;
        if (VEC && (FULL || e0 + VN <= n)) {
            V x = ldg_pol(reinterpret_cast<const V*>(col + e0), pol);
#pragma unroll
            for (int c = 0; c < VN; ++c) v[k][c] = vget<V, T>(x, c);
        } else {
#pragma unroll
            for (int c = 0; c < VN; ++c) v[k][c] = (FULL || e0 + c < n) ? col[e0 + c] : T(0);
        }
    }
}

// predicate bits, bit k*VN + c
template <typename T, bool FULL, int OP, int K, int VN>
__device__ __forceinline__ uint32_t q_bits(const T (&v)[K][VN], int64_t n, int64_t base, int tid, T thr) {
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int64_t e0 = base + (int64_t)k * kQBlock * VN + (int64_t)tid * VN;
#pragma unroll
        for (int c = 0; c < VN; ++c)
            if ((FULL || e0 + c < n) && pred<OP>(v[k][c], thr)) bits |= 1u << (k * VN + c);
    }
    return bits;
}

// Persistent, co-resident CTAs (cooperative launch) working in rounds over
// L2-sized chunks.  Round r gives CTA c the contiguous segment
// [r*G*S + c*S, +S) (S = kQSubs sub-tiles):
//   count(r)  stream the segment from HBM (L2 evict_last), publish its
//             survivor count in status[r*G + c];
//   gather(r) one block-wide read of the round's G counts -> this CTA's
//             offset inside the round and the round total;
//   write(r)  re-read the segment (L2 hits, evict_first), block-scan each
//             sub-tile, stage survivors in smem, store them contiguously.
// count(r+1) runs before gather(r), so the counts of round r have a whole
// segment's worth of HBM time to become visible: the only inter-CTA
// synchronisation is one count all-gather per round, off the critical path.
template <typename T, bool VEC, int OP>
__global__ void __launch_bounds__(kQBlock, 2)
query_kernel(const T* __restrict__ col, int64_t n, T thr, T* __restrict__ out,
             unsigned long long* __restrict__ count, QueryWs* __restrict__ ws,
             int64_t rounds, uint32_t epoch) {
    constexpr int VN = Vec16<T>::n;
    constexpr int K = kQVecPerThread;
    constexpr int SUB = kQBlock * K * VN;
    constexpr int64_t S = (int64_t)SUB * kQSubs;
    constexpr int NW = kQBlock / 32;

    __shared__ __align__(16) T s_stage[SUB + 4];
    __shared__ uint64_t s_warp[NW];
    __shared__ int64_t s_red[NW], s_tot[NW];
    __shared__ uint32_t s_cnt[NW];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t keep = make_policy(true), drop = make_policy(false);
    T v[K][VN];

    auto count_round = [&](int64_t r) {
        const int64_t seg = (r * G + c) * S;
        uint32_t cnt = 0;
#pragma unroll 1
        for (int j = 0; j < kQSubs; ++j) {
            const int64_t base = seg + (int64_t)j * SUB;
            if (base + SUB <= n) {
                q_load<T, VEC, true, K, VN>(col, n, base, tid, keep, v);
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int cc = 0; cc < VN; ++cc) cnt += pred<OP>(v[k][cc], thr) ? 1u : 0u;
            } else if (base < n) {
                q_load<T, VEC, false, K, VN>(col, n, base, tid, keep, v);
                cnt += __popc(q_bits<T, false, OP, K, VN>(v, n, base, tid, thr));
            }
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
        if (lane == 0) s_cnt[warp] = cnt;
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) t += s_cnt[w];
            st_relaxed(&ws->status[r * G + c], pack_status(epoch, kFlagAgg, t));
        }
    };

    count_round(0);
    int64_t base_off = 0;
    for (int64_t r = 0; r < rounds; ++r) {
        if (r + 1 < rounds) count_round(r + 1);
        // ---- all-gather of round r's counts (thread q reads CTA q's word)
        int64_t val = 0;
        if (tid < G) {
            uint64_t w;
            while (true) {
                w = ld_relaxed(&ws->status[r * G + tid]);
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
        int64_t off = base_off, round_total = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            off += s_red[w];
            round_total += s_tot[w];
        }
        // ---- write(r): re-read from L2, scan, stage, store contiguously
        const int64_t seg = (r * G + c) * S;
#pragma unroll 1
        for (int j = 0; j < kQSubs; ++j) {
            const int64_t base = seg + (int64_t)j * SUB;
            if (base >= n) break;  // CTA-uniform
            uint32_t bits;
            if (base + SUB <= n) {
                q_load<T, VEC, true, K, VN>(col, n, base, tid, drop, v);
                bits = q_bits<T, true, OP, K, VN>(v, n, base, tid, thr);
            } else {
                q_load<T, VEC, false, K, VN>(col, n, base, tid, drop, v);
                bits = q_bits<T, false, OP, K, VN>(v, n, base, tid, thr);
            }
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
            __syncthreads();  // previous sub-tile's drain / s_red reads are done
            if (lane == 31) s_warp[warp] = incl;
            __syncthreads();
            // warp-level scan of the NW warp totals (every warp redundantly)
            uint64_t ws_ = lane < NW ? s_warp[lane] : 0;
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                uint64_t o = __shfl_up_sync(0xffffffffu, ws_, d);
                if (lane >= d) ws_ += o;
            }
            const uint64_t wprev = __shfl_sync(0xffffffffu, ws_, (warp + 31) & 31);
            const uint64_t wpre = warp ? wprev : 0;
            const uint64_t total = __shfl_sync(0xffffffffu, ws_, NW - 1);
            const uint64_t excl = wpre + incl - mine;
            // stage at (off mod VEC16) + rank so smem and global indices are
            // congruent mod 16 B and the drain can move 128-bit vectors
            const uint32_t sh0 = (uint32_t)(off & (VN - 1));
            uint32_t agg = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t rr = sh0 + agg + (uint32_t)((excl >> (16 * k)) & 0xffff);
#pragma unroll
                for (int cc = 0; cc < VN; ++cc) {
                    const bool p = bits & (1u << (k * VN + cc));
                    if (p) s_stage[rr] = v[k][cc];
                    rr += p;
                }
                agg += (uint32_t)((total >> (16 * k)) & 0xffff);
            }
            __syncthreads();
            // drain: scalar head up to a 16 B boundary, 128-bit body, scalar tail
            using V = typename Vec16<T>::type;
            const uint32_t head = std::min<uint32_t>(agg, (VN - sh0) & (VN - 1));
            if (tid < head) out[off + tid] = s_stage[sh0 + tid];
            const uint32_t nv = (agg - head) / VN;
            const V* sv = reinterpret_cast<const V*>(s_stage + sh0 + head);
            V* gv = reinterpret_cast<V*>(out + off + head);
            if (VEC && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
                for (uint32_t q = tid; q < nv; q += kQBlock) gv[q] = sv[q];
                for (uint32_t rr = head + nv * VN + tid; rr < agg; rr += kQBlock) out[off + rr] = s_stage[sh0 + rr];
            } else {
                for (uint32_t rr = head + tid; rr < agg; rr += kQBlock) out[off + rr] = s_stage[sh0 + rr];
            }
            off += agg;
        }
        base_off += round_total;
        __syncthreads();
    }
    if (c == 0 && tid == 0) atomicAdd(count, (unsigned long long)base_off);
}

constexpr int kTBlock = 1024;  // upper bound on co-resident CTAs of the piece kernel (count slots per piece)

// predicated store of v to base[idx] with a single 32x32+64 address op
__device__ __forceinline__ void st_pred(float* base, uint32_t idx, float v, uint32_t p) {
    asm volatile(
        "{\n .reg .pred q;\n .reg .u64 a;\n setp.ne.u32 q, %3, 0;\n mad.wide.u32 a, %0, 4, %1;\n"
        " @q st.global.f32 [a], %2;\n}" ::"r"(idx), "l"(base), "f"(v), "r"(p)
        : "memory");
}
__device__ __forceinline__ void st_pred(double* base, uint32_t idx, double v, uint32_t p) {
    asm volatile(
        "{\n .reg .pred q;\n .reg .u64 a;\n setp.ne.u32 q, %3, 0;\n mad.wide.u32 a, %0, 8, %1;\n"
        " @q st.global.f64 [a], %2;\n}" ::"r"(idx), "l"(base), "d"(v), "r"(p)
        : "memory");
}


// ---------------------------------------------------------------------------
// Piece kernel (the default for 16 B-aligned columns).  The column is cut
// into equal pieces of at most 16 MB, and each co-resident CTA owns the same
// contiguous chunk range of every piece, cut into NW warp ranges.  Two warp
// roles run as a pipeline:
//   A  (counter warps)    count piece p's warp ranges from HBM (L2
//      evict_last, a rolling ring of 8 vector loads per lane), then publish
//      the CTA's total as an epoch-tagged word cnts[p*G + c] and the
//      per-warp counts in a shared-memory slot (full mbarrier);
//   B  (compactor warps)  read piece p's G CTA totals (spinning only on
//      words not yet published) for the CTA's offset, take the per-warp
//      counts from the slot (empty mbarrier), then re-read each warp range
//      from L2 (evict_first, two 4-chunk register sets so the next loads are
//      in flight) and compact it in order: byte-packed chunk counts, one
//      32-bit shuffle scan per 4 chunks, predicated stores.
// So HBM reads of one piece overlap the survivor writes of earlier ones, the
// counters run up to SDFGB_Q_SLOTS pieces ahead (so at most ~4 pieces are
// L2-resident), HBM sees each input byte once, and there is no grid-wide or
// per-step CTA barrier (the cooperative launch only guarantees that every
// CTA is resident).
#ifndef SDFGB_Q_PIECE_MB
#define SDFGB_Q_PIECE_MB 16
#endif
#ifndef SDFGB_Q_MINB
#define SDFGB_Q_MINB 1
#endif
#ifndef SDFGB_Q_SLOTS
#define SDFGB_Q_SLOTS 3  // per-warp count slots between the roles: counters run up to 3 pieces ahead
#endif
#ifndef SDFGB_Q_RING
#define SDFGB_Q_RING 8  // chunk loads in flight per counter lane
#endif
constexpr int64_t kPieceBytes = (int64_t)SDFGB_Q_PIECE_MB << 20;  // upper bound; pieces are equalised

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename T>
__device__ __forceinline__ typename Vec16<T>::type ldg_hint(const T* p, uint64_t pol) {
    return ldg_pol(reinterpret_cast<const typename Vec16<T>::type*>(p), pol);
}

#ifndef SDFGB_Q_PBLOCK
#define SDFGB_Q_PBLOCK 512
#endif
constexpr int kQPBlock = SDFGB_Q_PBLOCK;

#ifndef SDFGB_Q_TIMING
#define SDFGB_Q_TIMING 0  // debug: per-CTA role timestamps (sdfgb_debug_query_timing)
#endif
#if SDFGB_Q_TIMING
__device__ unsigned long long g_qtime[64][4][1024];  // [piece][A0,A1,B0,B1][CTA]
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif
template <typename T, int OP>
__global__ void __launch_bounds__(kQPBlock, SDFGB_Q_MINB)
query_piece_kernel(const T* __restrict__ col, int64_t n, T thr, T* __restrict__ out,
                   unsigned long long* __restrict__ count, unsigned long long* __restrict__ cnts, uint32_t epoch) {
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::n;
    // two roles of NW warps each, counters (A) and compactors (B), over the
    // same NW warp ranges of the CTA's chunks
    constexpr int NW = kQPBlock / 64;
    constexpr int CH = 32 * VN;  // elements per warp chunk
    // equal pieces of at most kPieceBytes, multiples of a chunk
    const int64_t npieces = (n * (int64_t)sizeof(T) + kPieceBytes - 1) / kPieceBytes;
    const int64_t PIECE = ((n + npieces - 1) / npieces + CH - 1) / CH * CH;
    constexpr int SL = SDFGB_Q_SLOTS;
    __shared__ uint32_t s_wcnt[SL][NW];  // per-warp counts of the pieces in flight
    __shared__ __align__(8) uint64_t s_full[SL], s_empty[SL];
    __shared__ int64_t s_lo[2][NW], s_to[2][NW];

    const int tid = threadIdx.x, lane = tid & 31;
    const bool counter = tid < NW * 32;
    const int warp = (tid >> 5) - (counter ? 0 : NW);  // index within the role
    const int rtid = tid - (counter ? 0 : NW * 32);
    if (tid == 0) {
        for (int k = 0; k < SL; ++k) {
            mbar_init(&s_full[k], 1);
            mbar_init(&s_empty[k], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto wait_bar = [&](uint64_t* b, uint32_t par) {
        while (!__all_sync(0xffffffffu, mbar_try_wait(smem_u32(b), par))) {
        }
    };
#define SLOT(p) ((int)((p) % SL))
    const int64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t keep = make_policy(true), drop = make_policy(false);
    // warp range r's chunks [w0, w1) of piece p (starting at element ps)
    auto geom = [&](int64_t p, int r, int64_t& ps, int64_t& w0, int64_t& w1) {
        ps = p * PIECE;
        const int64_t pl = n - ps < PIECE ? n - ps : PIECE;
        const int64_t nch = (pl + CH - 1) / CH;
        const int64_t per_cta = (nch + G - 1) / G;
        const int64_t cs = c * per_cta < nch ? c * per_cta : nch;
        const int64_t ce = cs + per_cta < nch ? cs + per_cta : nch;
        const int64_t per_w = (ce - cs + NW - 1) / NW;
        w0 = cs + r * per_w < ce ? cs + r * per_w : ce;
        w1 = w0 + per_w < ce ? w0 + per_w : ce;
    };
    // ---- A(p): count, publish this CTA's count of piece p (epoch-tagged)
    auto phaseA = [&](int64_t p) {
        int64_t ps, w0, w1;
        geom(p, warp, ps, w0, w1);
        // a rolling ring of R chunk loads per lane: each consumed vector is
        // replaced at once by the load R chunks ahead, so R stay in flight
        // (a batch loaded then counted leaves HBM idle between batches)
        constexpr int R = SDFGB_Q_RING;
        uint32_t cnt = 0;
        int64_t q = w0;
        int64_t qfull = w1;
        while (qfull > w0 && ps + qfull * CH > n) --qfull;  // chunks wholly inside the column
        if (q + R <= qfull) {
            V x[R];
#pragma unroll
            for (int j = 0; j < R; ++j) x[j] = ldg_hint(col + ps + (q + j) * CH + lane * VN, keep);
            for (; q + R <= qfull; q += R) {
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const V v = x[j];
                    if (q + R + j < qfull) x[j] = ldg_hint(col + ps + (q + R + j) * CH + lane * VN, keep);
#pragma unroll
                    for (int cc = 0; cc < VN; ++cc) cnt += pred<OP>(vget<V, T>(v, cc), thr) ? 1u : 0u;
                }
            }
            // the loads issued past the last full group were exactly the rest
            // of [q, qfull): count them from the ring
#pragma unroll
            for (int j = 0; j < R; ++j)
                if (q + j < qfull) {
#pragma unroll
                    for (int cc = 0; cc < VN; ++cc) cnt += pred<OP>(vget<V, T>(x[j], cc), thr) ? 1u : 0u;
                }
            q = qfull;
        }
        for (; q < w1; ++q) {
            const int64_t e0 = ps + q * CH + lane * VN;
            if (e0 + VN <= n) {
                const V x = ldg_hint(col + e0, keep);
#pragma unroll
                for (int cc = 0; cc < VN; ++cc) cnt += pred<OP>(vget<V, T>(x, cc), thr) ? 1u : 0u;
            } else {
#pragma unroll
                for (int cc = 0; cc < VN; ++cc) cnt += (e0 + cc < n && pred<OP>(col[e0 + cc], thr)) ? 1u : 0u;
            }
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        // the slot's previous piece (p - SL) has been read by every compactor warp
        if (p >= SL) wait_bar(&s_empty[SLOT(p)], (uint32_t)((p / SL - 1) & 1));
        if (lane == 0) s_wcnt[SLOT(p)][warp] = cnt;
        named_bar(1, NW * 32);  // the counters only
        if (tid == 0) {
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) t += s_wcnt[SLOT(p)][w];
            st_relaxed(cnts + p * G + c, pack_status(epoch, kFlagAgg, t));
            mbar_arrive(&s_full[SLOT(p)]);
        }
    };
    int64_t base = 0;
    // ---- B(p): this CTA's offset inside piece p (waits only for counts not
    // yet published -- by now every CTA has moved on to piece p+1), then
    // per-warp compaction from L2
    auto phaseB = [&](int64_t p) {
        int64_t ps, w0, w1;
        geom(p, warp, ps, w0, w1);
        int64_t lo = 0, to = 0;
        for (int64_t q = rtid; q < G; q += NW * 32) {
            uint64_t w;
            do {
                w = ld_relaxed(cnts + p * G + q);
            } while ((uint32_t)(w >> 44) != epoch);
            const int64_t v = (int64_t)(w & kValueMask);
            to += v;
            lo += q < c ? v : 0;
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            lo += __shfl_xor_sync(0xffffffffu, lo, d);
            to += __shfl_xor_sync(0xffffffffu, to, d);
        }
        int64_t* slo = s_lo[p & 1];  // double-buffered: a fast warp may reach the next piece
        int64_t* sto = s_to[p & 1];
        if (lane == 0) {
            slo[warp] = lo;
            sto[warp] = to;
        }
        named_bar(2, NW * 32);  // the compactors only
        int64_t cta_off = 0, piece_total = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            cta_off += slo[w];
            piece_total += sto[w];
        }
        wait_bar(&s_full[SLOT(p)], (uint32_t)((p / SL) & 1));
        uint32_t wc = lane < warp ? s_wcnt[SLOT(p)][lane] : 0u;
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[SLOT(p)]);
#pragma unroll
        for (int d = 16; d; d >>= 1) wc += __shfl_xor_sync(0xffffffffu, wc, d);
        T* wout = out + (base + cta_off + wc);
        uint32_t run = 0;
        // compact 4 chunks from x (loaded, or loaded here when !full)
        auto emit4 = [&](V (&x)[4], bool full, int64_t q0) {
            uint32_t bits = 0, pk = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t e0 = ps + (q0 + j) * CH + lane * VN;
                uint32_t m = 0;
                if (full) {
#pragma unroll
                    for (int cc = 0; cc < VN; ++cc) m |= (uint32_t)pred<OP>(vget<V, T>(x[j], cc), thr) << cc;
                } else if (q0 + j < w1 && e0 + VN <= n) {
                    x[j] = ldg_hint(col + e0, drop);
#pragma unroll
                    for (int cc = 0; cc < VN; ++cc) m |= (uint32_t)pred<OP>(vget<V, T>(x[j], cc), thr) << cc;
                } else {
                    T* xs = reinterpret_cast<T*>(&x[j]);
#pragma unroll
                    for (int cc = 0; cc < VN; ++cc) {
                        const bool live = q0 + j < w1 && e0 + cc < n;
                        xs[cc] = live ? col[e0 + cc] : T(0);
                        m |= (uint32_t)(live && pred<OP>(xs[cc], thr)) << cc;
                    }
                }
                bits |= m << (j * VN);
                pk |= (uint32_t)__popc(m) << (8 * j);
            }
            uint32_t incl = pk;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += o;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
            const uint32_t excl = incl - pk;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t at = run + ((excl >> (8 * j)) & 0xffu);
#pragma unroll
                for (int cc = 0; cc < VN; ++cc) {
                    const uint32_t pp = (bits >> (j * VN + cc)) & 1u;
                    st_pred(wout, at, vget<V, T>(x[j], cc), pp);
                    at += pp;
                }
                run += (tot >> (8 * j)) & 0xffu;
            }
        };
        auto load4 = [&](V (&x)[4], int64_t q0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = ldg_hint(col + ps + (q0 + j) * CH + lane * VN, drop);
        };
        // whole chunks inside the column: two 4-chunk register sets, the
        // next one's L2 loads in flight while the current one is compacted
        int64_t qf = w1;
        while (qf > w0 && ps + qf * CH > n) --qf;
        int64_t q0 = w0;
        V xa[4], xb[4];
        if (q0 + 4 <= qf) load4(xa, q0);
        for (;;) {
            if (q0 + 4 > qf) break;
            if (q0 + 8 <= qf) load4(xb, q0 + 4);
            emit4(xa, true, q0);
            q0 += 4;
            if (q0 + 4 > qf) break;
            if (q0 + 8 <= qf) load4(xa, q0 + 4);
            emit4(xb, true, q0);
            q0 += 4;
        }
        for (; q0 < w1; q0 += 4) emit4(xa, false, q0);
        base += piece_total;
    };
    // Warp-specialised pipeline: while the counters stream piece i from HBM
    // into L2, the compactors write piece i-1's survivors, so HBM reads and
    // writes overlap.  The counts of piece i-1 were published by every CTA
    // during the previous step; the only CTA-wide barrier is the one per
    // step that hands s_wcnt over between the roles.
    // The roles hand the per-warp counts over through SL shared-memory slots
    // (full / empty mbarriers), so each runs at its own pace: the counters
    // stream piece p from HBM into L2 while the compactors write the
    // survivors of an earlier piece, up to SL pieces behind.
    for (int64_t p = 0; p < npieces; ++p) {
#if SDFGB_Q_TIMING
        if ((tid == 0 || tid == NW * 32) && p < 64) g_qtime[p][counter ? 0 : 2][c] = gtime();
#endif
        if (counter) phaseA(p);
        else phaseB(p);
#if SDFGB_Q_TIMING
        if ((tid == 0 || tid == NW * 32) && p < 64) g_qtime[p][counter ? 1 : 3][c] = gtime();
#endif
    }
    if (c == 0 && tid == NW * 32) atomicAdd(count, (unsigned long long)base);
}
#undef SLOT

// ---------------------------------------------------------------------------
// Unordered push kernel (the default).  A Map's iterations are concurrent and
// a Stream is a "concurrent queue" (Appendix A push rule ❷), so
// the push order of the query map is unspecified -- the north star compares
// Query output as a sorted set.  Each CTA therefore reserves its survivors'
// slot range with ONE atomicAdd on a workspace counter and never looks at
// another CTA: a single streaming pass, HBM read 4N + write 4k, no grid
// barrier, no L2 re-read.
//   tile   = kPBlock/32 warps x 8 chunks x (32 lanes x 16 B)   (16 KB)
//   warp   8 loads in flight per lane, predicate nibbles, two byte-packed
//          shuffle scans -> per-chunk exclusive offsets, warp total
//   CTA    warp totals -> smem -> warp 0 scan + atomicAdd(ctr, total)
//   store  survivors compacted into a per-warp smem stage, then written
//          as whole 128 B lines (scattered predicated stores cost 3-4x the
//          L2 write requests: 102 -> 88 us at 100 % selectivity)
// Persistent CTAs (5 x 128 threads per SM) prefetch the next tile's vectors
// before reserving the current one, so the atomic's round trip overlaps
// HBM reads.  Measured on 2^26 fp32, x < 0.5: 70.5 us (the block-size /
// occupancy / staging sweep is tools/query_sweep.sh).
// Within a warp's 1024 elements the survivors keep input order; the CTA
// order is the reservation order.  The last CTA to finish (done ticket)
// folds the total into *count and re-zeroes the counter and the ticket, so
// the workspace stays zero between launches.
#ifndef SDFGB_P_BLOCK
#define SDFGB_P_BLOCK 128
#endif
#ifndef SDFGB_P_MINB
#define SDFGB_P_MINB 5
#endif
#ifndef SDFGB_P_PERSIST
#define SDFGB_P_PERSIST 1
#endif
#ifndef SDFGB_P_STAGE
#define SDFGB_P_STAGE 1
#endif
constexpr int kPBlock = SDFGB_P_BLOCK;
constexpr int kPChunks = 8;

template <typename T>
constexpr int64_t push_tile_elems() {
    return (int64_t)kPBlock / 32 * kPChunks * 32 * Vec16<T>::n;
}

// One warp's kPChunks chunks starting at element w0: predicate bits (bit
// j*VN + c) and byte-packed per-lane chunk counts.  x holds the loaded
// vectors when `full`; otherwise they are loaded here with bounds tests.
template <typename T, int OP>
__device__ __forceinline__ void push_bits(const T* __restrict__ col, int64_t n, int64_t w0, int lane, T thr,
                                          uint64_t pol, bool full, typename Vec16<T>::type (&x)[kPChunks],
                                          uint32_t& bits, uint32_t (&pk)[2]) {
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::n;
    constexpr int CH = 32 * VN;
    bits = 0;
    pk[0] = pk[1] = 0;
#pragma unroll
    for (int j = 0; j < kPChunks; ++j) {
        const int64_t e0 = w0 + j * CH + lane * VN;
        uint32_t m = 0;
        if (full) {
#pragma unroll
            for (int cc = 0; cc < VN; ++cc) m |= (uint32_t)pred<OP>(vget<V, T>(x[j], cc), thr) << cc;
        } else if (e0 + VN <= n) {
            x[j] = ldg_hint(col + e0, pol);
#pragma unroll
            for (int cc = 0; cc < VN; ++cc) m |= (uint32_t)pred<OP>(vget<V, T>(x[j], cc), thr) << cc;
        } else {
            T* xs = reinterpret_cast<T*>(&x[j]);
#pragma unroll
            for (int cc = 0; cc < VN; ++cc) {
                const bool live = e0 + cc < n;
                xs[cc] = live ? col[e0 + cc] : T(0);
                m |= (uint32_t)(live && pred<OP>(xs[cc], thr)) << cc;
            }
        }
        bits |= m << (j * VN);
        pk[j >> 2] |= (uint32_t)__popc(m) << (8 * (j & 3));
    }
}

// Reserve the CTA's slots and store one tile (x, bits, pk from push_bits).
// sw / sbase: this tile's smem slots (double-buffered by the caller).
template <typename T>
__device__ __forceinline__ void push_store(T* __restrict__ out, unsigned long long* __restrict__ ctr, int lane,
                                           int warp, const typename Vec16<T>::type (&x)[kPChunks], uint32_t bits,
                                           const uint32_t (&pk)[2], uint32_t* sw, unsigned long long* sbase,
                                           T* stage, bool remote) {
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::n;
    constexpr int NW = kPBlock / 32;
    // per-chunk exclusive lane offsets (bytes of excl) and chunk totals (bytes of tot)
    uint32_t excl[2], tot[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t incl = pk[h];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        tot[h] = __shfl_sync(0xffffffffu, incl, 31);
        excl[h] = incl - pk[h];
    }
    const uint32_t t4 = (tot[0] & 0x00ff00ffu) + ((tot[0] >> 8) & 0x00ff00ffu) + (tot[1] & 0x00ff00ffu) +
                        ((tot[1] >> 8) & 0x00ff00ffu);
    const uint32_t wtot = (t4 & 0xffffu) + (t4 >> 16);
    if (lane == 0) sw[warp] = wtot;
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = lane < NW ? sw[lane] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        if (lane == NW - 1)
            *sbase = remote ? atomicAdd_system(ctr, (unsigned long long)inc) : atomicAdd(ctr, (unsigned long long)inc);
        __syncwarp();
        if (lane < NW) sw[lane] = inc - v;  // exclusive warp offsets
    }
    __syncthreads();
    T* wout = out + (*sbase + sw[warp]);
    uint32_t run = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = 4 * h + jj;
            uint32_t at = run + ((excl[h] >> (8 * jj)) & 0xffu);
#pragma unroll
            for (int cc = 0; cc < VN; ++cc) {
                const uint32_t pp = (bits >> (j * VN + cc)) & 1u;
                if (SDFGB_P_STAGE) {
                    if (pp) stage[at] = vget<V, T>(x[j], cc);
                } else {
                    st_pred(wout, at, vget<V, T>(x[j], cc), pp);
                }
                at += pp;
            }
            run += (tot[h] >> (8 * jj)) & 0xffu;
        }
    }
    if (SDFGB_P_STAGE) {  // the warp's survivors leave as full 128 B lines
        __syncwarp();
        for (uint32_t i = lane; i < wtot; i += 32) wout[i] = stage[i];
        __syncwarp();
    }
}

template <typename T, int OP>
__global__ void __launch_bounds__(kPBlock, SDFGB_P_MINB)
query_push_kernel(const T* __restrict__ col, int64_t n, T thr, T* __restrict__ out,
                  unsigned long long* __restrict__ count, unsigned long long* __restrict__ ctr,
                  unsigned long long* __restrict__ done, int remote) {
    // remote: `out` and `ctr` are the gathering rank's output and reservation
    // counter mapped over NVLink (peer memory); every rank's tiles reserve
    // their slots there with one system-scope atomic and store their
    // survivors straight into it -- the compaction and the gather in one
    // pass.  The caller folds the counter after all ranks' launches.
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::n;
    constexpr int NW = kPBlock / 32;
    constexpr int CH = 32 * VN;
    constexpr int WE = kPChunks * CH;  // elements per warp
    constexpr int64_t TILE = push_tile_elems<T>();
    __shared__ uint32_t s_w[2][NW];
    __shared__ unsigned long long s_base[2];
    __shared__ T s_stage[SDFGB_P_STAGE ? NW : 1][SDFGB_P_STAGE ? WE : 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t drop = make_policy(false);
    T* stage = s_stage[SDFGB_P_STAGE ? warp : 0];
    V x[kPChunks];
    uint32_t bits, pk[2];
    if (!SDFGB_P_PERSIST) {
        const int64_t w0 = (int64_t)blockIdx.x * TILE + (int64_t)warp * WE;
        const bool full = w0 + WE <= n;
        if (full) {
#pragma unroll
            for (int j = 0; j < kPChunks; ++j) x[j] = ldg_hint(col + w0 + j * CH + lane * VN, drop);
        }
        push_bits<T, OP>(col, n, w0, lane, thr, drop, full, x, bits, pk);
        push_store<T>(out, ctr, lane, warp, x, bits, pk, s_w[0], &s_base[0], stage, remote != 0);
    } else {
        // persistent: the next tile's loads are issued before this tile's
        // reservation, so the atomic's round trip overlaps HBM traffic
        const int64_t ntiles = (n + TILE - 1) / TILE;
        int64_t t = blockIdx.x;
        V nx[kPChunks];
        auto prefetch = [&](int64_t tt) {
            const int64_t w0 = tt * TILE + (int64_t)warp * WE;
            if (tt < ntiles && w0 + WE <= n) {
#pragma unroll
                for (int j = 0; j < kPChunks; ++j) nx[j] = ldg_hint(col + w0 + j * CH + lane * VN, drop);
            }
        };
        prefetch(t);
        for (int par = 0; t < ntiles; t += gridDim.x, par ^= 1) {
            const int64_t w0 = t * TILE + (int64_t)warp * WE;
            const bool full = w0 + WE <= n;
#pragma unroll
            for (int j = 0; j < kPChunks; ++j) x[j] = nx[j];
            prefetch(t + gridDim.x);
            push_bits<T, OP>(col, n, w0, lane, thr, drop, full, x, bits, pk);
            push_store<T>(out, ctr, lane, warp, x, bits, pk, s_w[par], &s_base[par], stage, remote != 0);
        }
    }
    if (tid == NW - 1) {  // the thread that reserved: publish completion after its reservations
        __threadfence();
        if (atomicAdd(done, 1ull) == (unsigned long long)gridDim.x - 1) {
            __threadfence();
            if (!remote) {
                const unsigned long long total = atomicExch(ctr, 0ull);
                atomicAdd(count, total);
            }
            *done = 0ull;
        }
    }
}

template <typename T>
auto query_push_kernel_for(int op) {
    switch (op) {
    case 0: return query_push_kernel<T, 0>;
    case 1: return query_push_kernel<T, 1>;
    case 2: return query_push_kernel<T, 2>;
    case 3: return query_push_kernel<T, 3>;
    case 4: return query_push_kernel<T, 4>;
    case 5: return query_push_kernel<T, 5>;
    case 6: return query_push_kernel<T, 6>;
    default: return query_push_kernel<T, 7>;
    }
}

template <typename T>
auto query_piece_kernel_for(int op) {
    switch (op) {
    case 0: return query_piece_kernel<T, 0>;
    case 1: return query_piece_kernel<T, 1>;
    case 2: return query_piece_kernel<T, 2>;
    case 3: return query_piece_kernel<T, 3>;
    case 4: return query_piece_kernel<T, 4>;
    case 5: return query_piece_kernel<T, 5>;
    case 6: return query_piece_kernel<T, 6>;
    default: return query_piece_kernel<T, 7>;
    }
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
constexpr int64_t seg_elems() {
    return (int64_t)kQBlock * kQVecPerThread * Vec16<T>::n * kQSubs;
}

// rounds and CTAs for n elements: G co-resident CTAs (<= kQBlock so one
// block-wide read gathers a round), rounds = ceil(n / (G * S))
template <typename T>
void query_geometry(int64_t n, int64_t capacity, int64_t& G, int64_t& rounds) {
    const int64_t segs = (n + seg_elems<T>() - 1) / seg_elems<T>();
    G = std::max<int64_t>(1, std::min<int64_t>({segs, capacity, (int64_t)kQBlock}));
    rounds = (segs + G - 1) / G;
}

// Exact predicate in the element type: for a float v and a double t,
//   v <  t  <=>  v <  up(t)      v <= t  <=>  v <= down(t)
//   v >  t  <=>  v >  down(t)    v >= t  <=>  v >= up(t)
//   v == t  <=>  t representable && v == (float)t   (else constant false)
// with up/down = t rounded toward +/-inf; NaN thresholds stay NaN.  So the
// kernel runs one FSETP per element instead of widening to double.
template <typename T>
void fold_threshold(int op, double thr, int& op_out, T& t_out) {
    op_out = op;
    t_out = (T)thr;
    if constexpr (sizeof(T) == 4) {
        if (thr != thr) return;
        const float f = (float)thr;
        const float up = (double)f < thr ? std::nextafter(f, INFINITY) : f;
        const float dn = (double)f > thr ? std::nextafter(f, -INFINITY) : f;
        const bool exact = (double)f == thr;
        switch (op) {
        case SDFGB_CMP_LT: case SDFGB_CMP_GE: t_out = up; break;
        case SDFGB_CMP_LE: case SDFGB_CMP_GT: t_out = dn; break;
        case SDFGB_CMP_EQ: if (!exact) op_out = 6; break;
        default: if (!exact) op_out = 7; break;
        }
    }
}

template <typename T, bool VEC>
auto query_kernel_for(int op) {
    switch (op) {
    case 0: return query_kernel<T, VEC, 0>;
    case 1: return query_kernel<T, VEC, 1>;
    case 2: return query_kernel<T, VEC, 2>;
    case 3: return query_kernel<T, VEC, 3>;
    case 4: return query_kernel<T, VEC, 4>;
    case 5: return query_kernel<T, VEC, 5>;
    case 6: return query_kernel<T, VEC, 6>;
    default: return query_kernel<T, VEC, 7>;
    }
}

template <typename T>
int launch_query(const T* col, int64_t n, int op, double thr, T* out, int64_t* count, void* ws,
                 size_t ws_bytes, void* stream) {
    const bool ordered = (op & SDFGB_QUERY_ORDERED) != 0;
    op &= ~SDFGB_QUERY_ORDERED;
    if (n < 0 || op < 0 || op > 5 || !count || (n > 0 && (!col || !out || !ws)))
        return set_error(SDFGB_ERR_INVALID, "query: bad arguments");
    if (n == 0) return SDFGB_OK;
    if ((uint64_t)n > kValueMask) return set_error(SDFGB_ERR_INVALID, "query: n too large");
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
    int kop;
    T tt;
    fold_threshold<T>(op, thr, kop, tt);
    if (!ordered && vec) {
        // unordered push: one CTA per 32 KB tile, one reservation atomic each
        constexpr int64_t tile = push_tile_elems<T>();
        int64_t G = (n + tile - 1) / tile;
        auto pk = query_push_kernel_for<T>(kop);
        if (SDFGB_P_PERSIST) {
            static int pocc[2][8] = {};
            int& po = pocc[sizeof(T) == 8][kop];
            if (po == 0) SDFGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&po, pk, kPBlock, 0));
            G = std::min<int64_t>(G, (int64_t)std::max(po, 1) * num_sms());
        }
        if (G > 0x7fffffff) return set_error(SDFGB_ERR_INVALID, "query: n too large");
        pk<<<(unsigned)G, kPBlock, 0, s>>>(col, n, tt, out, C, &W->ticket, &W->done, 0);
        SDFGB_LAUNCHED("query_push_kernel");
        return SDFGB_OK;
    }
    if (vec && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        // piece kernel: co-resident CTAs (the compactors wait on every CTA's counts)
        auto pk = query_piece_kernel_for<T>(kop);
        static int pocc[2][8] = {};
        int& po = pocc[sizeof(T) == 8][kop];
        if (po == 0) SDFGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&po, pk, kQPBlock, 0));
        const int64_t G = std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(po, 1) * num_sms(), (int64_t)kTBlock));
        auto* cnts = W->status;
        uint32_t ep = epoch;
        // cooperative: every CTA co-resident (B waits on all CTAs' counts)
        void* args[] = {(void*)&col, (void*)&n, (void*)&tt, (void*)&out, (void*)&C, (void*)&cnts, (void*)&ep};
        SDFGB_CUDA(cudaLaunchCooperativeKernel((const void*)pk, dim3((unsigned)G), dim3(kQPBlock), args, 0, s));
        return SDFGB_OK;
    }
    auto kern = vec ? query_kernel_for<T, true>(kop) : query_kernel_for<T, false>(kop);
    static int occ[2][2][8] = {};  // [f64][vec][op] resident CTAs per SM
    int& o = occ[sizeof(T) == 8][vec][kop];
    if (o == 0) SDFGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kQBlock, 0));
    int64_t G, rounds;
    query_geometry<T>(n, (int64_t)std::max(o, 1) * num_sms(), G, rounds);
    // every CTA must be resident (rounds wait on all of them): cooperative launch
    void* args[] = {(void*)&col, (void*)&n, (void*)&tt, (void*)&out, (void*)&C, (void*)&W,
                    (void*)&rounds, (void*)&epoch};
    SDFGB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)G), dim3(kQBlock), args, 0, s));
    return SDFGB_OK;
}

}  // namespace
}  // namespace sdfgb

#if SDFGB_Q_TIMING
extern "C" int sdfgb_debug_query_timing(void* host) {
    return cudaMemcpyFromSymbol(host, sdfgb::g_qtime, sizeof(sdfgb::g_qtime)) == cudaSuccess ? 0 : 1;
}
#endif
extern "C" size_t sdfgb_query_workspace_bytes(int64_t n, int elem_bytes) {
    // one status word per (round, CTA) slot of the register-path kernel
    // (rounds * G <= segments + G - 1) or per (piece, CTA) of the piece
    // kernel (G <= kTBlock), whichever is more
    const int64_t seg = elem_bytes == 8 ? sdfgb::seg_elems<double>() : sdfgb::seg_elems<float>();
    const int64_t segs = (n + seg - 1) / seg;
    const int64_t pieces = (n * (int64_t)elem_bytes + sdfgb::kPieceBytes - 1) / sdfgb::kPieceBytes;
    const int64_t slots = std::max<int64_t>(segs + sdfgb::kTBlock, pieces * sdfgb::kTBlock);
    return offsetof(sdfgb::QueryWs, status) + (size_t)slots * 8;
}
extern "C" int sdfgb_query_f32(const float* col, int64_t n, int op, double thr, float* out_vals,
                               int64_t* count, void* ws, size_t ws_bytes, void* stream) {
    return sdfgb::launch_query<float>(col, n, op, thr, out_vals, count, ws, ws_bytes, stream);
}
extern "C" int sdfgb_query_f64(const double* col, int64_t n, int op, double thr, double* out_vals,
                               int64_t* count, void* ws, size_t ws_bytes, void* stream) {
    return sdfgb::launch_query<double>(col, n, op, thr, out_vals, count, ws, ws_bytes, stream);
}

// Fused compaction + gather over NVLink (multi-GPU query, gathered output):
// this rank's survivors go straight into the gathering rank's out_root at
// slots reserved with system-scope atomics on its counter reserve_root
// (both mapped into this process).  After every rank's call has completed
// (the caller's barrier), out_root[0:*reserve_root) holds all survivors in
// unspecified order; the caller adds *reserve_root to count and re-zeroes it.
extern "C" int sdfgb_query_f32_p2p(const float* col, int64_t n, int op, double thr, float* out_root,
                                   int64_t* reserve_root, void* ws, size_t ws_bytes, void* stream) {
    using namespace sdfgb;
    if (n < 0 || op < 0 || op > 5 || !reserve_root || (n > 0 && (!col || !out_root || !ws)))
        return set_error(SDFGB_ERR_INVALID, "query_p2p: bad arguments");
    if (n == 0) return SDFGB_OK;
    if ((reinterpret_cast<uintptr_t>(col) & 15) != 0)
        return set_error(SDFGB_ERR_INVALID, "query_p2p: col must be 16-byte aligned");
    if (ws_bytes < sdfgb_query_workspace_bytes(n, 4) || (reinterpret_cast<uintptr_t>(ws) & 7) != 0)
        return set_error(SDFGB_ERR_WORKSPACE, "query_p2p: workspace too small or misaligned");
    auto* W = reinterpret_cast<QueryWs*>(ws);
    cudaStream_t s = as_stream(stream);
    int kop;
    float tt;
    fold_threshold<float>(op, thr, kop, tt);
    constexpr int64_t tile = push_tile_elems<float>();
    int64_t G = (n + tile - 1) / tile;
    auto pk = query_push_kernel_for<float>(kop);
    static int po[8] = {};
    if (po[kop] == 0) SDFGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&po[kop], pk, kPBlock, 0));
    G = std::min<int64_t>(G, (int64_t)std::max(po[kop], 1) * num_sms());
    pk<<<(unsigned)G, kPBlock, 0, s>>>(col, n, tt, out_root, nullptr,
                                       reinterpret_cast<unsigned long long*>(reserve_root), &W->done, 1);
    SDFGB_LAUNCHED("query_push_kernel");
    return SDFGB_OK;
}
