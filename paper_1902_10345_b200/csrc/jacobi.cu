// jacobi.cu -- K4: the double-buffered 2-D stencil time loop.
//
// Reference: guard loop ``for (t = 0; t < T; t = t + 1)`` (loops.py:31-61 ->
// codegen.py:688-699) around a map over the interior [1:N-2]^2 whose tasklet
// reads A[t%2, i+di, j+dj] and writes A[(t+1)%2, i, j]; borders are never
// written; the result is in A[T%2] and both planes are outputs.  The tasklet
// ``o = coef * (c + n + s + w + e)`` evaluates left to right
// (tasklets.py:430-444): coef * ((((t0 + t1) + t2) + t3) + t4).  The kernel
// keeps that exact order (no FMA contraction is possible in it), so the fp32
// result is bit-identical to the fp32 restatement and the f64 result to the
// reference itself.
//
// B200 design (HBM-bound: 4N^2 read + 4(N-2)^2 write per step):
//   * a warp owns a 128-column strip (float4 per lane) and streams down a
//     chunk of rows with a sliding north/centre/south register window, so
//     each input element is loaded from DRAM once per step;
//   * west/east neighbours come from lane shuffles, only the two strip-edge
//     columns are extra (L1/L2-resident) loads;
//   * four rows are fetched per iteration to keep 4 x 16 B in flight/thread;
//   * the canonical c,n,s,w,e order is a compile-time fast path; any other
//     order of up to 9 neighbours runs the same kernel through a select chain.
#include <algorithm>

#include "common.cuh"

namespace sdfgb {
namespace {

constexpr int kJBlock = 256;
constexpr int kJRows = 32;   // rows per warp chunk
constexpr int kJAhead = 4;   // rows fetched per iteration

struct Terms {
    int n;
    int code[9];  // (di+1)*3 + (dj+1)
};

template <typename T, int VW>
struct RowVec {
    T v[VW];
};

template <typename T, int VW>
__device__ __forceinline__ RowVec<T, VW> load_row(const T* __restrict__ p, int64_t i, int64_t N,
                                                  int64_t j, bool in) {
    RowVec<T, VW> r;
    if (!in) {
#pragma unroll
        for (int c = 0; c < VW; ++c) r.v[c] = T(0);
        return r;
    }
    if constexpr (VW == 4 && sizeof(T) == 4) {
        float4 x = *reinterpret_cast<const float4*>(p + i * N + j);
        r.v[0] = x.x; r.v[1] = x.y; r.v[2] = x.z; r.v[3] = x.w;
    } else if constexpr (VW == 2 && sizeof(T) == 8) {
        double2 x = *reinterpret_cast<const double2*>(p + i * N + j);
        r.v[0] = x.x; r.v[1] = x.y;
    } else {
#pragma unroll
        for (int c = 0; c < VW; ++c) r.v[c] = (j + c < N) ? p[i * N + j + c] : T(0);
    }
    return r;
}

// neighbour (dj in -1..1) of component c within the strip, using shuffles
template <typename T, int VW>
__device__ __forceinline__ T horiz(const RowVec<T, VW>& r, T west_edge, T east_edge, int c, int dj,
                                   int lane) {
    const int cc = c + dj;
    if (cc >= 0 && cc < VW) return r.v[cc];
    if (cc < 0) {
        T w = __shfl_up_sync(0xffffffffu, r.v[VW - 1], 1);
        return lane == 0 ? west_edge : w;
    }
    T e = __shfl_down_sync(0xffffffffu, r.v[0], 1);
    return lane == 31 ? east_edge : e;
}

template <typename T, int VW, bool CANON>
__global__ void __launch_bounds__(kJBlock)
jacobi_step_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t N, int64_t rows,
                   int64_t g0, int64_t r0, int64_t r1, T coef, Terms terms) {
    // plane rows are local [0, rows); global row = g0 + local.  Interior rows
    // written: local rows in [r0, r1) (caller clips to global [1, N-2]).
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * kJBlock + threadIdx.x) >> 5;
    const int64_t strip_w = 32 * VW;
    const int64_t nstrips = (N + strip_w - 1) / strip_w;
    const int64_t strip = gw % nstrips;
    const int64_t chunk = gw / nstrips;
    const int64_t i_begin = r0 + chunk * kJRows;
    if (i_begin >= r1) return;
    const int64_t i_end = min(r1, i_begin + kJRows);
    const int64_t j0 = strip * strip_w;
    const int64_t j = j0 + (int64_t)lane * VW;
    const bool jin = j < N;

    auto edge = [&](int64_t i, bool west) -> T {
        if (west) return (lane == 0 && j0 > 0) ? src[i * N + j0 - 1] : T(0);
        return (lane == 31 && j0 + strip_w < N) ? src[i * N + j0 + strip_w] : T(0);
    };

    RowVec<T, VW> rn = load_row<T, VW>(src, i_begin - 1, N, j, jin);
    RowVec<T, VW> rc = load_row<T, VW>(src, i_begin, N, j, jin);
    T wn = edge(i_begin - 1, true), en = edge(i_begin - 1, false);
    T wc = edge(i_begin, true), ec = edge(i_begin, false);

    for (int64_t i = i_begin; i < i_end; i += kJAhead) {
        RowVec<T, VW> rs[kJAhead];
        T ws_[kJAhead], es_[kJAhead];
#pragma unroll
        for (int a = 0; a < kJAhead; ++a) {
            const bool live = i + a < i_end;
            rs[a] = load_row<T, VW>(src, i + a + 1, N, j, jin && live);
            ws_[a] = live ? edge(i + a + 1, true) : T(0);
            es_[a] = live ? edge(i + a + 1, false) : T(0);
        }
#pragma unroll
        for (int a = 0; a < kJAhead; ++a) {
            if (i + a >= i_end) break;  // warp-uniform
            const RowVec<T, VW>& S = rs[a];
            RowVec<T, VW> o;
#pragma unroll
            for (int c = 0; c < VW; ++c) {
                T acc;
                if constexpr (CANON) {
                    // ((((c + n) + s) + w) + e) * coef, reference order
                    acc = rc.v[c] + rn.v[c];
                    acc = acc + S.v[c];
                    acc = acc + horiz<T, VW>(rc, wc, ec, c, -1, lane);
                    acc = acc + horiz<T, VW>(rc, wc, ec, c, +1, lane);
                } else {
                    T nb[9];
#pragma unroll
                    for (int di = 0; di < 3; ++di) {
                        const RowVec<T, VW>& R = di == 0 ? rn : (di == 1 ? rc : S);
                        const T we = di == 0 ? wn : (di == 1 ? wc : ws_[a]);
                        const T ea = di == 0 ? en : (di == 1 ? ec : es_[a]);
#pragma unroll
                        for (int dj = 0; dj < 3; ++dj) nb[di * 3 + dj] = horiz<T, VW>(R, we, ea, c, dj - 1, lane);
                    }
                    auto pick = [&](int code) -> T {
                        T r = nb[0];
#pragma unroll
                        for (int q = 1; q < 9; ++q) r = code == q ? nb[q] : r;
                        return r;
                    };
                    acc = pick(terms.code[0]);
#pragma unroll
                    for (int k = 1; k < 9; ++k)
                        if (k < terms.n) acc = acc + pick(terms.code[k]);
                }
                o.v[c] = coef * acc;
            }
            const int64_t gi = i + a;
            if (jin) {
                const bool full = (j >= 1) && (j + VW - 1 <= N - 2);
                if (full && (VW == 4 && sizeof(T) == 4)) {
                    *reinterpret_cast<float4*>(dst + gi * N + j) =
                        make_float4((float)o.v[0], (float)o.v[1 % VW], (float)o.v[2 % VW], (float)o.v[3 % VW]);
                } else if (full && (VW == 2 && sizeof(T) == 8)) {
                    *reinterpret_cast<double2*>(dst + gi * N + j) =
                        make_double2((double)o.v[0], (double)o.v[1 % VW]);
                } else {
#pragma unroll
                    for (int c = 0; c < VW; ++c) {
                        const int64_t jj = j + c;
                        if (jj >= 1 && jj <= N - 2) dst[gi * N + jj] = o.v[c];
                    }
                }
            }
            rn = rc; wn = wc; en = ec;
            rc = S; wc = ws_[a]; ec = es_[a];
        }
    }
}

bool parse_terms(const int32_t* di, const int32_t* dj, int nterms, Terms& t, bool& canon) {
    if (nterms < 1 || nterms > 9 || !di || !dj) return false;
    t.n = nterms;
    for (int k = 0; k < 9; ++k) t.code[k] = 4;
    for (int k = 0; k < nterms; ++k) {
        if (di[k] < -1 || di[k] > 1 || dj[k] < -1 || dj[k] > 1) return false;
        t.code[k] = (di[k] + 1) * 3 + (dj[k] + 1);
    }
    static const int kCanon[5] = {4, 1, 7, 3, 5};  // c, n, s, w, e
    canon = nterms == 5;
    for (int k = 0; canon && k < 5; ++k) canon = t.code[k] == kCanon[k];
    return true;
}

template <typename T>
int launch_step(const T* src, T* dst, int64_t N, int64_t rows, int64_t g0, int64_t r0, int64_t r1,
                T coef, const Terms& terms, bool canon, cudaStream_t s) {
    if (r1 <= r0) return SDFGB_OK;
    constexpr int VWv = sizeof(T) == 4 ? 4 : 2;
    const bool vec = (N % VWv) == 0 && (reinterpret_cast<uintptr_t>(src) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(dst) % 16 == 0);
    const int VW = vec ? VWv : 1;
    const int64_t nstrips = (N + 32 * VW - 1) / (32 * VW);
    const int64_t chunks = (r1 - r0 + kJRows - 1) / kJRows;
    const int64_t warps = nstrips * chunks;
    const unsigned blocks = (unsigned)((warps * 32 + kJBlock - 1) / kJBlock);
    if (vec) {
        if (canon)
            jacobi_step_kernel<T, VWv, true><<<blocks, kJBlock, 0, s>>>(src, dst, N, rows, g0, r0, r1, coef, terms);
        else
            jacobi_step_kernel<T, VWv, false><<<blocks, kJBlock, 0, s>>>(src, dst, N, rows, g0, r0, r1, coef, terms);
    } else {
        if (canon)
            jacobi_step_kernel<T, 1, true><<<blocks, kJBlock, 0, s>>>(src, dst, N, rows, g0, r0, r1, coef, terms);
        else
            jacobi_step_kernel<T, 1, false><<<blocks, kJBlock, 0, s>>>(src, dst, N, rows, g0, r0, r1, coef, terms);
    }
    SDFGB_LAUNCHED("jacobi_step_kernel");
    return SDFGB_OK;
}

template <typename T>
int launch_jacobi(T* A, int64_t N, int64_t T_, double coef, const int32_t* di, const int32_t* dj,
                  int nterms, void* stream) {
    Terms terms;
    bool canon;
    if (N < 0 || T_ < 0 || (N > 0 && !A) || !parse_terms(di, dj, nterms, terms, canon))
        return set_error(SDFGB_ERR_INVALID, "jacobi2d: bad arguments (N=%lld T=%lld nterms=%d)",
                         (long long)N, (long long)T_, nterms);
    if (N < 3 || T_ == 0) return SDFGB_OK;  // empty interior map
    cudaStream_t s = as_stream(stream);
    T* P[2] = {A, A + N * N};
    for (int64_t t = 0; t < T_; ++t)
        SDFGB_TRY(launch_step<T>(P[t & 1], P[(t + 1) & 1], N, N, 0, 1, N - 1, (T)coef, terms, canon, s));
    return SDFGB_OK;
}

}  // namespace
}  // namespace sdfgb

extern "C" int sdfgb_jacobi2d_f32(float* A, int64_t N, int64_t T, double coef, const int32_t* di,
                                  const int32_t* dj, int nterms, void* stream) {
    return sdfgb::launch_jacobi<float>(A, N, T, coef, di, dj, nterms, stream);
}
extern "C" int sdfgb_jacobi2d_f64(double* A, int64_t N, int64_t T, double coef, const int32_t* di,
                                  const int32_t* dj, int nterms, void* stream) {
    return sdfgb::launch_jacobi<double>(A, N, T, coef, di, dj, nterms, stream);
}
extern "C" int sdfgb_jacobi2d_step_f32(const float* src, float* dst, int64_t N, int64_t rows,
                                       int64_t g0, int64_t r0, int64_t r1, double coef,
                                       const int32_t* di, const int32_t* dj, int nterms,
                                       void* stream) {
    sdfgb::Terms terms;
    bool canon;
    if (N < 3 || rows < 0 || !src || !dst || !sdfgb::parse_terms(di, dj, nterms, terms, canon))
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_step: bad arguments");
    (void)g0;
    return sdfgb::launch_step<float>(src, dst, N, rows, g0, r0, r1, (float)coef, terms, canon,
                                     sdfgb::as_stream(stream));
}
