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
#include <atomic>
#include <type_traits>

#include "tma.cuh"

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

// ---------------------------------------------------------------------------
// Temporal blocking (canonical 5-point order, fp32): one launch advances KT
// (odd) time steps.  A CTA TMA-loads its 112 x 96 output tile plus a halo
// (8 columns, KT rows each side: a 128 x (96 + 2KT) region) into shared
// memory and ping-pongs KT steps between two smem buffers; only the tile
// centre -- whose KT-step dependency cone lies inside the region -- is
// written back.  Per KT steps HBM sees ~1.3 plane reads + 1 plane write
// instead of KT of each, and every point is still
// coef * ((((c + n) + s) + w) + e) in fp32: bit-identical to one-step.
//
// Borders: the reference never writes the global border, and step t reads
// plane t % 2 -- whose border is that plane's own.  Buffer 0 (states read
// from plane p) holds plane p's border from the TMA load; buffer 1 (states
// of plane p^1) gets plane p^1's border copied in once; steps never write
// border points, so each buffer keeps the right plane's border.
//
// Work mapping: warp w owns a band of rows, lane l owns columns 4l..4l+3
// (one float4); a north/centre register window slides down the band so each
// step costs one LDS.128 + two shuffles per 4 points.
#ifndef SDFGB_J_TY
#define SDFGB_J_TY 96
#endif
#ifndef SDFGB_J_THREADS
#define SDFGB_J_THREADS 256
#endif
#ifndef SDFGB_J_MINB
#define SDFGB_J_MINB 2
#endif
constexpr int kTbRX = 128, kTbPad = 8, kTbX = kTbRX - 2 * kTbPad, kTbY = SDFGB_J_TY, kTbThreads = SDFGB_J_THREADS;
constexpr int kTbWarps = kTbThreads / 32;

__host__ __device__ constexpr int tb_rows(int k) { return kTbY + 2 * k; }
// two region buffers + kTbPadRows pad rows (a fused sweep of F steps may
// read rows up to RY+F-2 of a buffer: halo garbage, but it must be inside
// the allocation) + mbarrier
constexpr int kTbPadRows = 2;
#ifndef SDFGB_J_ONE_SWEEP
#define SDFGB_J_ONE_SWEEP 1
#endif
#ifndef SDFGB_J_F3
#define SDFGB_J_F3 1  // odd step counts start with a 3-step sweep (else a 1-step one)
#endif
__host__ __device__ constexpr size_t tb_smem(int k) {
    return (size_t)(2 * tb_rows(k) + kTbPadRows) * kTbRX * 4 + 128 + 64;
}

template <int KT>
__global__ void __launch_bounds__(kTbThreads, SDFGB_J_MINB)
jacobi_tb_kernel(const __grid_constant__ CUtensorMap src, const float* dst_in,
                 float* __restrict__ dst, int M, int N, float coef, int steps) {
    // planes are M rows x N columns; the border is the plane's edge (rows 0
    // and M-1, columns 0 and N-1) -- the reference's square case is M == N,
    // a multi-GPU slab puts ghost rows there (multigpu.jacobi)
    constexpr int RY = tb_rows(KT);
    // dynamic smem starts at the CTA window base (no static smem here), so it
    // is 1 KB-aligned for TMA; indexing the extern array directly keeps the
    // accesses in the shared state space (LDS/STS, not generic LD/ST)
    extern __shared__ __align__(1024) float tb_smem_f[];
    float* buf0 = tb_smem_f;
    float* buf1 = tb_smem_f + kTbRX * RY;
    uint64_t* bar = reinterpret_cast<uint64_t*>(tb_smem_f + (2 * RY + kTbPadRows) * kTbRX);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = blockIdx.x * kTbX, y0 = blockIdx.y * kTbY;
    const int gx0 = x0 - kTbPad, gy0 = y0 - KT;  // region origin (may be negative: TMA zero-fills)
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, (uint32_t)(kTbRX * RY * 4));
        tma_load_2d(buf0, &src, bar, gx0, gy0);
    }
    // does the region touch the global border (or beyond)?  CTA-uniform
    const bool edge = gx0 <= 0 || gy0 <= 0 || gx0 + kTbRX - 1 >= N - 1 || gy0 + RY - 1 >= M - 1;
    if (edge) {  // buffer 1 carries plane p^1's border: copy just the border lines in the region
        for (int q = threadIdx.x; q < 2 * kTbRX + 2 * RY; q += kTbThreads) {
            int ry, rx;  // region coordinates of candidate q
            if (q < 2 * kTbRX) {  // border rows 0 and N-1
                ry = (q < kTbRX ? 0 : M - 1) - gy0;
                rx = q % kTbRX;
            } else {  // border columns 0 and N-1
                const int k = q - 2 * kTbRX;
                ry = k % RY;
                rx = (k < RY ? 0 : N - 1) - gx0;
            }
            const int gy = gy0 + ry, gx = gx0 + rx;
            if (ry >= 0 && ry < RY && rx >= 0 && rx < kTbRX && gy >= 0 && gy < M && gx >= 0 && gx < N)
                buf1[ry * kTbRX + rx] = dst_in[(int64_t)gy * N + gx];
        }
    }
    __syncthreads();
    mbar_wait(bar, 0);

    // this warp's row band inside [1, RY-2]
    const int rb = 1 + (warp * (RY - 2)) / kTbWarps, re = 1 + ((warp + 1) * (RY - 2)) / kTbWarps;
    const int gx = gx0 + 4 * lane;
    bool colb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) colb[j] = gx + j <= 0 || gx + j >= N - 1;

    // one stencil row from its north/centre/south float4s, reference order
    auto calc = [&](const float4& nq, const float4& cq, const float4& sq) -> float4 {
        const float lft = __shfl_up_sync(0xffffffffu, cq.w, 1);   // lane 0: region edge, unused
        const float rgt = __shfl_down_sync(0xffffffffu, cq.x, 1); // lane 31: region edge, unused
        const float cc[4] = {cq.x, cq.y, cq.z, cq.w};
        const float nn[4] = {nq.x, nq.y, nq.z, nq.w};
        const float ss[4] = {sq.x, sq.y, sq.z, sq.w};
        const float ww[4] = {lft, cq.x, cq.y, cq.z};
        const float ee[4] = {cq.y, cq.z, cq.w, rgt};
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float acc = __fadd_rn(cc[j], nn[j]);
            acc = __fadd_rn(acc, ss[j]);
            acc = __fadd_rn(acc, ww[j]);
            acc = __fadd_rn(acc, ee[j]);
            o[j] = __fmul_rn(coef, acc);
        }
        return make_float4(o[0], o[1], o[2], o[3]);
    };
    auto ldrow = [&](const float* in, int rr) {
        rr = rr < 0 ? 0 : (rr > RY - 1 ? RY - 1 : rr);  // beyond the region: halo garbage, never kept
        return *reinterpret_cast<const float4*>(in + rr * kTbRX + 4 * lane);
    };

    const float* cur = buf0;
    float* oth = buf1;
    auto flip = [&]() {
        const float* t = cur;
        cur = oth;
        oth = const_cast<float*>(t);
    };
    // one step cur -> oth, one smem row load + store per output row
    auto single_step = [&]() {
        const float* in = cur;
        float* out = oth;
        float4 n4 = ldrow(in, rb - 1);
        float4 c4 = ldrow(in, rb);
        auto row = [&](int r, const float4& nq, const float4& cq, const float4& sq) {
            const float4 o4 = calc(nq, cq, sq);
            float* op = out + r * kTbRX + 4 * lane;
            if (!edge) {
                *reinterpret_cast<float4*>(op) = o4;
            } else {
                const float o[4] = {o4.x, o4.y, o4.z, o4.w};
                const int gy = gy0 + r;
                const bool rowb = gy <= 0 || gy >= M - 1;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (!rowb && !colb[j]) op[j] = o[j];
            }
        };
        // three rows per iteration with the window's names rotating
        // (n4, c4, s4) -> (c4, s4, n4) -> (s4, n4, c4): every load lands in a
        // register whose old row is dead, so the loop carries no moves
        // (the two-row version spent ~12 MOVs per row on the rotation)
        int r = rb;
        float4 s4;
        auto ld = [&](int rr) { return *reinterpret_cast<const float4*>(in + rr * kTbRX + 4 * lane); };
        for (; r + 2 < re; r += 3) {
            s4 = ld(r + 1);
            row(r, n4, c4, s4);
            n4 = ld(r + 2);
            row(r + 1, c4, s4, n4);
            c4 = ld(r + 3);
            row(r + 2, s4, n4, c4);  // the window for row r+3 is (n4, c4) again
        }
        if (r < re) {
            s4 = ld(r + 1);
            row(r, n4, c4, s4);
            if (r + 1 < re) row(r + 1, c4, s4, ld(r + 2));
        }
        __syncthreads();
        flip();
    };

    if (!edge) {
        // Interior regions (no global border inside): F steps per sweep.
        // The intermediate states never touch smem -- each warp recomputes
        // them for its band plus a shrinking margin -- so shared-memory
        // traffic and barriers per step drop F-fold (the one-step sweep is
        // bound by LDS/STS/SHFL bandwidth).  Intermediate values outside
        // the band's cone are garbage exactly like the halo of the one-step
        // path: the valid area still shrinks one row/column per step.  The
        // last sweep stores the tile centre straight from registers to HBM.
        //
        // Level k (0 = the sweep's input state) keeps a 3-row window; row r
        // of level k lives in slot (r + k - base) mod 3, so every sub-step
        // writes the same slot at every level and the unrolled loop needs no
        // register moves.  Streaming input row j computes level k row j - k.
        auto sweep = [&](auto f_tag, auto last_tag) {
            constexpr int F = decltype(f_tag)::value;
            constexpr bool LAST = decltype(last_tag)::value;
            auto put = [&](int r, const float4& v) {
                if constexpr (!LAST) {
                    *reinterpret_cast<float4*>(oth + r * kTbRX + 4 * lane) = v;
                } else {
                    if (r >= KT && r < KT + kTbY && lane >= kTbPad / 4 && lane < (kTbPad + kTbX) / 4)
                        *reinterpret_cast<float4*>(dst + (int64_t)(gy0 + r) * N + gx) = v;
                }
            };
            float4 w[F][3];
            const int j0 = rb - F;  // first input row of the cone
            // prologue: input rows j0 .. j0+2F-1 fill the windows; level k
            // row j-k is valid (and computed) once j >= j0 + 2k
#pragma unroll
            for (int p = 0; p < 2 * F; ++p) {
                const int sl = ((p - 2 * F + 1) % 3 + 3) % 3;
                const int sn = (sl + 1) % 3, sc = (sl + 2) % 3;  // north / centre slots of the level below
                w[0][sl] = ldrow(cur, j0 + p);
#pragma unroll
                for (int k = 1; k < F; ++k)
                    if (p >= 2 * k) w[k][sl] = calc(w[k - 1][sn], w[k - 1][sc], w[k - 1][sl]);
            }
            // main stream: input row j = i + 1 + u produces output row j - F
            auto sub = [&](int i, int u) {
                const int sl = (1 + u) % 3, sn = (u + 2) % 3, sc = u % 3;  // south (new) / north / centre
                w[0][sl] = *reinterpret_cast<const float4*>(cur + (i + 1 + u) * kTbRX + 4 * lane);
#pragma unroll
                for (int k = 1; k < F; ++k) w[k][sl] = calc(w[k - 1][sn], w[k - 1][sc], w[k - 1][sl]);
                put(i + 1 + u - F, calc(w[F - 1][sn], w[F - 1][sc], w[F - 1][sl]));
            };
            int i = j0 + 2 * F - 1;  // rows read below reach re-1+F <= RY-2+F: the pad rows
            for (; i + 3 - F <= re - 1; i += 3) {
                sub(i, 0);
                sub(i, 1);
                sub(i, 2);
            }
            if (i + 1 - F <= re - 1) sub(i, 0);
            if (i + 2 - F <= re - 1) sub(i, 1);
        };
        int st = 0;
        auto run = [&](auto f_tag) {
            constexpr int F = decltype(f_tag)::value;
            if (st + F == steps) {
                sweep(f_tag, std::true_type{});
            } else {
                sweep(f_tag, std::false_type{});
                __syncthreads();
                flip();
            }
            st += F;
        };
        // without SDFGB_J_ONE_SWEEP: KT = 7 -> 3 + 2 + 2;  5 -> 3 + 2;  3 -> 3
        if (steps == 1) {
            single_step();
            st = 1;
        } else {
#if SDFGB_J_ONE_SWEEP
            // one fused sweep of all `steps` levels: no intermediate smem
            // round trip or barrier at all (7 steps: 29.4 -> 28.2 us/step;
            // 4+3 measured 28.4, 5+2 29.2, 3+2+2 29.4).  Level-0 reads reach
            // row RY + steps - 2 of buffer 0, inside buffer 1: halo garbage
            // that never reaches the kept centre.
            if constexpr (KT >= 3 && (KT & 1)) {
                if (steps == KT) {
                    run(std::integral_constant<int, KT>{});
                    return;
                }
            }
#endif
            if (steps & 1) {
                if (SDFGB_J_F3) {
                    run(std::integral_constant<int, 3>{});
                } else {
                    single_step();
                    st = 1;
                }
            }
            while (st < steps) run(std::integral_constant<int, 2>{});
            return;  // the centre is already in HBM
        }
        // only a one-step launch gets here: its result is in smem
    } else {
        for (int st = 0; st < steps; ++st) single_step();
    }
    // write the tile centre (global interior only)
    const float* fin = cur;
    constexpr int CG = kTbX / 4;
    for (int it = threadIdx.x; it < kTbY * CG; it += kTbThreads) {
        const int r = it / CG, g = it % CG;
        const int gy = y0 + r, gxx = x0 + 4 * g;
        if (gy < 1 || gy > M - 2) continue;
        const float4 v = *reinterpret_cast<const float4*>(fin + (KT + r) * kTbRX + kTbPad + 4 * g);
        float* d = dst + (int64_t)gy * N + gxx;
        if (gxx >= 1 && gxx + 3 <= N - 2) {
            *reinterpret_cast<float4*>(d) = v;
        } else {
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (gxx + j >= 1 && gxx + j <= N - 2) d[j] = vv[j];
        }
    }
}

// ---------------------------------------------------------------------------
// Strip streaming (the default temporal-blocking kernel).  One launch still
// advances F (odd) steps, but the unit of work is a WARP, not a CTA tile:
// a warp owns a 128-column strip (112 kept + 8 halo columns each side) of
// H output rows and streams the strip's H + 2F input rows top to bottom.
// Input rows arrive by TMA (128 x 3-row boxes, zero-filled outside the
// plane) into a per-warp 4-stage shared-memory ring -- the next three
// stages are in flight while one is consumed -- and every level 1..F of the
// sweep is computed in registers from a 3-row window of the level below
// (same slot rotation as jacobi_tb_kernel: row r of level k in slot
// (r + k) mod 3, so at input row p every level writes slot p mod 3).
//
// Why: the tile kernel's warps each recompute a shrinking cone of
// 2(F-k) rows per level for a 13-row band, 1.86 computed points per kept
// point at F = 7; a warp that streams 256 rows recomputes 2.3 % in rows,
// 1.14x in columns (16 halo of 128).  The kernel is instruction-issue
// bound, so recomputation is time.
//
// Borders: level k of a launch from plane p holds state t + k, which lives
// in plane p ^ (k & 1); the reference never writes a plane's border, so a
// level's border rows / columns are re-imposed from that plane.  Values
// outside the plane are garbage that only ever feeds border points.
//   * border rows: level k reaches plane row 0 only at input rows p <= F+k
//     (the unrolled prologue, where the test is on compile-time p, k) and
//     row M-1 only in the last 2F input rows (a checked tail loop); the
//     steady-state loop carries no row test.
//   * border columns (the first / last strip only): both planes' border
//     column over the strip's rows is staged in shared memory once, and a
//     row step reads its F-1 values before computing, off the dependency
//     chain of the levels.
#ifndef SDFGB_JSP_F32X2
#define SDFGB_JSP_F32X2 0
#endif
#ifndef SDFGB_JSP_PDL
#define SDFGB_JSP_PDL 1  // programmatic dependent launch between consecutive strip launches
#endif
#ifndef SDFGB_JSP_MINB
#define SDFGB_JSP_MINB 4  // resident CTAs per SM the strip kernel is compiled for (128 registers)
#endif
#ifndef SDFGB_JSP_L0REG
#define SDFGB_JSP_L0REG 1  // level 0 kept in the register window (1 LDS per row instead of 3; 19.43 -> 19.2 ms per J1 loop)
#endif
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
constexpr int kSpWarps = 4, kSpStages = 6, kSpRX = 128, kSpPad = 8, kSpX = kSpRX - 2 * kSpPad;
constexpr int kSpStageF = 3 * kSpRX;  // floats per stage (3 rows)
// the strip kernel needs >= 2 strips (each holds at most one border column)
inline bool strip_ok(int64_t N) { return N > kSpX + kSpPad + 4; }
// per warp: the TMA ring, then [plane 0/1][rows] of its border column
// (rows rounded to 16: every warp's ring stays 128 B aligned for TMA)
__host__ __device__ constexpr int sp_rows(int nrows) { return (nrows + 15) / 16 * 16; }
__host__ __device__ constexpr int sp_warp_floats(int nrows) { return kSpStages * kSpStageF + 2 * sp_rows(nrows); }
__host__ __device__ constexpr size_t sp_smem(int nrows) {
    return (size_t)kSpWarps * sp_warp_floats(nrows) * 4 + kSpWarps * kSpStages * 8;
}

#ifndef SDFGB_JSP_TIMING
#define SDFGB_JSP_TIMING 0  // debug builds: per-warp start/end times (tools/jacobi_timing.py)
#endif
#if SDFGB_JSP_TIMING
constexpr int kSpTimingMax = 1 << 16;
__device__ uint64_t g_sp_timing[kSpTimingMax * 4];
#endif
// How one launch cuts its output rows [ra, rb) of every strip into tiles:
// nbig tall tiles over [ra, rsplit) and nsmall short ones over [rsplit, rb)
// (nbigb / nsmallb for the two border-column strips).
struct StripPlan {
    int ra, rb, rsplit, nbig, nsmall, nbigb, nsmallb, nstrips, hmax;
    __host__ __device__ int group(int g) const {
        return g == 0 ? 2 * nbigb + (nstrips - 2) * nbig : 2 * nsmallb + (nstrips - 2) * nsmall;
    }
    __host__ __device__ int total() const { return group(0) + group(1); }
    // queue entry t -> strip and output rows [y0, ye)
    __host__ __device__ void tile(int t, int& strip, int& y0, int& ye) const {
        const bool big = t < group(0);
        const int u = big ? t : t - group(0);
        const int n = big ? nbig : nsmall, nb = big ? nbigb : nsmallb;
        const int lo = big ? ra : rsplit, hi = big ? rsplit : rb;
        int tl, nt;
        if (u < 2 * nb) {  // (the host guarantees nstrips >= 2)
            strip = (u & 1) ? nstrips - 1 : 0;
            tl = u >> 1;
            nt = nb;
        } else {
            const int ui = u - 2 * nb, ni = nstrips - 2;
            strip = 1 + ui % ni;
            tl = ui / ni;
            nt = n;
        }
        y0 = lo + (int)((int64_t)tl * (hi - lo) / nt);
        ye = lo + (int)((int64_t)(tl + 1) * (hi - lo) / nt);
    }
};

constexpr int kSpSchedSlots = 4096;
// per-launch work counters (next tile, warps done), zero between launches:
// the last warp of a launch re-zeroes its pair; launches (of every F, from
// every host thread) rotate over the slots, so concurrent launches on
// different streams use different counters
__device__ int g_sp_sched[kSpSchedSlots * 2];
std::atomic<int> g_sp_launches{0};

// MIRROR: output rows [mr0, mr1) are also stored moff elements further on --
// into a neighbour rank's ghost rows over NVLink (peer memory), so a slab's
// edge band and its ghost-row transfer are one kernel (multigpu.jacobi, p2p)
template <int F, bool MIRROR = false>
__global__ void __launch_bounds__(kSpWarps * 32, SDFGB_JSP_MINB)
jacobi_strip_kernel(const __grid_constant__ CUtensorMap src_map, const float* src, const float* dst_in,
                    float* dst, int M, int N, StripPlan plan, int nwarps, int sched_slot, float coef,
                    int64_t moff, int mr0, int mr1) {
    // output rows [ra, rb) of the plane (the whole plane, or one band of it).
    // Persistent warps: each takes tiles from the launch's counter until
    // none are left, so the tiles' uneven durations balance out and no
    // block-launch gaps open between waves.
    extern __shared__ __align__(1024) float sp_smem_f[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = blockIdx.x * kSpWarps + warp;
    if (g >= nwarps) return;  // warp-uniform; warps never synchronise with each other
#if SDFGB_JSP_PDL
    // programmatic dependent launch: the CTA launch overlaps the previous
    // kernel's end; nothing is read or written before it has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    int* sched = g_sp_sched + 2 * sched_slot;
    const int nstrips = plan.nstrips;
    const int RP = sp_rows(plan.hmax + 2 * F);  // border-column rows per plane, as sized on the host
    float* ring = sp_smem_f + warp * (kSpStages * kSpStageF + 2 * RP);
    float* bcol = ring + kSpStages * kSpStageF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sp_smem_f + kSpWarps * (kSpStages * kSpStageF + 2 * RP)) +
                     warp * kSpStages;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kSpStages; ++s) mbar_init(bars + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
#if SDFGB_JSP_TIMING
    uint64_t t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int ntaken = 0;
#endif
    auto grab = [&]() {
        int t = 0;
        if (lane == 0) t = atomicAdd(sched, 1);
        return __shfl_sync(0xffffffffu, t, 0);
    };

#if SDFGB_JSP_F32X2
    // packed pairs (points 0,1) and (2,3): per point still
    // coef * ((((c + n) + s) + w) + e), each add.rn/mul.rn.f32x2 lane rounding
    // exactly like the scalar op; w/e of the pairs: (lft, c0) / (c1, c2) and
    // (c1, c2) / (c3, rgt)
    const uint64_t cf2 = pk2(coef, coef);
    auto calc = [&](const float4& nq, const float4& cq, const float4& sq) -> float4 {
        const float lft = __shfl_up_sync(0xffffffffu, cq.w, 1);
        const float rgt = __shfl_down_sync(0xffffffffu, cq.x, 1);
        const uint64_t x12 = pk2(cq.y, cq.z);
        uint64_t a = add2(pk2(cq.x, cq.y), pk2(nq.x, nq.y));
        uint64_t b = add2(pk2(cq.z, cq.w), pk2(nq.z, nq.w));
        a = add2(a, pk2(sq.x, sq.y));
        b = add2(b, pk2(sq.z, sq.w));
        a = add2(a, pk2(lft, cq.x));
        b = add2(b, x12);
        a = add2(a, x12);
        b = add2(b, pk2(cq.w, rgt));
        float4 o;
        up2(mul2(cf2, a), o.x, o.y);
        up2(mul2(cf2, b), o.z, o.w);
        return o;
    };
#else
    auto calc = [&](const float4& nq, const float4& cq, const float4& sq) -> float4 {
        const float lft = __shfl_up_sync(0xffffffffu, cq.w, 1);
        const float rgt = __shfl_down_sync(0xffffffffu, cq.x, 1);
        const float cc[4] = {cq.x, cq.y, cq.z, cq.w};
        const float nn[4] = {nq.x, nq.y, nq.z, nq.w};
        const float ss[4] = {sq.x, sq.y, sq.z, sq.w};
        const float ww[4] = {lft, cq.x, cq.y, cq.z};
        const float ee[4] = {cq.y, cq.z, cq.w, rgt};
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float acc = __fadd_rn(cc[j], nn[j]);
            acc = __fadd_rn(acc, ss[j]);
            acc = __fadd_rn(acc, ww[j]);
            acc = __fadd_rn(acc, ee[j]);
            o[j] = __fmul_rn(coef, acc);
        }
        return make_float4(o[0], o[1], o[2], o[3]);
    };
#endif
    uint32_t sbase = 0;  // stages this warp has consumed before the current tile (ring slot / parity)
    for (int t = grab(); t < plan.total(); t = grab()) {
    // The queue: every strip's tall tiles (rows [ra, rsplit)), then its
    // short ones ([rsplit, rb)), so the short tiles even out the end of the
    // launch.  In each group the two border-column strips come first, cut
    // into up to twice the tiles (their per-row fix-ups cost more); then the
    // interior strips, row-tile major.  Tiles split their rows evenly,
    // >= 16 rows each, so only a tile's checked tail can meet plane row M-1
    // and only its prologue row 0.
    int strip, y0, ye;
    plan.tile(t, strip, y0, ye);
    const int gx0 = strip * kSpX - kSpPad, gx = gx0 + 4 * lane;
    const int nrows = (ye - y0) + 2 * F;  // input rows y0-F .. ye-1+F
    const int nst = (nrows + 2) / 3;
    __syncwarp();  // the previous tile's last ring reads are done
    if (lane == 0) {
        for (int s = 0; s < kSpStages && s < nst; ++s) {
            const int sl = (int)((sbase + s) % kSpStages);
            mbar_expect_tx(bars + sl, kSpStageF * 4);
            tma_load_2d(ring + sl * kSpStageF, &src_map, bars + sl, gx0, y0 - F + 3 * s);
        }
    }
    // a strip holds at most one border column (the host sends planes
    // narrower than two strips to the one-step kernel)
    const bool colb = gx0 <= 0 || gx0 + kSpRX - 1 >= N - 1;
    if (colb) {  // both planes' border column over the strip's input rows
        // (one float per row, 32 KB apart: eight rows per lane in flight at
        // once, or the scattered loads' latency stalls this warp ~10 us)
        const int c = gx0 <= 0 ? 0 : N - 1;
        for (int i0 = 0; i0 < nrows; i0 += 8 * 32) {
            float vs[8], vd[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = i0 + j * 32 + lane, r = y0 - F + i;
                const bool in = i < nrows && r >= 0 && r < M;
                const int64_t o = (int64_t)(in ? r : 0) * N + c;
                vs[j] = in ? __ldg(src + o) : 0.f;
                vd[j] = in ? dst_in[o] : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = i0 + j * 32 + lane;
                if (i < nrows) {
                    bcol[i] = vs[j];
                    bcol[RP + i] = vd[j];
                }
            }
        }
    }
    __syncwarp();
    // level k's border row r (0 or M-1) from plane p ^ (k & 1).  gx and N
    // are multiples of 4: a lane's four columns are all inside the plane or
    // all outside; column 0 is a lane's .x, column N-1 a lane's .w
    auto fix_row = [&](int k, int r, float4& v) {
        if (gx >= 0 && gx < N) v = *reinterpret_cast<const float4*>(((k & 1) ? dst_in : src) + (int64_t)r * N + gx);
    };
    const bool cw = gx == 0, ce = gx == N - 4;

    auto sweep = [&](auto colb_tag) {
        constexpr bool COLB = decltype(colb_tag)::value;
        float4 w[F][3];
#pragma unroll
        for (int k = 0; k < F; ++k)
#pragma unroll
            for (int u = 0; u < 3; ++u) w[k][u] = make_float4(0.f, 0.f, 0.f, 0.f);

        // input row p (plane row y0 - F + p): level k computes row y0-F+p-k,
        // valid once p >= 2k; level F (p >= 2F) is output row y0 + p - 2F.
        // MODE 0: steady state; 1: prologue (PRO = p, compile time); 2: tail
        // (rows may reach M-1)
        // stage state carried from step to step (no per-row division or
        // modulo): `it` = this tile's stage (p / 3), `slot` its ring slot,
        // `par` its mbarrier parity; the ring runs on across tiles
        int it = 0, slot = (int)(sbase % kSpStages);
        uint32_t par = (uint32_t)((sbase / kSpStages) & 1);
        // output row y0 + p - 2F of this lane, advanced by one row per step
        float* drow = dst + (int64_t)(y0 - 2 * F) * N + gx;
        auto step = [&](auto u_tag, int p, auto pro_tag, auto mode_tag) {
            constexpr int u = decltype(u_tag)::value;  // p mod 3
            constexpr int PRO = decltype(pro_tag)::value;
            constexpr int MODE = decltype(mode_tag)::value;
            constexpr int sn = (u + 1) % 3, sc = (u + 2) % 3;
            const int pslot = slot == 0 ? kSpStages - 1 : slot - 1;
            float* stage = ring + slot * kSpStageF;
            const float* prev = ring + pslot * kSpStageF;
            if constexpr (u == 0) {
                // every lane polls and the loop condition is a warp vote, so
                // the warp stays provably converged and the shuffles stay
                // plain SHFLs
                const uint32_t a = smem_u32(bars + slot);
                while (!__all_sync(0xffffffffu, mbar_try_wait(a, par))) {
                }
            }

            // level 0 is read from the ring, not kept in registers: rows
            // p-2 .. p (the previous stage is refilled one stage late)
            auto l0 = [&](int q) {  // q = u - 2 .. u
                const float* b = q >= 0 ? stage + q * kSpRX : prev + (q + 3) * kSpRX;
                return *reinterpret_cast<const float4*>(b + 4 * lane);
            };
#if SDFGB_JSP_L0REG
            // the new row only; rows p-2 and p-1 are still in the register window
            w[0][u] = *reinterpret_cast<const float4*>(stage + u * kSpRX + 4 * lane);
#endif
#pragma unroll
            for (int k = 1; k < F; ++k) {
                if (MODE != 1 || PRO >= 2 * k) {
#if SDFGB_JSP_L0REG
                    w[k][u] = calc(w[k - 1][sn], w[k - 1][sc], w[k - 1][u]);
#else
                    w[k][u] = k == 1 ? calc(l0(u - 2), l0(u - 1), l0(u))
                                     : calc(w[k - 1][sn], w[k - 1][sc], w[k - 1][u]);
#endif
                    if constexpr (COLB) {  // this level's border column value (plane p ^ (k & 1))
                        const float bk = bcol[(k & 1) * RP + p - k];
                        if (cw) w[k][u].x = bk;
                        if (ce) w[k][u].w = bk;
                    }
                    const int r = y0 - F + p - k;
                    if constexpr (MODE == 1) {
                        if (PRO - k <= F && r == 0) fix_row(k, r, w[k][u]);
                    } else if constexpr (MODE == 2) {
                        if (r == M - 1) fix_row(k, r, w[k][u]);
                    }
                }
            }
            if (MODE != 1 || PRO >= 2 * F) {
                const float4 o = calc(w[F - 1][sn], w[F - 1][sc], w[F - 1][u]);
                const int r = y0 + p - 2 * F;
                bool keep = lane >= kSpPad / 4 && lane < (kSpPad + kSpX) / 4;
                if constexpr (MODE == 1) keep = keep && r >= 1;
                if constexpr (MODE == 2) keep = keep && r <= M - 2;
                float* d = drow;
                if constexpr (!COLB) {
                    if (keep) *reinterpret_cast<float4*>(d) = o;
                    if constexpr (MIRROR) {
                        if (keep && r >= mr0 && r < mr1) *reinterpret_cast<float4*>(d + moff) = o;
                    }
                } else {
                    // predicated stores only (no lane-divergent branch, which
                    // would wrap the next shuffles in warp re-convergence):
                    // whole float4s inside the interior, single columns at
                    // the border lanes
                    const bool full = keep && gx >= 1 && gx + 3 <= N - 2;
                    const bool part = keep && !full;
                    if (full) *reinterpret_cast<float4*>(d) = o;
                    if (part && gx >= 1 && gx <= N - 2) d[0] = o.x;
                    if (part && gx + 1 >= 1 && gx + 1 <= N - 2) d[1] = o.y;
                    if (part && gx + 2 >= 1 && gx + 2 <= N - 2) d[2] = o.z;
                    if (part && gx + 3 >= 1 && gx + 3 <= N - 2) d[3] = o.w;
                    if constexpr (MIRROR) {
                        float* m = d + moff;
                        const bool mk = r >= mr0 && r < mr1;
                        if (full && mk) *reinterpret_cast<float4*>(m) = o;
                        if (mk && part && gx >= 1 && gx <= N - 2) m[0] = o.x;
                        if (mk && part && gx + 1 >= 1 && gx + 1 <= N - 2) m[1] = o.y;
                        if (mk && part && gx + 2 >= 1 && gx + 2 <= N - 2) m[2] = o.z;
                        if (mk && part && gx + 3 >= 1 && gx + 3 <= N - 2) m[3] = o.w;
                    }
                }
            }
#if SDFGB_JSP_L0REG
            if constexpr (u == 2) {  // this stage's three rows are in registers: refill it
                __syncwarp();
                const int nx = it + kSpStages;
                if (lane == 0 && nx < nst) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(bars + slot, kSpStageF * 4);
                    tma_load_2d(stage, &src_map, bars + slot, gx0, y0 - F + 3 * nx);
                }
            }
#else
            if constexpr (u == 2) {  // the previous stage is consumed (its last reads fed level 1): refill it
                __syncwarp();
                const int nx = it - 1 + kSpStages;
                if (lane == 0 && it >= 1 && nx < nst) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(bars + pslot, kSpStageF * 4);
                    tma_load_2d(const_cast<float*>(prev), &src_map, bars + pslot, gx0,
                                y0 - F + 3 * nx);
                }
            }
#endif
            if constexpr (u == 2) {  // next stage
                ++it;
                if (++slot == kSpStages) {
                    slot = 0;
                    par ^= 1u;
                }
            }
            drow += N;
        };
        using I0 = std::integral_constant<int, 0>;
        using I1 = std::integral_constant<int, 1>;
        using I2 = std::integral_constant<int, 2>;
        using NP = std::integral_constant<int, -1>;
        using M0 = std::integral_constant<int, 0>;
        using M2 = std::integral_constant<int, 2>;
        constexpr int L = (2 * F + 3) / 3 * 3;  // prologue rows: multiple of 3, > 2F (holds output row y0)
        // prologue, fully unrolled so the level guards fold
        [&]<int... Q>(std::integer_sequence<int, Q...>) {
            (step(std::integral_constant<int, Q % 3>{}, Q, std::integral_constant<int, Q>{},
                  std::integral_constant<int, 1>{}),
             ...);
        }(std::make_integer_sequence<int, L>{});
        // rows from pt on may reach plane row M-1 (level k at p = M-1-y0+F+k)
        const int pt = min(nrows, M - y0 + F);
        int p = L;
        for (; p + 3 <= pt; p += 3) {
            step(I0{}, p, NP{}, M0{});
            step(I1{}, p + 1, NP{}, M0{});
            step(I2{}, p + 2, NP{}, M0{});
        }
        for (; p < nrows; p += 3) {  // checked tail
            step(I0{}, p, NP{}, M2{});
            if (p + 1 < nrows) step(I1{}, p + 1, NP{}, M2{});
            if (p + 2 < nrows) step(I2{}, p + 2, NP{}, M2{});
        }
    };
    if (colb) sweep(std::true_type{});
    else sweep(std::false_type{});
    sbase += nst;
#if SDFGB_JSP_TIMING
    ntaken += 1 + (colb ? 1000 : 0);
#endif
    }  // tiles
    // the launch's last warp re-zeroes the counters for the next launch on this slot
    if (lane == 0 && atomicAdd(sched + 1, 1) == nwarps - 1) {
        sched[0] = 0;
        sched[1] = 0;
        __threadfence();
    }
#if SDFGB_JSP_TIMING
    uint64_t t1 = 0;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (lane == 0 && g < kSpTimingMax) {
        g_sp_timing[g * 4 + 0] = t0;
        g_sp_timing[g * 4 + 1] = t1;
        g_sp_timing[g * 4 + 2] = smid;
        g_sp_timing[g * 4 + 3] = (uint64_t)(ntaken >= 1000) | ((uint64_t)(ntaken % 1000) << 8);
    }
#endif
}

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

// Tiles of one launch: tall tiles (SDFGB_J_STRIP_H rows, default 256: the
// cone recomputation of a tile's first 2F rows is 2 % there) for most rows,
// then about one short tile (SDFGB_J_STRIP_HS rows, default 16) per
// resident warp, queued last, so the persistent warps finish together
// (profiles/r2_jacobi_persistent.txt).
StripPlan strip_plan(int64_t ra, int64_t rb, int64_t nstrips, int64_t resident_warps) {
    static const int hb = std::max(32, env_int("SDFGB_J_STRIP_H", 256));
    static const int hs = std::max(16, env_int("SDFGB_J_STRIP_HS", 16));
    static const int spw = std::max(0, env_int("SDFGB_J_STRIP_SMALL", 1));  // short tiles per warp
    StripPlan p{};
    p.ra = (int)ra;
    p.rb = (int)rb;
    p.nstrips = (int)nstrips;
    const int64_t rows = rb - ra;
    int64_t rs = std::min<int64_t>(rows, (resident_warps * spw + nstrips - 1) / nstrips * hs);
    int64_t nbig = (rows - rs) / hb;
    if (nbig == 0) rs = rows;  // too few rows for a tall tile: all short
    p.rsplit = (int)(rb - rs);
    p.nbig = (int)nbig;
    p.nsmall = (int)std::max<int64_t>(1, std::min<int64_t>(rs / hs, rs / 16));
    if (rs < 16) p.nsmall = 1;  // a band of 8..15 rows: one tile
    if (rs == 0) p.nsmall = 0;  // no short tiles at all (SDFGB_J_STRIP_SMALL=0)
    p.nbigb = (int)std::min<int64_t>(2 * nbig, (rows - rs) / 16);
    p.nsmallb = rs ? (int)std::max<int64_t>(1, std::min<int64_t>(2 * p.nsmall, rs / 16)) : 0;
    const int64_t hbig = nbig ? (rows - rs + nbig - 1) / nbig : 0;
    p.hmax = (int)std::max<int64_t>(hbig, p.nsmall ? (rs + p.nsmall - 1) / p.nsmall : 0);
    return p;
}

template <int F, bool MIRROR = false>
int launch_strip(const float* src, float* dst, int64_t M, int64_t N, int64_t ra, int64_t rb, float coef,
                 cudaStream_t s, int64_t moff = 0, int mr0 = 0, int mr1 = 0) {
    const int64_t nstrips = (N + kSpX - 1) / kSpX;
    // persistent: one co-resident wave of warps (4 CTAs x 4 warps per SM)
    const int64_t resident = (int64_t)num_sms() * SDFGB_JSP_MINB * kSpWarps;
    const StripPlan plan = strip_plan(ra, rb, nstrips, resident);
    const size_t smem = sp_smem(plan.hmax + 2 * F);
    static size_t attr = 0;
    if (smem > attr) {
        SDFGB_CUDA(cudaFuncSetAttribute(jacobi_strip_kernel<F, MIRROR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
        attr = smem;
    }
    CUtensorMap map;
    SDFGB_TRY(encode_tiled_2d(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, src, M, N, kSpRX, 3,
                              CU_TENSOR_MAP_SWIZZLE_NONE));
    static int per_sm = 0;
    static size_t per_sm_smem = 0;
    if (!per_sm || per_sm_smem != smem) {
        per_sm_smem = smem;
        SDFGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_strip_kernel<F, MIRROR>,
                                                                 kSpWarps * 32, smem));
        per_sm = std::max(per_sm, 1);
    }
    const int64_t nwarps = std::min<int64_t>(plan.total(), (int64_t)num_sms() * per_sm * kSpWarps);
    const unsigned blocks = (unsigned)((nwarps + kSpWarps - 1) / kSpWarps);
    const int slot = g_sp_launches.fetch_add(1) & (kSpSchedSlots - 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kSpWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = SDFGB_JSP_PDL;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    const float* dsrc = src;
    float* ddst = dst;
    const float* din = dst;
    int Mi = (int)M, Ni = (int)N, nw = (int)nwarps;
    SDFGB_CUDA(cudaLaunchKernelEx(&cfg, jacobi_strip_kernel<F, MIRROR>, map, dsrc, din, ddst, Mi, Ni, plan, nw, slot,
                                  coef, moff, mr0, mr1));
    SDFGB_LAUNCHED("jacobi_strip_kernel");
    return SDFGB_OK;
}

bool use_strip() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("SDFGB_J_KERNEL");
        v = !(e && e[0] == 't');  // SDFGB_J_KERNEL=tile selects jacobi_tb_kernel
    }
    return v;
}

template <int KT>
int launch_tb(const float* src_plane, float* dst, int64_t M, int64_t N, float coef, cudaStream_t s) {
    // the strip kernel needs >= 2 strips (each holds at most one border column)
    if (use_strip() && N > kSpX + kSpPad + 4) return launch_strip<KT>(src_plane, dst, M, N, 0, M, coef, s);
    static bool attr = false;
    if (!attr) {
        SDFGB_CUDA(cudaFuncSetAttribute(jacobi_tb_kernel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)tb_smem(KT)));
        attr = true;
    }
    CUtensorMap map;
    SDFGB_TRY(encode_tiled_2d(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, src_plane, M, N, kTbRX, tb_rows(KT),
                              CU_TENSOR_MAP_SWIZZLE_NONE));
    dim3 grid((unsigned)((N + kTbX - 1) / kTbX), (unsigned)((M + kTbY - 1) / kTbY));
    jacobi_tb_kernel<KT><<<grid, kTbThreads, tb_smem(KT), s>>>(map, dst, dst, (int)M, (int)N, coef, KT);
    SDFGB_LAUNCHED("jacobi_tb_kernel");
    return SDFGB_OK;
}

int launch_block(const float* src, float* dst, int64_t M, int64_t N, int64_t k, float coef, const Terms& terms,
                 cudaStream_t s) {
    if (k == 7) return launch_tb<7>(src, dst, M, N, coef, s);
    if (k == 5) return launch_tb<5>(src, dst, M, N, coef, s);
    if (k == 3) return launch_tb<3>(src, dst, M, N, coef, s);
    if (k == 1) return launch_step<float>(src, dst, N, M, 0, 1, M - 1, coef, terms, true, s);
    return set_error(SDFGB_ERR_INVALID, "jacobi2d block: k must be 1, 3, 5 or 7 (got %lld)", (long long)k);
}

// T steps on A[2, M, N] in fp32 with temporal blocking.  Launches advance an
// odd number of steps each (so state s stays in plane s % 2, as in the
// reference), and the last step is a one-step launch so the other plane ends
// holding state T-1 exactly like A[(T+1) % 2] of the reference.
int jacobi_f32_blocked(float* A, int64_t M, int64_t N, int64_t T_, float coef, const Terms& terms,
                       cudaStream_t s) {
    float* P[2] = {A, A + M * N};
    int64_t t = 0;
    while (T_ - t > 1) {
        int64_t k = std::min<int64_t>(7, T_ - 1 - t);
        if ((k & 1) == 0) k -= 1;
        const int p = (int)(t & 1);
        SDFGB_TRY(launch_block(P[p], P[p ^ 1], M, N, k, coef, terms, s));
        t += k;
    }
    const int p = (int)(t & 1);
    return launch_block(P[p], P[p ^ 1], M, N, 1, coef, terms, s);
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
    if constexpr (sizeof(T) == 4) {
        // temporal blocking needs 16 B rows (TMA) and enough steps to pay off
        if (canon && (N % 4) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 && T_ >= 4 && N >= 16)
            return jacobi_f32_blocked(reinterpret_cast<float*>(A), N, N, T_, (float)coef, terms, s);
    }
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

extern "C" int sdfgb_jacobi2d_rect_f32(float* A, int64_t M, int64_t N, int64_t T, double coef, const int32_t* di,
                                       const int32_t* dj, int nterms, void* stream) {
    sdfgb::Terms terms;
    bool canon;
    if (M < 0 || N < 0 || T < 0 || ((M > 0 && N > 0) && !A) || !sdfgb::parse_terms(di, dj, nterms, terms, canon))
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_rect: bad arguments");
    if (M < 3 || N < 3 || T == 0) return SDFGB_OK;
    cudaStream_t s = sdfgb::as_stream(stream);
    if (canon && (N % 4) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 && T >= 4 && N >= 16 && M >= 16)
        return sdfgb::jacobi_f32_blocked(A, M, N, T, (float)coef, terms, s);
    float* P[2] = {A, A + M * N};
    for (int64_t t = 0; t < T; ++t)
        SDFGB_TRY(sdfgb::launch_step<float>(P[t & 1], P[(t + 1) & 1], N, M, 0, 1, M - 1, (float)coef, terms, canon,
                                            s));
    return SDFGB_OK;
}
extern "C" int sdfgb_jacobi2d_block_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k, double coef,
                                        void* stream) {
    if (M < 3 || N < 16 || (N % 4) != 0 || !src || !dst || (reinterpret_cast<uintptr_t>(src) & 15) != 0 ||
        (reinterpret_cast<uintptr_t>(dst) & 15) != 0 || (k > 1 && M < 16))
        return sdfgb::set_error(SDFGB_ERR_INVALID,
                                "jacobi2d_block: needs M >= 16, N >= 16, N %% 4 == 0 and 16 B aligned planes");
    sdfgb::Terms terms;
    bool canon;
    const int32_t di[5] = {0, -1, 1, 0, 0}, dj[5] = {0, 0, 0, -1, 1};
    sdfgb::parse_terms(di, dj, 5, terms, canon);
    return sdfgb::launch_block(src, dst, M, N, k, (float)coef, terms, sdfgb::as_stream(stream));
}

// Output rows [r0, r1) only (clipped to the interior [1, M-2]) of one k-step
// launch src (state t) -> dst (state t+k): the multi-GPU slab runner
// computes its edge bands first, sends them, and overlaps the exchange with
// the interior band.  k > 1 needs the strip kernel (N >= 128).
extern "C" int sdfgb_jacobi2d_band_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k, int64_t r0,
                                       int64_t r1, double coef, void* stream) {
    if (M < 16 || N < 16 || (N % 4) != 0 || !src || !dst || (reinterpret_cast<uintptr_t>(src) & 15) != 0 ||
        (reinterpret_cast<uintptr_t>(dst) & 15) != 0 || r0 < 0 || r1 > M || r0 > r1)
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band: bad arguments");
    r0 = std::max<int64_t>(r0, 1);
    r1 = std::min<int64_t>(r1, M - 1);
    if (r1 <= r0) return SDFGB_OK;
    cudaStream_t s = sdfgb::as_stream(stream);
    if (k == 1) {
        sdfgb::Terms terms;
        bool canon;
        const int32_t di[5] = {0, -1, 1, 0, 0}, dj[5] = {0, 0, 0, -1, 1};
        sdfgb::parse_terms(di, dj, 5, terms, canon);
        return sdfgb::launch_step<float>(src, dst, N, M, 0, r0, r1, (float)coef, terms, true, s);
    }
    if (!sdfgb::strip_ok(N))
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band: k > 1 bands need N >= 128 (strip kernel)");
    if (r1 - r0 < 8)  // a strip tile needs >= 8 rows (its prologue never meets plane row M-1)
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band: k > 1 bands are at least 8 interior rows");
    if (k == 7) return sdfgb::launch_strip<7>(src, dst, M, N, r0, r1, (float)coef, s);
    if (k == 5) return sdfgb::launch_strip<5>(src, dst, M, N, r0, r1, (float)coef, s);
    if (k == 3) return sdfgb::launch_strip<3>(src, dst, M, N, r0, r1, (float)coef, s);
    return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band: k must be 1, 3, 5 or 7 (got %lld)", (long long)k);
}

// The band, with its output rows r in [m0, m1) also stored at
// mirror + (r - m0) * N (a neighbour's ghost rows in peer memory): compute
// and ghost transfer in one kernel.  k == 1 runs the one-step kernel and
// then copies those rows.
extern "C" int sdfgb_jacobi2d_band_mirror_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k,
                                              int64_t r0, int64_t r1, double coef, float* mirror, int64_t m0,
                                              int64_t m1, void* stream) {
    if (!mirror || m0 > m1) return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band_mirror: bad mirror");
    if (k == 1) {
        SDFGB_TRY(sdfgb_jacobi2d_band_f32(src, dst, M, N, 1, r0, r1, coef, stream));
        const int64_t a = std::max<int64_t>({r0, m0, 1}), b = std::min<int64_t>({r1, m1, M - 1});
        if (b <= a) return SDFGB_OK;
        return sdfgb::check_cuda(cudaMemcpyAsync(mirror + (a - m0) * N, dst + a * N, (size_t)((b - a) * N) * 4,
                                                 cudaMemcpyDeviceToDevice, sdfgb::as_stream(stream)),
                                 "jacobi2d_band_mirror copy");
    }
    if (M < 16 || N < 16 || (N % 4) != 0 || !src || !dst || (reinterpret_cast<uintptr_t>(src) & 15) != 0 ||
        (reinterpret_cast<uintptr_t>(dst) & 15) != 0 || (reinterpret_cast<uintptr_t>(mirror) & 15) != 0 ||
        r0 < 0 || r1 > M || r0 > r1)
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band_mirror: bad arguments");
    const int64_t moff = (int64_t)(mirror - (dst + m0 * N));  // elements from a dst row to its mirror
    r0 = std::max<int64_t>(r0, 1);
    r1 = std::min<int64_t>(r1, M - 1);
    if (r1 <= r0) return SDFGB_OK;
    cudaStream_t s = sdfgb::as_stream(stream);
    if (!sdfgb::strip_ok(N))
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band_mirror: k > 1 bands need N >= 128 (strip kernel)");
    if (r1 - r0 < 8)
        return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band_mirror: k > 1 bands are at least 8 interior rows");
    const int a = (int)std::max<int64_t>(m0, 0), b = (int)std::min<int64_t>(m1, M);
    if (k == 7) return sdfgb::launch_strip<7, true>(src, dst, M, N, r0, r1, (float)coef, s, moff, a, b);
    if (k == 5) return sdfgb::launch_strip<5, true>(src, dst, M, N, r0, r1, (float)coef, s, moff, a, b);
    if (k == 3) return sdfgb::launch_strip<3, true>(src, dst, M, N, r0, r1, (float)coef, s, moff, a, b);
    return sdfgb::set_error(SDFGB_ERR_INVALID, "jacobi2d_band_mirror: k must be 1, 3, 5 or 7 (got %lld)", (long long)k);
}

#if SDFGB_JSP_TIMING
extern "C" int sdfgb_debug_strip_timing(uint64_t* host, int64_t n) {
    return sdfgb::check_cuda(cudaMemcpyFromSymbol(host, sdfgb::g_sp_timing, (size_t)n * 32), "timing");
}
#endif

// The tile queue of one strip-kernel launch over output rows [r0, r1) of an
// M x N plane with `resident` persistent warps: tiles[3 t + {0,1,2}] =
// (strip, y0, ye) of queue entry t, for up to max_tiles entries.  Returns
// the number of entries (host only: the CPU tests check that the queue
// covers every strip's rows exactly once, in tiles of >= 16 rows).
extern "C" int64_t sdfgb_debug_strip_tiles(int64_t M, int64_t N, int64_t r0, int64_t r1, int64_t resident,
                                           int32_t* tiles, int64_t max_tiles) {
    (void)M;
    const int64_t nstrips = (N + sdfgb::kSpX - 1) / sdfgb::kSpX;
    const sdfgb::StripPlan plan = sdfgb::strip_plan(r0, r1, nstrips, resident);
    const int total = plan.total();
    for (int t = 0; t < total && t < max_tiles; ++t) plan.tile(t, tiles[3 * t], tiles[3 * t + 1], tiles[3 * t + 2]);
    return total;
}
