/*
 * oracle.c -- CPU restatement of the reference's hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity checker for libsdfgb200.so.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product path never does.
 *
 * Each function restates one motif exactly as the reference executes it:
 * the interpreter (pkg/src/sdfg/interpreter.py) is the ground truth and the
 * reference's C dispatcher (pkg/src/sdfg/codegen.py) fixes loop order and
 * arithmetic order.  Double/int64 variants are the reference's own types
 * (ir.py:33-35); the float variants restate the same op order in fp32 so the
 * GPU's fp32 path can be compared bit-for-bit where the op order is kept.
 * Compiled with -ffp-contract=off so no FMA contraction changes rounding.
 *
 * Parity pin: tests/test_oracle.py checks every function against the
 * reference-interpreter fixtures in tests/golden/cases (make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---------------------------------------------------------------------
 * Histogram: map over [0:H-1, 0:W-1]; tasklet ``bi = v * S // D`` (int64
 * connector -> (int64_t)floor(...), tasklets.py:432-433, :480-481), then
 * subscript write ``h[k] = 1`` with WCR sum (codegen.py:733-747,
 * interpreter.py:262-278).  hist accumulates into existing contents.
 * Out-of-range index: the interpreter raises OutOfBoundsError
 * (interpreter.py:265-268); here we count the violations and skip.
 * ------------------------------------------------------------------- */
int64_t orc_histogram_f64(const double* img, int64_t n, int64_t* hist, int64_t bins,
                          double scale, double div)
{
    int64_t oob = 0;
    for (int64_t p = 0; p < n; ++p) {
        double q = floor((img[p] * scale) / div);
        if (!(q >= 0.0 && q < (double)bins)) { ++oob; continue; }
        hist[(int64_t)q] += 1;
    }
    return oob;
}

/* Integer-image variant: gallery.py:354-386, ``h[v] = 1``. */
int64_t orc_histogram_i64(const int64_t* img, int64_t n, int64_t* hist, int64_t bins)
{
    int64_t oob = 0;
    for (int64_t p = 0; p < n; ++p) {
        int64_t v = img[p];
        if (v < 0 || v >= bins) { ++oob; continue; }
        hist[v] += 1;
    }
    return oob;
}

/* fp32 input, binning computed in double like the reference (exact for the
 * fp32-representable inputs of SURVEY §8d). */
int64_t orc_histogram_f32(const float* img, int64_t n, int64_t* hist, int64_t bins,
                          double scale, double div)
{
    int64_t oob = 0;
    for (int64_t p = 0; p < n; ++p) {
        double q = floor(((double)img[p] * scale) / div);
        if (!(q >= 0.0 && q < (double)bins)) { ++oob; continue; }
        hist[(int64_t)q] += 1;
    }
    return oob;
}

/* ---------------------------------------------------------------------
 * Query: map over [0:N-1]; ``if v OP limit: sv = v; c = 1`` (gallery.py:314-315).
 * sv is pushed to stream S in map order (codegen.py:462-471), S is drained
 * FIFO into out_vals[0:n) after the map (codegen.py:363-376,
 * interpreter.py:447-481); out_vals[n:] untouched; count += n (WCR sum).
 * op: 0 '<', 1 '<=', 2 '>', 3 '>=', 4 '==', 5 '!='.
 * ------------------------------------------------------------------- */
static inline int orc_cmp(double v, int op, double t)
{
    switch (op) {
    case 0: return v < t;
    case 1: return v <= t;
    case 2: return v > t;
    case 3: return v >= t;
    case 4: return v == t;
    default: return v != t;
    }
}

int64_t orc_query_f64(const double* col, int64_t n, int op, double thr,
                      double* out_vals, int64_t* count)
{
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i)
        if (orc_cmp(col[i], op, thr)) out_vals[k++] = col[i];
    count[0] += k;
    return k;
}

int64_t orc_query_f32(const float* col, int64_t n, int op, double thr,
                      float* out_vals, int64_t* count)
{
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i)
        if (orc_cmp((double)col[i], op, thr)) out_vals[k++] = col[i];
    count[0] += k;
    return k;
}

/* ---------------------------------------------------------------------
 * CSR SpMV: outer map i in [0:H-1], inner map j in [row_b:row_e-1] with the
 * data-dependent range connectors (gallery.py:171-176, codegen.py:503-508),
 * x[A_col[j]] through the indirection tasklet (ir.py:608-639),
 * ``out = a * in_x`` and WCR sum into b[i] (gallery.py:184-189).  j runs
 * sequentially, so b[i] accumulates left to right onto its prior value.
 * ------------------------------------------------------------------- */
void orc_spmv_f64(const int64_t* rowptr, const int64_t* col, const double* val,
                  const double* x, double* b, int64_t H)
{
    for (int64_t i = 0; i < H; ++i)
        for (int64_t j = rowptr[i]; j <= rowptr[i + 1] - 1; ++j)
            b[i] += val[j] * x[col[j]];
}

void orc_spmv_f32(const int32_t* rowptr, const int32_t* col, const float* val,
                  const float* x, float* b, int64_t H)
{
    for (int64_t i = 0; i < H; ++i)
        for (int64_t j = rowptr[i]; j <= (int64_t)rowptr[i + 1] - 1; ++j)
            b[i] += val[j] * x[col[j]];
}

/* ---------------------------------------------------------------------
 * Jacobi-2D: guard loop ``for (t = 0; t < T; t = t + 1)`` (loops.py:31-61,
 * codegen.py:688-699) around a map over the interior [1:N-2]^2 reading
 * A[t%2, i+di_k, j+dj_k] and writing A[(t+1)%2, i, j]; borders are never
 * written.  The tasklet is ``o = coef * (t0 + t1 + ... )`` which the
 * reference evaluates left to right: coef * ((((t0 + t1) + t2) + t3) + t4)
 * (tasklets.py:430-444).  ``di/dj`` give the term order.
 * ------------------------------------------------------------------- */
#define JACOBI_ORACLE(NAME, T)                                                        \
void NAME(T* A, int64_t N, int64_t TT, T coef, const int32_t* di, const int32_t* dj,    \
          int32_t nterms)                                                               \
{                                                                                       \
    int64_t off[9];                                                                     \
    for (int32_t k = 0; k < nterms && k < 9; ++k) off[k] = (int64_t)di[k] * N + dj[k];  \
    for (int64_t t = 0; t < TT; ++t) {                                                  \
        const T* src = A + (t % 2) * N * N;                                             \
        T* dst = A + ((t + 1) % 2) * N * N;                                             \
        /* rows are independent within a step: threads change no rounding */          \
        _Pragma("omp parallel for schedule(static) if (N > 256)")                       \
        for (int64_t i = 1; i <= N - 2; ++i) {                                          \
            const T* r = src + i * N;                                                   \
            T* d = dst + i * N;                                                         \
            if (nterms == 5) {  /* same left-to-right order, unrolled */               \
                const int64_t o0 = off[0], o1 = off[1], o2 = off[2], o3 = off[3],      \
                              o4 = off[4];                                              \
                for (int64_t j = 1; j <= N - 2; ++j)                                    \
                    d[j] = coef * ((((r[j + o0] + r[j + o1]) + r[j + o2])               \
                                    + r[j + o3]) + r[j + o4]);                          \
            } else {                                                                    \
                for (int64_t j = 1; j <= N - 2; ++j) {                                  \
                    T s = r[j + off[0]];                                                \
                    for (int32_t k = 1; k < nterms; ++k) s = s + r[j + off[k]];        \
                    d[j] = coef * s;                                                    \
                }                                                                       \
            }                                                                           \
        }                                                                               \
    }                                                                                   \
}

JACOBI_ORACLE(orc_jacobi2d_f64, double)
JACOBI_ORACLE(orc_jacobi2d_f32, float)

/* ---------------------------------------------------------------------
 * Matrix multiplication after MapReduceFusion (library.py:461-554): an
 * init state writes C = 0 (the sum identity, ir.py:91-96), then the fused
 * map accumulates C[i,j] += A[i,k] * B[k,j] with k ascending for every
 * (i, j) (codegen.py:500-524 loop nest; tiling keeps the per-element order).
 * Rows [r0, r1) only, so a row sample of a huge GEMM can be checked.
 * ------------------------------------------------------------------- */
void orc_matmul_f64(const double* A, const double* B, double* C,
                    int64_t M, int64_t N, int64_t K, int64_t r0, int64_t r1)
{
    (void)M;
    /* rows are independent: threads change no rounding */
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = r0; i < r1; ++i) {
        double* c = C + i * N;
        for (int64_t j = 0; j < N; ++j) c[j] = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            double a = A[i * K + k];
            const double* b = B + k * N;
            for (int64_t j = 0; j < N; ++j) c[j] += a * b[j];
        }
    }
}

/* fp32 inputs, double accumulation (a float64 reference on fp32 data). */
void orc_matmul_f32in_f64acc(const float* A, const float* B, double* C,
                             int64_t M, int64_t N, int64_t K, int64_t r0, int64_t r1)
{
    (void)M;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = r0; i < r1; ++i) {
        double* c = C + (i - r0) * N;
        for (int64_t j = 0; j < N; ++j) c[j] = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            double a = (double)A[i * K + k];
            const float* b = B + k * N;
            for (int64_t j = 0; j < N; ++j) c[j] += a * (double)b[j];
        }
    }
}
