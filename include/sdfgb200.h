/*
 * sdfgb200.h -- C ABI of libsdfgb200.so, the B200 (sm_100a) execution backend
 * for SDFG Map scopes with write-conflict resolution (WCR) and stream memlets.
 *
 * The reference (arXiv 1902.10345 SDFG toolkit, /root/reference/pkg) has no
 * native library: its CPU dispatcher EMITS one C function per graph,
 *     void <sdfg.name>(T* container..., int64_t symbol...)      codegen.py:839-846
 * with containers = non-transient arrays in Sdfg.data order and symbols in
 * Sdfg.symbols order (codegen.py:620-627), compiles it with cc -shared
 * (codegen.py:890-913) and binds it through ctypes in CompiledSdfg.run
 * (codegen.py:866-887).  This library is what that ctypes binding calls
 * instead when an SDFG state was matched by GPUTransformMap:
 *
 *   1. host entries  (sdfgb_host_*): the drop-in for CompiledSdfg._fn --
 *      host pointers in the reference's own types (double*, int64_t*),
 *      synchronous, containers in the reference's argument order.
 *   2. device entries (sdfgb_*): device pointers, asynchronous on a CUDA
 *      stream passed as void* -- the timed path and the multi-GPU building
 *      block (one process per GPU; collectives live above this ABI).
 *
 * Conventions
 *   - Every entry returns SDFGB_OK (0) or an error code; the message is in
 *     sdfgb_last_error() (thread-local).  The reference's entry returns void
 *     and reports failures as Python exceptions (CodegenError, ToolchainError,
 *     interpreter OutOfBoundsError, interpreter.py:56-57,265-268); the Python
 *     layer maps these codes onto exceptions with the same names.
 *   - WCR targets ACCUMULATE into existing contents, exactly like the
 *     reference (hist_out = hist_in + counts, gallery.py:374-377;
 *     count += n; b += A x).  Nothing is zeroed implicitly.
 *   - Precision: *_f32 entries compute in fp32 (BASELINE.json configs);
 *     *_f64 / *_i64 entries compute in the reference's own basetypes
 *     (ir.py:33-35).
 *   - No entry falls back to the CPU.  Without a usable CUDA device every
 *     entry fails with SDFGB_ERR_CUDA.
 */
#ifndef SDFGB200_H
#define SDFGB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDFGB_ABI_VERSION 1

#define SDFGB_OK 0
#define SDFGB_ERR_INVALID 1     /* bad argument / unsupported shape        */
#define SDFGB_ERR_CUDA 2        /* CUDA runtime / launch failure            */
#define SDFGB_ERR_OOB 3         /* out-of-bounds WCR index (OutOfBoundsError) */
#define SDFGB_ERR_WORKSPACE 4   /* workspace too small                       */
#define SDFGB_ERR_COMM 5        /* NCCL missing or a collective failed        */

/* comparison operators of a stream-push predicate (tasklets.py _CMPOPS) */
#define SDFGB_CMP_LT 0
#define SDFGB_CMP_LE 1
#define SDFGB_CMP_GT 2
#define SDFGB_CMP_GE 3
#define SDFGB_CMP_EQ 4
#define SDFGB_CMP_NE 5

/* ---------------------------------------------------------------- misc */
int sdfgb_abi_version(void);
const char* sdfgb_last_error(void);
int sdfgb_device_count(int* count);
/* Pinned host memory for zero-staging H2D/D2H in the host entries. */
int sdfgb_host_alloc(void** ptr, size_t bytes);
int sdfgb_host_free(void* ptr);
/* Status of the last host entry (sdfgb_host_*) called on this thread: the
 * per-graph shims keep the reference's `void <name>(...)` signature
 * (codegen.py:839-846), so their callers read the status here afterwards. */
int sdfgb_last_status(void);
/* Host threads the host entries convert and stage with (SDFGB_HOST_THREADS,
 * default: all hardware threads). */
int sdfgb_host_threads(void);
/* The host entries' staging conversions (no device needed; CPU tests):
 * kind 0 f64->f32 round to nearest, 1 f64->f32 toward -inf, 2 f64->f32
 * returning 1 iff every element round-trips, 3 f32->f64, 4 int64->int32
 * returning the count outside [lo, hi), 5 returns 1 iff int64 src is
 * non-decreasing (dst unused). */
int64_t sdfgb_host_convert(int kind, const void* src, void* dst, int64_t n, int64_t lo, int64_t hi);

/* ------------------------------------------------------ device entries */

/* Histogram, WCR sum with a dynamic subscript (tasklets.py:297-300 ->
 * interpreter.py:262-278; codegen.py:733-747).  For each element v:
 *     k = floor((double)v * scale / div)          (f32/f64;  bi = v*S//D)
 *     k = v                                       (i64;      h[v] = 1)
 *     hist[k] += 1         for 0 <= k < bins, else *oob += 1 (not counted)
 * hist is int64 device memory (the reference container type). */
int sdfgb_hist_f32(const float* img, int64_t n, double scale, double div,
                   int64_t* hist, int64_t bins, uint64_t* oob, void* stream);
int sdfgb_hist_f64(const double* img, int64_t n, double scale, double div,
                   int64_t* hist, int64_t bins, uint64_t* oob, void* stream);
int sdfgb_hist_i64(const int64_t* img, int64_t n,
                   int64_t* hist, int64_t bins, uint64_t* oob, void* stream);

/* Query = predicated stream push + drain (codegen.py:462-471, :363-376;
 * interpreter.py:346-365, :447-481).  out_vals[0:k) = {v : v OP thr};
 * out_vals[k:] untouched; count[0] += k.  thr is read on the host side.
 * By default the survivors' ORDER is unspecified (a Map's iterations push
 * concurrently into the stream): a single-pass reservation
 * kernel.  OR SDFGB_QUERY_ORDERED into op for input order (the CPU FIFO
 * order of the generated C code) at the cost of a second, L2-resident pass.
 * ws must hold sdfgb_query_workspace_bytes(n) bytes, zeroed ONCE before
 * its first use (it resets itself afterwards). */
#define SDFGB_QUERY_ORDERED 0x100
size_t sdfgb_query_workspace_bytes(int64_t n, int elem_bytes);
int sdfgb_query_f32(const float* col, int64_t n, int op, double thr,
                    float* out_vals, int64_t* count,
                    void* ws, size_t ws_bytes, void* stream);
int sdfgb_query_f64(const double* col, int64_t n, int op, double thr,
                    double* out_vals, int64_t* count,
                    void* ws, size_t ws_bytes, void* stream);

/* CSR SpMV: data-dependent inner map over [rowptr[i], rowptr[i+1]) with the
 * indirection x[col[j]] and WCR sum into b[i] (gallery.py:152-213):
 *     b[i] += sum_j val[j] * x[col[j]]               i in [0, H) */
/* Measurement probe (not a motif): SpMV's memory pattern without its rows --
 * col/val (nnz % 4 == 0, 16 B aligned) streamed, x[col[j]] gathered, products
 * summed into *sink.  bench.py times it on the SpMV's own arrays: the live
 * L2-gather ceiling the SpMV kernel is measured against. */
int sdfgb_probe_gather_f32(const float* x, const int32_t* col, const float* val, int64_t nnz,
                           float* sink, void* stream);
int sdfgb_spmv_csr_f32(const int32_t* rowptr, const int32_t* col, const float* val,
                       const float* x, float* b, int64_t H, void* stream);
int sdfgb_spmv_csr_f64(const int64_t* rowptr, const int64_t* col, const double* val,
                       const double* x, double* b, int64_t H, void* stream);

/* 2-D Jacobi time loop (loops.py:31-61 guard loop around a stencil map):
 *     for t in [0, T): A[(t+1)%2, i, j] = coef * (((A[t%2, i+di0, j+dj0]
 *                         + A[t%2, i+di1, j+dj1]) + ...)      i, j in [1, N-2]
 * A is [2, N, N] row-major; borders are never written.  The nterms offsets
 * (|di|,|dj| <= 1, nterms <= 9) fix the summation order of the tasklet. */
int sdfgb_jacobi2d_f32(float* A, int64_t N, int64_t T, double coef,
                       const int32_t* di, const int32_t* dj, int nterms, void* stream);
int sdfgb_jacobi2d_f64(double* A, int64_t N, int64_t T, double coef,
                       const int32_t* di, const int32_t* dj, int nterms, void* stream);
/* One row-block of one step (multi-GPU building block): rows [r0, r1) of the
 * destination plane, reading src and writing dst (both [rows, N] planes whose
 * row 0 is global row g0). */
int sdfgb_jacobi2d_step_f32(const float* src, float* dst, int64_t N, int64_t rows,
                            int64_t g0, int64_t r0, int64_t r1, double coef,
                            const int32_t* di, const int32_t* dj, int nterms, void* stream);

/* The same time loop on rectangular planes A[2, M, N] (fp32): the border is
 * the plane's edge.  The multi-GPU slab decomposition puts ghost rows at the
 * slab edges and global rows 0 / Ng-1 at the first / last rank's edge. */
int sdfgb_jacobi2d_rect_f32(float* A, int64_t M, int64_t N, int64_t T, double coef,
                            const int32_t* di, const int32_t* dj, int nterms, void* stream);
/* One temporal-blocking launch (canonical 5-point order): k in {1, 3, 5, 7}
 * steps from plane src (state t) to plane dst (state t+k), both [M, N],
 * N % 4 == 0, 16 B aligned.  Rows/columns within k of the plane edge are
 * halo: exact only where the edge is the true border. */
int sdfgb_jacobi2d_block_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k,
                             double coef, void* stream);
/* Rows [r0, r1) (clipped to the interior) of one k-step launch src -> dst:
 * the banded form of sdfgb_jacobi2d_block_f32 that lets a slab runner send
 * its edge bands while the interior band computes (multigpu.jacobi).  k > 1
 * needs N >= 128 and at least 8 interior rows. */
int sdfgb_jacobi2d_band_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k,
                            int64_t r0, int64_t r1, double coef, void* stream);
/* The same band, its output rows r in [m0, m1) also stored at
 * mirror + (r - m0) * N: a neighbour rank's ghost rows in peer memory
 * (NVLink), so an edge band and its ghost-row transfer are one kernel
 * (multigpu.jacobi with PeerJacobi).  k == 1 runs the one-step kernel and
 * then copies those rows. */
int sdfgb_jacobi2d_band_mirror_f32(const float* src, float* dst, int64_t M, int64_t N, int64_t k,
                                   int64_t r0, int64_t r1, double coef, float* mirror, int64_t m0,
                                   int64_t m1, void* stream);
/* Host-only introspection of the strip kernel's tile queue for output rows
 * [r0, r1) of an M x N plane and `resident` persistent warps: tiles[3t..3t+2]
 * = (strip, y0, ye) of entry t (at most max_tiles written); returns the
 * number of entries.  Used by the CPU tests. */
int64_t sdfgb_debug_strip_tiles(int64_t M, int64_t N, int64_t r0, int64_t r1, int64_t resident,
                                int32_t* tiles, int64_t max_tiles);

/* GEMM after MapReduceFusion (library.py:461-554): C = A(MxK) * B(KxN),
 * row-major fp32, fp32-accurate through 3xTF32 on tcgen05 tensor cores.
 * ws must hold sdfgb_gemm_workspace_bytes(M, N, K) bytes. */
size_t sdfgb_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);
int sdfgb_gemm_f32(const float* A, const float* B, float* C,
                   int64_t M, int64_t N, int64_t K,
                   void* ws, size_t ws_bytes, void* stream);
/* The same with flags.  SDFGB_GEMM_B_SPLIT: B's split operands are already in
 * ws from an earlier call with the same B (same K, N) -- row pieces of one
 * product (the multi-GPU A-piece pipeline) split B once.  B's part of the
 * workspace does not depend on M. */
#define SDFGB_GEMM_B_SPLIT 1
int sdfgb_gemm_f32_ex(const float* A, const float* B, float* C,
                      int64_t M, int64_t N, int64_t K,
                      void* ws, size_t ws_bytes, int flags, void* stream);
/* SIMT fp32 FFMA GEMM (k-sequential per element) used as the on-device
 * cross-check of the tensor-core path in tests. */
int sdfgb_gemm_f32_simt(const float* A, const float* B, float* C,
                        int64_t M, int64_t N, int64_t K, void* stream);
/* Native precision (float64): k-ordered IEEE multiply + add per element,
 * bit-identical to the reference's MapReduceFusion loop after init_C. */
int sdfgb_gemm_f64(const double* A, const double* B, double* C,
                   int64_t M, int64_t N, int64_t K, void* stream);

/* ------------------------------------------------- multi-GPU entries
 * One process per GPU: each call is this rank's share of a motif plus the
 * exchange step of SURVEY.md §8e, on the caller's NCCL communicator
 * (ncclComm_t as void*) and stream.  Results are bit-identical to the
 * one-GPU entries.  NCCL is loaded at run time (libnccl.so.2); without it
 * these return SDFGB_ERR_COMM.  Python counterpart: multigpu.py.        */
int sdfgb_nccl_available(void);
/* Kernels on the current device may access memory on device `peer` (the
 * P2P entries' peer mappings); already-enabled is success. */
int sdfgb_enable_peer_access(int peer);
/* Stream-ordered cross-rank flags for kernels that write peer memory:
 * signal stores `value` into `flag` (system-scope release) after all work
 * queued before it on the stream; wait holds the stream until `flag` (this
 * device's memory) reaches `value`.  Flags only grow. */
int sdfgb_flag_signal(int* flag, int value, void* stream);
int sdfgb_flag_wait(const int* flag, int value, void* stream);
int sdfgb_nccl_unique_id(void* id_out /* 128 bytes */);
int sdfgb_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank);
int sdfgb_nccl_comm_destroy(void* comm);
/* hist += counts of the union of all ranks' shards (every rank ends with the
 * same hist and oob): local partial -> ncclAllReduce(sum) -> fold. */
size_t sdfgb_hist_mgpu_workspace_bytes(int64_t bins);
int sdfgb_hist_f32_mgpu(const float* img, int64_t n, double scale, double div,
                        int64_t* hist, int64_t bins, uint64_t* oob,
                        void* ws, size_t ws_bytes, void* comm, void* stream);
/* The same histogram with the all-reduce fused into the kernel: this rank's
 * counts are added (system-scope atomics, over NVLink) straight into the hist
 * and oob of every one of the npeers <= 8 ranks, given as device pointers
 * mapped into this process (CUDA IPC).  After every rank's call has
 * completed (the caller's barrier), each hist holds hist_in + all counts.
 * No collective, no workspace; bins <= 12287. */
int sdfgb_hist_f32_p2p(const float* img, int64_t n, double scale, double div,
                       int64_t* const* peer_hist, uint64_t* const* peer_oob, int npeers,
                       int64_t bins, void* stream);
/* The gathered multi-GPU query with the gather fused into the compaction:
 * this rank's survivors are stored over NVLink straight into the gathering
 * rank's out_root, at slots reserved with system-scope atomics on its
 * int64 counter reserve_root (both mapped into this process, CUDA IPC).
 * After every rank's call has completed (the caller's barrier),
 * out_root[0:*reserve_root) holds all survivors in unspecified order (a
 * stream's push order); the caller adds *reserve_root to count
 * and re-zeroes it.  col 16-byte aligned; ws as for sdfgb_query_f32. */
int sdfgb_query_f32_p2p(const float* col, int64_t n, int op, double thr, float* out_root,
                        int64_t* reserve_root, void* ws, size_t ws_bytes, void* stream);
/* Sharded query: this rank's survivors -> out_vals[0:k); counts[world]
 * (device) receives every rank's k by ncclAllGather; count[0] += total and
 * offset[0] = this rank's global output offset (survivors on lower ranks). */
int sdfgb_query_f32_mgpu(const float* col, int64_t n, int op, double thr, float* out_vals,
                         int64_t* count, int64_t* offset, int64_t* counts,
                         void* ws, size_t ws_bytes, void* comm, void* stream);
/* Row-block SpMV: ncclAllGather of the equal x shards (w_shard each) into
 * x_full, then b[i] += ... over this rank's H_local rows (col holds global
 * column ids). */
int sdfgb_spmv_csr_f32_mgpu(const int32_t* rowptr, const int32_t* col, const float* val,
                            const float* x_shard, int64_t w_shard, float* x_full, float* b,
                            int64_t H_local, void* comm, void* stream);
/* Jacobi on a row slab A[2, top + rows + bot, N] (N % 4 == 0): top / bot are
 * 7 ghost rows towards each neighbour (0 at the global edge, whose plane edge
 * is the true border).  One grouped ncclSend/ncclRecv of ghost rows per
 * temporal block of up to 7 steps, issued on an internal side stream once the
 * edge bands are computed and overlapped with the interior band (N >= 128,
 * rows >= 48); canonical 5-point order. */
int sdfgb_jacobi2d_f32_mgpu(float* A, int64_t top, int64_t rows, int64_t bot, int64_t N, int64_t T,
                            double coef, void* comm, void* stream);
/* P x Q grid GEMM: C block (i, j) = A row panel i x B column panel j.  A_piece
 * (a_rows x K) is this rank's share of panel i, gathered over row_comm (size
 * Q) into A_panel (a_rows*Q x K); B_piece (b_rows x nq) its share of panel j,
 * gathered over col_comm (size P, b_rows*P == K) into B_panel (K x nq).  The
 * A pieces are broadcast on an internal side stream and each piece's C rows
 * computed as soon as it lands (the exchange overlaps the MMA).
 * ws: sdfgb_gemm_workspace_bytes(a_rows*Q, nq, K). */
int sdfgb_gemm_f32_mgpu(const float* A_piece, int64_t a_rows, const float* B_piece, int64_t b_rows,
                        int64_t K, int64_t nq, float* A_panel, float* B_panel, float* C_block,
                        void* ws, size_t ws_bytes, void* row_comm, void* col_comm, void* stream);

/* -------------------------------------------------------- host entries
 * Drop-in for CompiledSdfg._fn(*ptrs, *syms) (codegen.py:886): host
 * buffers in the reference's types (pageable is fine); staged through a
 * pinned ring by host threads, kernel(s), copied back; synchronous.
 * precision: 0 = fp32 on device (BASELINE: inputs rounded to nearest fp32),
 * 1 = native (the reference's float64 / int64 results; histogram with
 * power-of-two binning and the query still ship 4 B per element where that
 * is lossless).  Each records its status for sdfgb_last_status().        */
#define SDFGB_PREC_FP32 0
#define SDFGB_PREC_NATIVE 1

/* void histogram(double* img, int64_t* hist, int64_t H, int64_t W) */
int sdfgb_host_histogram(const double* img, int64_t* hist, int64_t H, int64_t W,
                         int64_t bins, double scale, double div, int precision);
/* void histogram(int64_t* img, int64_t* hist, int64_t H, int64_t W, int64_t B)  gallery.py:354 */
int sdfgb_host_histogram_i64(const int64_t* img, int64_t* hist, int64_t H, int64_t W,
                             int64_t bins);
/* void query(double* col, double* thr, double* out_vals, int64_t* count, int64_t N) */
int sdfgb_host_query(const double* col, const double* thr, double* out_vals,
                     int64_t* count, int64_t N, int op, int precision);
/* void spmv(int64_t* A_row, int64_t* A_col, double* A_val, double* x, double* b,
 *           int64_t H, int64_t W, int64_t nnz) */
int sdfgb_host_spmv(const int64_t* A_row, const int64_t* A_col, const double* A_val,
                    const double* x, double* b, int64_t H, int64_t W, int64_t nnz,
                    int precision);
/* void jacobi2d(double* A, int64_t N, int64_t T) */
int sdfgb_host_jacobi2d(double* A, int64_t N, int64_t T, double coef,
                        const int32_t* di, const int32_t* dj, int nterms, int precision);
/* void matmul(double* A, double* B, double* C, int64_t M, int64_t N, int64_t K) */
int sdfgb_host_matmul(const double* A, const double* B, double* C,
                      int64_t M, int64_t N, int64_t K);
int sdfgb_host_matmul_f64(const double* A, const double* B, double* C,
                          int64_t M, int64_t N, int64_t K);

#ifdef __cplusplus
}
#endif
#endif /* SDFGB200_H */
