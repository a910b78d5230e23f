// hostpool.h -- host threads for the drop-in entries' staging.
//
// The reference's entry takes float64 / int64 host buffers
// (CompiledSdfg.run, codegen.py:875-887).  Shipping them as they are costs
// twice the PCIe bytes the fp32/int32 kernels read, and from pageable
// memory the driver's own staging runs at ~11 GB/s (tools/micro/host_narrow.cu,
// profiles/r2_host_narrow.txt).  Instead, host threads convert each chunk
// into a small pinned slot (L3-resident) that the copy engine drains while
// the threads convert the next one.  Conversions are either declared
// (fp32 precision rounds to nearest) or lossless by construction (rounding
// toward -inf for power-of-two binning; a round-trip check per chunk for
// the query), so native-precision results stay the reference's.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <functional>

namespace sdfgb {
namespace host {

// Run fn(task) for every task in [0, ntasks) on the pool's threads and the
// caller; returns when all tasks are done.  One job at a time per process.
void parallel_for(int64_t ntasks, const std::function<void(int64_t)>& fn);
int threads();

// dst[i] = (float)src[i], rounded to nearest (fp32 precision semantics)
void narrow_rn(const double* src, float* dst, int64_t n);
// dst[i] = largest float <= src[i] (floor-exact for power-of-two binning)
void narrow_rd(const double* src, float* dst, int64_t n);
// rounded to nearest; true iff every element round-trips exactly (NaN counts
// as inexact, so its chunk keeps the double path and its payload)
bool narrow_exact(const double* src, float* dst, int64_t n);
// dst[i] = (double)src[i]; streaming stores (the destination is the
// caller's cold buffer: no read-for-ownership)
void widen(const float* src, double* dst, int64_t n);
// parallel memcpy into the caller's cold buffer, streaming stores
void copy_out(void* dst, const void* src, size_t bytes);
// dst[i] = (int32_t)src[i]; returns how many elements lie outside [lo, hi)
int64_t narrow_index(const int64_t* src, int32_t* dst, int64_t n, int64_t lo, int64_t hi);
// true iff src[0..n) is non-decreasing
bool non_decreasing(const int64_t* src, int64_t n);
// parallel memcpy
void copy(void* dst, const void* src, size_t bytes);
// dst row r = src row r narrowed (rn) and padded with zeros to dcols columns
void narrow_rows_rn(const double* src, float* dst, int64_t rows, int64_t cols, int64_t dcols);

}  // namespace host
}  // namespace sdfgb
