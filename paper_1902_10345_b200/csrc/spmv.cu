// spmv.cu -- K3: CSR SpMV, the spmv motif (gallery.py:152-213):
//   map i in [0:H-1]:
//     map j in [row_b:row_e-1]   (data-dependent range, A_row[i], A_row[i+1])
//       x_val = x[A_col[j]]       (indirection tasklet, ir.py:608-639)
//       b[i] (+)= A_val[j] * x_val   (WCR sum, accumulates onto b_in)
//
// B200 design: warp per row.  Lanes stream the row's col/val coalesced
// (the matrix is 8 B/nnz of HBM traffic, read once), gather x through
// L1/L2 (x is 16 MB at the BASELINE shape -> L2-resident), reduce with
// shuffles, lane 0 commits b[i] += sum.  Two rows per warp iteration keep
// more independent gathers in flight.  The per-row summation is a lane
// tree rather than the reference's left-to-right j order, so results agree
// to rounding (1e-5 rel for fp32).
#include <algorithm>

#include "common.cuh"

namespace sdfgb {
namespace {

constexpr int kSpmvBlock = 256;
#ifndef SDFGB_SPMV_PF
#define SDFGB_SPMV_PF 1  // next row bounds and this row's b loaded a row ahead (1.094 -> 1.086 ms at S1)
#endif

template <typename I, typename T>
__global__ void __launch_bounds__(kSpmvBlock)
spmv_warp_row_kernel(const I* __restrict__ rowptr, const I* __restrict__ col,
                     const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ b,
                     int64_t H) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kSpmvBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kSpmvBlock) >> 5;
    for (int64_t r0 = warp * 2; r0 < H; r0 += nwarps * 2) {
        const int64_t r1 = r0 + 1;
        const int64_t b0 = rowptr[r0], e0 = rowptr[r0 + 1];
        const int64_t b1 = r1 < H ? (int64_t)rowptr[r1] : 0;
        const int64_t e1 = r1 < H ? (int64_t)rowptr[r1 + 1] : 0;
        T s0 = T(0), s1 = T(0);
        const int64_t l0 = e0 - b0, l1 = e1 - b1;
        const int64_t lmax = l0 > l1 ? l0 : l1;
        for (int64_t o = lane; o < lmax; o += 32) {
            if (o < l0) {
                const int64_t j = b0 + o;
                s0 += __ldg(val + j) * __ldg(x + __ldg(col + j));
            }
            if (o < l1) {
                const int64_t j = b1 + o;
                s1 += __ldg(val + j) * __ldg(x + __ldg(col + j));
            }
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, d);
            s1 += __shfl_xor_sync(0xffffffffu, s1, d);
        }
        if (lane == 0) {
            b[r0] += s0;
            if (r1 < H) b[r1] += s1;
        }
    }
}

// L2 policies: the 2 GB matrix streams through with evict_first so it cannot
// push the 16 MB x vector out of L2; x gathers carry evict_last.  (Without the
// split, a no_allocate x gather measured 11 GB of DRAM reads -- x fell out.)
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// read-only loads: not volatile, so the scheduler may hoist the next row's
// col/val streams above the current row's gathers
#ifndef SDFGB_SPMV_VOL
#define SPMV_ASM asm
#else
#define SPMV_ASM asm volatile
#endif
__device__ __forceinline__ float ldg_keep(const float* p, uint64_t pol) {
    float r;
    // random 4 B gathers: allocating their lines in L1 only evicts the
    // rowptr / b lines (no reuse across 4 M columns); 1112 -> 1094 us
    SPMV_ASM("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int4 ldg_stream_i4(const int32_t* p, uint64_t pol) {
    int4 r;
    SPMV_ASM("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
             : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ float4 ldg_stream_f4(const float* p, uint64_t pol) {
    float4 r;
    SPMV_ASM("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
             : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
    return r;
}

// fp32/int32 path: half-warp per row, 4 consecutive nnz per lane through
// 128-bit col/val loads (one LDG.128 pair covers 64 nnz per half-warp);
// matrix streams evict_first, x gathers evict_last.
__global__ void __launch_bounds__(kSpmvBlock)
spmv_hw_vec4_kernel(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                    const float* __restrict__ val, const float* __restrict__ x, float* __restrict__ b,
                    int64_t H) {
    const int lane = threadIdx.x & 31, hl = lane & 15;
    const unsigned hmask = (lane < 16) ? 0x0000ffffu : 0xffff0000u;
    const int64_t hw = (((int64_t)blockIdx.x * kSpmvBlock + threadIdx.x) >> 4);
    const int64_t nhw = ((int64_t)gridDim.x * kSpmvBlock) >> 4;
    const uint64_t pstream = policy_evict_first(), pkeep = policy_evict_last();
    auto ldg_na = [&](const float* p) { return ldg_keep(p, pkeep); };
#if SDFGB_SPMV_PF
    // the next row's bounds and this row's b are loaded a row ahead, so a
    // row's chain is col/val -> gathers only (not rowptr -> col/val ->
    // gathers -> b)
    int64_t rbn = hw < H ? (int64_t)rowptr[hw] : 0, ren = hw < H ? (int64_t)rowptr[hw + 1] : 0;
    for (int64_t r = hw; r < H; r += nhw) {
        const int64_t rb = rbn, re = ren;
        const float bold = hl == 0 ? b[r] : 0.f;
        if (r + nhw < H) {
            rbn = rowptr[r + nhw];
            ren = rowptr[r + nhw + 1];
        }
        float s = 0.f;
#else
    for (int64_t r = hw; r < H; r += nhw) {
        const int64_t rb = rowptr[r], re = rowptr[r + 1];
        float s = 0.f;
#endif
        if ((rb & 3) == 0) {
            for (int64_t j = rb + 4 * hl; j < re; j += 64) {
                if (j + 3 < re) {
                    const int4 c = ldg_stream_i4(col + j, pstream);
                    const float4 v = ldg_stream_f4(val + j, pstream);
                    const float x0 = ldg_na(x + c.x), x1 = ldg_na(x + c.y);
                    const float x2 = ldg_na(x + c.z), x3 = ldg_na(x + c.w);
                    s += v.x * x0;
                    s += v.y * x1;
                    s += v.z * x2;
                    s += v.w * x3;
                } else {
                    for (int64_t q = j; q < re; ++q) s += __ldg(val + q) * ldg_na(x + __ldg(col + q));
                }
            }
        } else {
            for (int64_t j = rb + hl; j < re; j += 16) s += __ldg(val + j) * ldg_na(x + __ldg(col + j));
        }
#pragma unroll
        for (int d = 8; d; d >>= 1) s += __shfl_xor_sync(hmask, s, d, 16);
#if SDFGB_SPMV_PF
        if (hl == 0) b[r] = bold + s;
#else
        if (hl == 0) b[r] += s;
#endif
    }
}

template <typename I, typename T>
int launch_spmv(const I* rowptr, const I* col, const T* val, const T* x, T* b, int64_t H,
                void* stream) {
    if (H < 0 || (H > 0 && (!rowptr || !b)))
        return set_error(SDFGB_ERR_INVALID, "spmv: bad arguments");
    if (H == 0) return SDFGB_OK;
    if constexpr (sizeof(T) == 4 && sizeof(I) == 4) {
        if ((reinterpret_cast<uintptr_t>(col) & 15) == 0 && (reinterpret_cast<uintptr_t>(val) & 15) == 0) {
            const int64_t need = (H * 16 + kSpmvBlock - 1) / kSpmvBlock;
            const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)num_sms() * 8));
            spmv_hw_vec4_kernel<<<(unsigned)blocks, kSpmvBlock, 0, as_stream(stream)>>>(
                reinterpret_cast<const int32_t*>(rowptr), reinterpret_cast<const int32_t*>(col),
                reinterpret_cast<const float*>(val), reinterpret_cast<const float*>(x),
                reinterpret_cast<float*>(b), H);
            SDFGB_LAUNCHED("spmv_hw_vec4_kernel");
            return SDFGB_OK;
        }
    }
    const int64_t warps_needed = (H + 1) / 2;
    const int64_t blocks_needed = (warps_needed * 32 + kSpmvBlock - 1) / kSpmvBlock;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(blocks_needed, (int64_t)num_sms() * 8));
    spmv_warp_row_kernel<I, T><<<(unsigned)blocks, kSpmvBlock, 0, as_stream(stream)>>>(
        rowptr, col, val, x, b, H);
    SDFGB_LAUNCHED("spmv_warp_row_kernel");
    return SDFGB_OK;
}

// Measurement probe (not a motif): the SpMV's memory pattern without its
// row structure -- col/val streamed as int4/float4 with evict_first, one
// random x gather per nonzero with evict_last, the products summed into a
// sink.  bench.py times it on the same arrays as the SpMV to measure the
// L2-gather ceiling live (the bound the SpMV kernel runs against).
__global__ void __launch_bounds__(kSpmvBlock)
gather_probe_kernel(const float* __restrict__ x, const int32_t* __restrict__ col, const float* __restrict__ val,
                    int64_t n4, float* __restrict__ sink) {
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    float acc = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * kSpmvBlock + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kSpmvBlock) {
        const int4 c = ldg_stream_i4(col + 4 * i, first);
        const float4 v = ldg_stream_f4(val + 4 * i, first);
        acc += v.x * ldg_keep(x + c.x, last) + v.y * ldg_keep(x + c.y, last) + v.z * ldg_keep(x + c.z, last) +
               v.w * ldg_keep(x + c.w, last);
    }
    if (acc == -1.2345e-30f) sink[0] = acc;  // keeps the loads alive
}

}  // namespace
}  // namespace sdfgb

extern "C" int sdfgb_probe_gather_f32(const float* x, const int32_t* col, const float* val, int64_t nnz, float* sink,
                                      void* stream) {
    if (nnz < 0 || (nnz % 4) != 0 || (nnz > 0 && (!x || !col || !val || !sink)) ||
        (reinterpret_cast<uintptr_t>(col) & 15) || (reinterpret_cast<uintptr_t>(val) & 15))
        return sdfgb::set_error(SDFGB_ERR_INVALID, "probe_gather: nnz % 4 == 0 and 16 B aligned col/val");
    if (nnz == 0) return SDFGB_OK;
    const int64_t blocks = (int64_t)sdfgb::num_sms() * 8;  // the SpMV kernel's residency (8 x 256 threads per SM)
    sdfgb::gather_probe_kernel<<<(unsigned)blocks, sdfgb::kSpmvBlock, 0, sdfgb::as_stream(stream)>>>(
        x, col, val, nnz / 4, sink);
    SDFGB_LAUNCHED("gather_probe_kernel");
    return SDFGB_OK;
}

extern "C" int sdfgb_spmv_csr_f32(const int32_t* rowptr, const int32_t* col, const float* val,
                                  const float* x, float* b, int64_t H, void* stream) {
    return sdfgb::launch_spmv<int32_t, float>(rowptr, col, val, x, b, H, stream);
}
extern "C" int sdfgb_spmv_csr_f64(const int64_t* rowptr, const int64_t* col, const double* val,
                                  const double* x, double* b, int64_t H, void* stream) {
    return sdfgb::launch_spmv<int64_t, double>(rowptr, col, val, x, b, H, stream);
}

// native precision with int32 indices (the host entry narrows the int64
// index arrays losslessly when nnz and W fit): same kernel, half the index bytes
int sdfgb::spmv_csr_f64_i32(const int32_t* rowptr, const int32_t* col, const double* val, const double* x,
                            double* b, int64_t H, cudaStream_t s) {
    return sdfgb::launch_spmv<int32_t, double>(rowptr, col, val, x, b, H, s);
}
