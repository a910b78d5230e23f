// common.cuh -- shared helpers for libsdfgb200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/sdfgb200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libsdfgb200 targets sm_100a only"
#endif

namespace sdfgb {

constexpr int kNumSMs = 148;  // B200; queried at runtime where it matters

int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
int num_sms();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// internal building blocks of the host entries (capi.cu), not exported
// B's operands after the split: hi / lo K-major transposed ([N][K]), or (mn)
// B itself and its lo part, row-major [K][N], read MN-major by the pair kernel
struct GemmB {
    const float* hi;
    const float* lo;
    bool mn;
};
int gemm_split_b(const float* B, float* Bhi, float* Blo, int64_t K, int64_t N, cudaStream_t s, GemmB* out);
GemmB gemm_b_operands(const float* B, float* Bhi, float* Blo, int64_t K, int64_t N);  // after gemm_split_b
int gemm_f32_presplit(const float* A, const GemmB& b, float* C, int64_t M, int64_t N, int64_t K, float* Ahi,
                      float* Alo, cudaStream_t s);
int spmv_csr_f64_i32(const int32_t* rowptr, const int32_t* col, const double* val, const double* x, double* b,
                     int64_t H, cudaStream_t s);

#define SDFGB_TRY(expr)                                         \
    do {                                                        \
        int _rc = (expr);                                       \
        if (_rc != SDFGB_OK) return _rc;                        \
    } while (0)

#define SDFGB_CUDA(expr) SDFGB_TRY(::sdfgb::check_cuda((expr), #expr))
#define SDFGB_LAUNCHED(name) SDFGB_TRY(::sdfgb::check_cuda(cudaGetLastError(), name))

// ---------------------------------------------------------------- device
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldg_stream(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ longlong2 ldg_stream(const longlong2* p) {
    longlong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0,%1}, [%2];"
                 : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };
template <> struct Vec16<int64_t> { using type = longlong2; static constexpr int n = 2; };

template <typename V, typename T>
__device__ __forceinline__ T vget(const V& v, int c) { return reinterpret_cast<const T*>(&v)[c]; }

__device__ __forceinline__ int cmp_apply(double v, int op, double t) {
    switch (op) {
    case SDFGB_CMP_LT: return v < t;
    case SDFGB_CMP_LE: return v <= t;
    case SDFGB_CMP_GT: return v > t;
    case SDFGB_CMP_GE: return v >= t;
    case SDFGB_CMP_EQ: return v == t;
    default: return v != t;
    }
}

}  // namespace sdfgb
