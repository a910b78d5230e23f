// Ceiling for the SpMV x gathers: 2^28 random 4 B reads from a 16 MB
// (L2-resident) vector, (a) with hashed indices (no index stream) and (b)
// with the indices and values streamed from HBM like CSR col/val.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__global__ void gather_hash(const float* __restrict__ x, uint32_t mask, int64_t n, float* out) {
    float acc = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += __ldg(x + (hash((uint32_t)i) & mask));
    if (acc == 12345.f) out[0] = acc;
}

__global__ void gather_stream(const float* __restrict__ x, const int4* __restrict__ col, const float4* __restrict__ val,
                              int64_t n4, float* out) {
    float acc = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 c = __ldcs(col + i);
        const float4 v = __ldcs(val + i);
        acc += v.x * __ldg(x + c.x) + v.y * __ldg(x + c.y) + v.z * __ldg(x + c.z) + v.w * __ldg(x + c.w);
    }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void fill_idx(int* col, int64_t n, uint32_t mask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        col[i] = hash((uint32_t)i * 2654435761u) & mask;
}

int main() {
    const int64_t W = 1 << 22, n = (int64_t)1 << 28;
    float *x, *val, *out;
    int* col;
    cudaMalloc(&x, W * 4); cudaMalloc(&val, n * 4); cudaMalloc(&col, n * 4); cudaMalloc(&out, 4);
    cudaMemset(x, 0, W * 4); cudaMemset(val, 0, n * 4);
    fill_idx<<<1184, 256>>>(col, n, W - 1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int occ : {4, 8, 16}) {
        for (int k = 0; k < 2; ++k) {
            float ms;
            for (int w = 0; w < 2; ++w) {
                cudaEventRecord(a);
                if (k == 0) gather_hash<<<sms * occ, 256>>>(x, W - 1, n, out);
                else gather_stream<<<sms * occ, 256>>>(x, (const int4*)col, (const float4*)val, n / 4, out);
                cudaEventRecord(b); cudaEventSynchronize(b);
            }
            cudaEventElapsedTime(&ms, a, b);
            printf("%s occ=%2d  %.3f ms  %.1f Ggathers/s  %.0f GB/s sectors\n", k ? "stream" : "hash  ", occ, ms,
                   n / ms / 1e6, n * 32.0 / ms / 1e6);
        }
    }
    return 0;
}
