// Does add.rn.f32x2 / mul.rn.f32x2 round like add.rn.f32 / mul.rn.f32?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(const float* a, const float* b, unsigned long long* bad_add, unsigned long long* bad_mul, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    float a0 = a[2 * i], a1 = a[2 * i + 1], b0 = b[2 * i], b1 = b[2 * i + 1];
    uint64_t pa, pb, r, m;
    asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(b0), "f"(b1));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pa), "l"(pb));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(pa), "l"(pb));
    float r0, r1, m0, m1;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r0), "=f"(r1) : "l"(r));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(m0), "=f"(m1) : "l"(m));
    if (__float_as_uint(r0) != __float_as_uint(__fadd_rn(a0, b0)) || __float_as_uint(r1) != __float_as_uint(__fadd_rn(a1, b1)))
        atomicAdd(bad_add, 1ull);
    if (__float_as_uint(m0) != __float_as_uint(__fmul_rn(a0, b0)) || __float_as_uint(m1) != __float_as_uint(__fmul_rn(a1, b1)))
        atomicAdd(bad_mul, 1ull);
}
int main() {
    const int n = 1 << 24;
    float *a, *b;
    unsigned long long* c;
    cudaMallocManaged(&a, n * 4);
    cudaMallocManaged(&b, n * 4);
    cudaMallocManaged(&c, 16);
    uint32_t s = 12345;
    for (int i = 0; i < n; ++i) {
        s = s * 1664525u + 1013904223u;
        a[i] = (float)(s >> 8) / 16777216.0f;
        s = s * 1664525u + 1013904223u;
        b[i] = (float)(s >> 8) / 16777216.0f * ((i % 3) ? 1.0f : 0.2f);
    }
    c[0] = c[1] = 0;
    k<<<(n / 2 + 255) / 256, 256>>>(a, b, c, c + 1, n);
    cudaDeviceSynchronize();
    printf("pairs %d  add mismatches %llu  mul mismatches %llu\n", n / 2, c[0], c[1]);
    return 0;
}
