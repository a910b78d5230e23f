// FP32 issue-rate probe on B200: how many FADD / FMUL / FADD2 (add.rn.f32x2)
// warp-instructions per cycle per SM partition, with register operands --
// the Jacobi sweep's instruction mix.  8 (or 16) independent chains per
// thread, 48 warps per SM.  Prints warp-instructions / SMSP / cycle.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, float b, float c, int iters) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    float bb = b + threadIdx.x * 1e-7f, cc = c - threadIdx.x * 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) a[i] = __fadd_rn(a[i], (i & 1) ? bb : cc);     // FADD R, R, R
                if (MODE == 1) a[i] = __fmul_rn(a[i], (i & 1) ? bb : cc);     // FMUL R, R, R
                if (MODE == 2) a[i] = __fadd_rn(a[i], a[(i + 1) & 7]);        // FADD, both sources change
            }
            if (MODE == 3) {  // FADD2: 4 packed pairs
#pragma unroll
                for (int i = 0; i < 8; i += 2) {
                    uint64_t pa, pb, r2;
                    asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a[i]), "f"(a[i + 1]));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(bb), "f"(cc));
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r2) : "l"(pa), "l"(pb));
                    asm("mov.b64 {%0, %1}, %2;" : "=f"(a[i]), "=f"(a[i + 1]) : "l"(r2));
                }
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.f) out[0] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
    const int iters = 4096, threads = 256, blocks = sms * 6;
    const char* names[4] = {"FADD R,R,R", "FMUL R,R,R", "FADD R,R,R (dep sources)", "FADD2 (add.rn.f32x2)"};
    for (int mode = 0; mode < 4; ++mode) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(out, 1.0001f, 0.9999f, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(out, 1.0001f, 0.9999f, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(out, 1.0001f, 0.9999f, iters);
            if (mode == 3) k<3><<<blocks, threads>>>(out, 1.0001f, 0.9999f, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double per_thread = (double)iters * 16 * (mode == 3 ? 4 : 8);
        const double warp_inst = per_thread * threads / 32 * blocks;
        const double cycles = ms * 1e-3 * clk * 1e3;
        printf("%-28s %8.3f ms  %.3f warp-inst/SMSP/cycle (at %d MHz nominal)  %.1f T lane-ops/s\n", names[mode], ms,
               warp_inst / (sms * 4) / cycles, clk / 1000, per_thread * threads * blocks * (mode == 3 ? 2 : 1) / (ms * 1e-3) / 1e12);
    }
    return 0;
}
