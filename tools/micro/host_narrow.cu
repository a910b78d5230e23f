// Host-side narrowing probe: can host threads turn the reference's float64
// buffers into fp32 pinned staging faster than PCIe drains it?
//   (1) pinned / pageable H2D and D2H copy rates (the e2e ceiling)
//   (2) f64 -> f32 narrowing rate into pinned memory for 1..64 threads
//   (3) narrow + H2D pipelined in 8 MB chunks (double-buffered staging)
// nvcc -O3 -std=c++17 -Xcompiler -fopenmp host_narrow.cu -o host_narrow
#include <cuda_runtime.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <chrono>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void narrow(const double* s, float* d, size_t n, int threads) {
#pragma omp parallel for num_threads(threads) schedule(static)
    for (long i = 0; i < (long)n; ++i) d[i] = (float)s[i];
}

int main() {
    const size_t N = (size_t)1 << 26;  // 2^26 doubles = 512 MiB (the Q1 column)
    printf("hardware threads: %u, omp max: %d\n", std::thread::hardware_concurrency(), omp_get_max_threads());
    double* pageable = (double*)malloc(N * 8);
    double* pinned8;
    float* pinned4;
    cudaHostAlloc((void**)&pinned8, N * 8, cudaHostAllocPortable);
    cudaHostAlloc((void**)&pinned4, N * 4, cudaHostAllocPortable);
#pragma omp parallel for
    for (long i = 0; i < (long)N; ++i) pageable[i] = pinned8[i] = (double)(i % 1000) * 1e-3;
    memset(pinned4, 0, N * 4);
    void* dev;
    cudaMalloc(&dev, N * 8);
    cudaStream_t s;
    cudaStreamCreate(&s);
    auto copy = [&](void* dst, const void* src, size_t b, cudaMemcpyKind k) {
        cudaMemcpyAsync(dst, src, b, k, s);
        cudaStreamSynchronize(s);
        double t0 = now();
        for (int r = 0; r < 3; ++r) cudaMemcpyAsync(dst, src, b, k, s);
        cudaStreamSynchronize(s);
        return 3.0 * b / (now() - t0) / 1e9;
    };
    printf("H2D pinned   f64 512MB: %6.1f GB/s\n", copy(dev, pinned8, N * 8, cudaMemcpyHostToDevice));
    printf("H2D pageable f64 512MB: %6.1f GB/s\n", copy(dev, pageable, N * 8, cudaMemcpyHostToDevice));
    printf("D2H pinned   f64 512MB: %6.1f GB/s\n", copy(pinned8, dev, N * 8, cudaMemcpyDeviceToHost));
    printf("D2H pageable f64 512MB: %6.1f GB/s\n", copy(pageable, dev, N * 8, cudaMemcpyDeviceToHost));
    for (int th : {1, 2, 4, 8, 16, 24, 32, 48, 64}) {
        if (th > (int)std::thread::hardware_concurrency()) break;
        narrow(pageable, pinned4, N, th);
        double t0 = now();
        for (int r = 0; r < 3; ++r) narrow(pageable, pinned4, N, th);
        double t = (now() - t0) / 3;
        printf("narrow f64->f32 pageable->pinned, %2d threads: %6.1f GB/s of f64 read (%6.1f GB/s f32 out)\n", th,
               N * 8 / t / 1e9, N * 4 / t / 1e9);
    }
    // pipelined: narrow chunk i+1 while chunk i copies
    for (int th : {8, 16, 32}) {
        if (th > (int)std::thread::hardware_concurrency()) break;
        for (size_t chunk : {(size_t)1 << 20, (size_t)1 << 21, (size_t)1 << 22}) {
            const size_t nch = N / chunk;
            cudaEvent_t ev[2];
            cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                double t0 = now();
                for (size_t i = 0; i < nch; ++i) {
                    const int slot = i & 1;
                    if (i >= 2) cudaEventSynchronize(ev[slot]);
                    float* stage = pinned4 + slot * chunk;
                    narrow(pageable + i * chunk, stage, chunk, th);
                    cudaMemcpyAsync((float*)dev + i * chunk, stage, chunk * 4, cudaMemcpyHostToDevice, s);
                    cudaEventRecord(ev[slot], s);
                }
                cudaStreamSynchronize(s);
                best = std::min(best, now() - t0);
            }
            printf("pipelined narrow+H2D %2d threads chunk %5zu K: %6.2f ms (%6.1f GB/s f64-equivalent)\n", th,
                   chunk >> 10, best * 1e3, N * 8 / best / 1e9);
        }
    }
    return 0;
}
