// Issue-rate ceiling of the Jacobi strip sweep's instruction mix: the same
// 7-level register window and calc (2 SHFL + 16 FADD + 4 FMUL per level per
// lane), fed by (0) a synthetic level-0 row in registers, (1) three LDS.128
// per row from a shared-memory ring (the strip kernel's level 0), (2) plus
// one STG.128 per row (the output level), (3) plus a TMA refill of the ring
// every three rows with the warp-vote mbarrier wait.  Prints warp
// instructions / SMSP / cycle and lane-op throughput per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

constexpr int F = 7;

__device__ __forceinline__ float4 calc(const float4& nq, const float4& cq, const float4& sq, float coef) {
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
}

#include <cuda.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int V>
__global__ void __launch_bounds__(128, 4) k(float4* out, float coef, int rows, const __grid_constant__ CUtensorMap map) {
    __shared__ __align__(128) float ring[4][6][384];
    __shared__ uint64_t bars[4][6];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* rg = ring[warp][0];
    if (V >= 3 && lane == 0) {
        for (int s = 0; s < 6; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[warp][s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < 6; ++s) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[warp][s])), "r"(1536) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(su32(rg + s * 384)), "l"(&map), "r"(su32(&bars[warp][s])), "r"(0), "r"(3 * s) : "memory");
        }
    }
    if (V >= 1 && V < 3) for (int i = lane; i < 6 * 384; i += 32) rg[i] = i * 1e-4f;
    __syncwarp();
    float4 w[F][3];
#pragma unroll
    for (int a = 0; a < F; ++a)
#pragma unroll
        for (int u = 0; u < 3; ++u) w[a][u] = make_float4(threadIdx.x, a, u, 1.f);
    float4 acc = make_float4(0, 0, 0, 0);
    auto step = [&](auto u_tag, int p) {
        constexpr int u = decltype(u_tag)::value, sn = (u + 1) % 3, sc = (u + 2) % 3;
        const int it = p / 3, slot = it % 6, pslot = (it + 5) % 6;
        const float* stage = rg + slot * 384;
        const float* prev = rg + pslot * 384;
        if constexpr (V >= 3 && u == 0) {
            const uint32_t a = su32(&bars[warp][slot]), par = (uint32_t)((it / 6) & 1);
            uint32_t ok = 0;
            do {
                asm volatile("{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n"
                             : "=r"(ok) : "r"(a), "r"(par) : "memory");
            } while (!__all_sync(0xffffffffu, ok));
        }
        auto l0 = [&](int q) {
            const float* b = q >= 0 ? stage + q * 128 : prev + (q + 3) * 128;
            return *reinterpret_cast<const float4*>(b + 4 * lane);
        };
        if constexpr (V == 0) {
            w[0][u] = make_float4(p * 1e-6f, w[0][sc].x * 0.5f, 0.25f, w[0][sn].w);
#pragma unroll
            for (int kk = 1; kk < F; ++kk) w[kk][u] = calc(w[kk - 1][sn], w[kk - 1][sc], w[kk - 1][u], coef);
        } else {
            w[1][u] = calc(l0(u - 2), l0(u - 1), l0(u), coef);
#pragma unroll
            for (int kk = 2; kk < F; ++kk) w[kk][u] = calc(w[kk - 1][sn], w[kk - 1][sc], w[kk - 1][u], coef);
        }
        const float4 o = calc(w[F - 1][sn], w[F - 1][sc], w[F - 1][u], coef);
        if constexpr (V >= 2) {
            out[((size_t)blockIdx.x * 4 + warp) * 4096 + (p & 4095) * 32 + lane] = o;
        } else {
            acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
        }
        if constexpr (V >= 3 && u == 2) {
            __syncwarp();
            const int nx = it - 1 + 6;
            if (lane == 0 && it >= 1 && nx < rows / 3) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[warp][pslot])), "r"(1536) : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(su32(prev)), "l"(&map), "r"(su32(&bars[warp][pslot])), "r"(0), "r"((3 * nx) & 8191) : "memory");
            }
        }
    };
    for (int p = 0; p < rows; p += 3) {
        step(std::integral_constant<int, 0>{}, p);
        step(std::integral_constant<int, 1>{}, p + 1);
        step(std::integral_constant<int, 2>{}, p + 2);
    }
    if (acc.x == 123.f) out[threadIdx.x] = acc;
    if constexpr (V >= 3) {  // drain the refills still in flight
        for (int s = 0; s < 6; ++s) {
            const int it = rows / 3 + s - 1;
            (void)it;
        }
        __syncwarp();
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    float4* out;
    cudaMalloc(&out, (size_t)148 * 4 * 4 * 4096 * 32 * 16);
    float* plane;
    cudaMalloc(&plane, (size_t)8192 * 128 * 4);
    cudaMemset(plane, 0, (size_t)8192 * 128 * 4);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {128, 8192}, strides[1] = {128 * 4};
    cuuint32_t box[2] = {128, 3}, es[2] = {1, 1};
    ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, plane, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int rows = 3 * 2000;
    const char* names[4] = {"registers only", "+ level 0 from smem (3 LDS/row)", "+ STG.128 per row",
                            "+ TMA ring refill + mbarrier vote"};
    for (int v = 0; v < 4; ++v) {
        const int blocks = sms * 4;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (v == 0) k<0><<<blocks, 128>>>(out, 0.2f, rows, map);
            if (v == 1) k<1><<<blocks, 128>>>(out, 0.2f, rows, map);
            if (v == 2) k<2><<<blocks, 128>>>(out, 0.2f, rows, map);
            if (v == 3) k<3><<<blocks, 128>>>(out, 0.2f, rows, map);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double warps = blocks * 4.0;
        const double lane_pts = warps * 32 * 4 * rows * F;
        printf("%-36s %.3f ms  %.1f T lane-ops/s (5 per point-level)  %s\n", names[v], ms,
               lane_pts * 5 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
