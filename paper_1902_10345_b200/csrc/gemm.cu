// gemm.cu -- K5: the MapReduceFusion'd matmul map on tcgen05 tensor cores.
//
// Reference: gallery.matmul (gallery.py:107-144) after MapReduceFusion
// (library.py:461-554): an init state writes C = 0, then the 3-D map
// (i, j, k) accumulates C[i, j] += A[i, k] * B[k, j] through a WCR-sum memlet.
// Only this motif is a dense contraction, so only it goes to the tensor pipe.
//
// fp32 accuracy from TF32 tensor cores via the 3xTF32 split:
//     A = Ahi + Alo, Ahi = tf32(A), Alo = A - Ahi (exact in fp32)
//     C ~= Ahi*Bhi + Ahi*Blo + Alo*Bhi        (Alo*Blo ~ 2^-20 dropped)
// 1xTF32 would miss the 1e-4 tolerance (6.8e-4 at K=4096).
// The tensor core keeps the top 19 bits of a kind::tf32 operand (it
// truncates), so the pair kernel reads A and B themselves as the hi
// operands -- A K-major, B MN-major straight from its row-major [K][N]
// layout -- and the pre-pass writes only Alo and Blo = x - trunc_tf32(x)
// (round 2; the older kernels below still take rna-split, K-major B^T).
//
// v1 structure (one 128x128 C tile per CTA, 256 threads):
//   * split pre-pass writes Ahi/Alo (M x K) and Bt_hi/Bt_lo (N x K), all
//     K-major so every operand is a TMA SWIZZLE_128B K-major tile;
//   * warp 0: TMA producer over a 3-stage smem ring (64 KB/stage), mbarrier
//     full/empty pipeline;
//   * warp 1: single-thread tcgen05.mma.kind::tf32 issuer, M=128 N=128 K=8,
//     3 MMAs per K=8 step; k-blocks go round-robin into NACC = 4 TMEM
//     accumulators (4 x 128 cols = all 512 columns).  The tensor core's fp32
//     accumulation is biased (measured: -1.7e-4 rel at K=16384 with one
//     accumulator on positive data); four partial sums cut the accumulated
//     magnitude per accumulator by 4x and are combined in the epilogue with
//     IEEE round-to-nearest adds;
//   * tcgen05.commit frees smem stages and finally signals the epilogue;
//   * warp 2: TMEM allocator; warps 4-7: tcgen05.ld -> registers -> C.
#include <algorithm>
#include <mutex>

#include <cstdlib>

#include "tma.cuh"

namespace sdfgb {
namespace {

// UMMA shared-memory descriptor, K-major SWIZZLE_128B (cute::UMMA::SmemDescriptor):
// start>>4 [0,14) | LBO=1 [16,30) | SBO=1024>>4 [32,46) | version=1 [46,48) | layout=2 [61,64)
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}
// UMMA shared-memory descriptor, MN-major SWIZZLE_128B: atoms of 32 MN-contiguous
// fp32 (128 B) x 8 K rows (1 KB); LBO = byte stride between MN atoms, SBO =
// byte stride between 8-row K groups (cute::UMMA::make_umma_desc<Major::MN>)
#ifndef SDFGB_BMN_LAYOUT
#define SDFGB_BMN_LAYOUT 1  // descriptor layout type: 1 = SWIZZLE_128B_BASE32B (MN-major tf32), 2 = SWIZZLE_128B
#endif
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)SDFGB_BMN_LAYOUT << 61);
}
// instruction descriptor kind::tf32, fp32 accumulate, A/B K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------------ split pre-pass
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

#ifndef SDFGB_GEMM_PDL
#define SDFGB_GEMM_PDL 1  // programmatic dependent launch: split pre-pass and pair kernel
#endif
#ifndef SDFGB_GEMM_RAW_AHI
#define SDFGB_GEMM_RAW_AHI 1  // 4096^3: 0.592 -> 0.584 ms, same error class (profiles/r2_gemm_variants.txt)
#endif
// A's hi part read straight from A (the tensor core keeps the top 19 bits of
// a kind::tf32 operand, i.e. truncates): only lo = a - trunc_tf32(a) is written
__global__ void split_lo_kernel(const float4* __restrict__ A, float4* __restrict__ lo, int64_t n4) {
#if SDFGB_GEMM_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the previous kernel (a GEMM reading lo) is done
#endif
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = A[i];
        auto l = [](float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); };
        lo[i] = make_float4(l(a.x), l(a.y), l(a.z), l(a.w));
    }
}

// the lo pre-pass with programmatic dependent launch (SDFGB_GEMM_PDL)
int launch_split(const float4* a, float4* lo, int64_t n4, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(num_sms() * 8));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = SDFGB_GEMM_PDL;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    return check_cuda(cudaLaunchKernelEx(&cfg, split_lo_kernel, a, lo, n4), "split_lo launch");
}

__global__ void split_rows_kernel(const float* __restrict__ A, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float a = A[i];
        float h = tf32_rna(a);
        hi[i] = h;
        lo[i] = a - h;
    }
}

// B (K x N, row-major) -> Bt_hi / Bt_lo (N x K, row-major) via 32x32 smem tiles
__global__ void split_transpose_kernel(const float* __restrict__ B, float* __restrict__ hi,
                                       float* __restrict__ lo, int64_t K, int64_t N) {
    __shared__ float t[32][33];
    const int64_t k0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t k = k0 + r, n = n0 + threadIdx.x;
        t[r][threadIdx.x] = (k < K && n < N) ? B[k * N + n] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t n = n0 + r, k = k0 + threadIdx.x;
        if (n < N && k < K) {
            float a = t[threadIdx.x][r];
            float h = tf32_rna(a);
            hi[n * K + k] = h;
            lo[n * K + k] = a - h;
        }
    }
}

// 64 x 64 tiles, float4 both ways (the 32 x 32 scalar version ran at
// 4.1 TB/s of 192 MB): rows k of B in, rows n of Bt_hi / Bt_lo out
__global__ void __launch_bounds__(256)
split_transpose64_kernel(const float* __restrict__ B, float* __restrict__ hi, float* __restrict__ lo,
                         int64_t K, int64_t N) {
    __shared__ float t[64][65];
    const int64_t k0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
    const int tid = threadIdx.x;
#pragma unroll
    for (int p = 0; p < 4; ++p) {  // 64 rows x 16 float4
        const int r = p * 16 + tid / 16, c4 = (tid % 16) * 4;
        const int64_t k = k0 + r, n = n0 + c4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < K && n + 3 < N) {
            v = *reinterpret_cast<const float4*>(B + k * N + n);
        } else if (k < K) {
            float e[4] = {0.f, 0.f, 0.f, 0.f};
            for (int q = 0; q < 4; ++q)
                if (n + q < N) e[q] = B[k * N + n + q];
            v = make_float4(e[0], e[1], e[2], e[3]);
        }
        t[r][c4] = v.x;
        t[r][c4 + 1] = v.y;
        t[r][c4 + 2] = v.z;
        t[r][c4 + 3] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; ++p) {  // 64 rows (n) x 16 float4 (k)
        const int r = p * 16 + tid / 16, c4 = (tid % 16) * 4;
        const int64_t n = n0 + r, k = k0 + c4;
        if (n >= N) continue;
        float h[4], l[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            h[q] = tf32_rna(t[c4 + q][r]);
            l[q] = t[c4 + q][r] - h[q];
        }
        if (k + 3 < K) {
            *reinterpret_cast<float4*>(hi + n * K + k) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(lo + n * K + k) = make_float4(l[0], l[1], l[2], l[3]);
        } else {
            for (int q = 0; q < 4; ++q)
                if (k + q < K) {
                    hi[n * K + k + q] = h[q];
                    lo[n * K + k + q] = l[q];
                }
        }
    }
}

// ------------------------------------------------------------ tcgen05 GEMM
constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3;
constexpr int TILE_BYTES = BM * BK * 4;              // 16 KB (BM == BN)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;          // Ahi, Alo, Bhi, Blo
constexpr int GEMM_THREADS = 256;
#ifndef SDFGB_GEMM_NACC
#define SDFGB_GEMM_NACC 4
#endif
#ifndef SDFGB_GEMM_GROUP
#define SDFGB_GEMM_GROUP 16
#endif
#ifndef SDFGB_GEMM_TMEM_COLS
#define SDFGB_GEMM_TMEM_COLS (BN * SDFGB_GEMM_NACC)
#endif
constexpr int NACC = SDFGB_GEMM_NACC;                // TMEM accumulators
constexpr int TMEM_COLS = SDFGB_GEMM_TMEM_COLS;      // power of two >= 32
constexpr int GEMM_SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                   const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                   float* __restrict__ C, int M, int N, int K) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // grouped rasterisation: consecutive CTAs cover SDFGB_GEMM_GROUP tile rows
    // x a few tile columns, so a wave of co-resident CTAs shares ~26 operand
    // panels instead of ~5 A + 148 B panels (row-major order re-read every B
    // panel from DRAM once per tile row: ~280 GB at 16384^3)
    int m0, n0;
    {
        const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
        const int pid = blockIdx.x, group = SDFGB_GEMM_GROUP * tiles_n;
        const int first_m = (pid / group) * SDFGB_GEMM_GROUP;
        const int gm = min(tiles_m - first_m, SDFGB_GEMM_GROUP);
        const int in_group = pid % group;
        m0 = (first_m + in_group % gm) * BM;
        n0 = (in_group / gm) * BN;
    }
    const int KB = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAlo)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBlo)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                mbar_expect_tx(&full[s], STAGE_BYTES);
                tma_load_2d(st + 0 * TILE_BYTES, &mAhi, &full[s], kb * BK, m0);
                tma_load_2d(st + 1 * TILE_BYTES, &mAlo, &full[s], kb * BK, m0);
                tma_load_2d(st + 2 * TILE_BYTES, &mBhi, &full[s], kb * BK, n0);
                tma_load_2d(st + 3 * TILE_BYTES, &mBlo, &full[s], kb * BK, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(BM, BN);
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
                const uint32_t dacc = tmem_d + (uint32_t)((kb % NACC) * BN);
                const uint32_t first = kb < NACC;
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {
                    const uint32_t off = k * 32;  // 8 tf32 = 32 B along K inside the 128 B atom
                    const uint64_t ahi = sw128_kmajor_desc(base + 0 * TILE_BYTES + off);
                    const uint64_t alo = sw128_kmajor_desc(base + 1 * TILE_BYTES + off);
                    const uint64_t bhi = sw128_kmajor_desc(base + 2 * TILE_BYTES + off);
                    const uint64_t blo = sw128_kmajor_desc(base + 3 * TILE_BYTES + off);
                    tc_mma_tf32(dacc, alo, bhi, idesc, !(first && k == 0));
                    tc_mma_tf32(dacc, ahi, blo, idesc, 1u);
                    tc_mma_tf32(dacc, ahi, bhi, idesc, 1u);
                }
                tc_commit(&empty[s]);
            }
            tc_commit(tmem_full);
        }
    } else if (warp >= 4) {
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int rw = (warp & 3) * 32;
        const int row = m0 + rw + lane;
        const int nacc = KB < NACC ? KB : NACC;
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
            uint32_t r[16];
            tmem_ld16(tmem_d + ((uint32_t)rw << 16) + c, r);
            for (int q = 1; q < nacc; ++q) {  // (acc0 + acc1) + acc2 ... in RN fp32
                uint32_t o[16];
                tmem_ld16(tmem_d + ((uint32_t)rw << 16) + q * BN + c, o);
#pragma unroll
                for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) + __uint_as_float(o[e]));
            }
            if (row < M) {
                float* dst = C + (int64_t)row * N + n0 + c;
                if (n0 + c + 16 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        reinterpret_cast<float4*>(dst)[q] =
                            make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                        __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        if (n0 + c + q < N) dst[q] = __uint_as_float(r[q]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(TMEM_COLS));
    }
}

// ------------------------------------------------------------ CTA-pair GEMM
// cta_group::2: the two CTAs of a cluster form one 256 x 128 tile.  Each CTA
// stages its own 128 rows of A and its half (64 rows) of the B tile; the
// leader issues M = 256, N = 128 MMAs that read both CTAs' shared memory,
// and each CTA's TMEM receives its 128 rows.  Per 128 x 128 x 8 step a CTA's
// shared memory then takes 48 KB of operand fill and 6 KB of MMA reads
// instead of 64 / 8 KB (profiles/r1_gemm_bound_experiment.txt: shared-memory
// bytes per flop are what bounds the one-CTA kernel).
#ifndef SDFGB_GEMM_WD
#define SDFGB_GEMM_WD 0  // 1: trap instead of hanging on a stuck barrier (bring-up)
#endif
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity) {
#if SDFGB_GEMM_WD
    long long spins = 0;
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            " selp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (++spins > (1LL << 28)) __trap();
    }
#else
    mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ uint32_t pair_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void pair_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// both CTAs load their halves; the bytes count on the LEADER's barrier
// (shared::cluster address with the peer bit cleared)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u)
        : "memory");
}
// the same MMA with an A-collector hint: FILL keeps the A tile in the
// tensor core's operand collector, LASTUSE reads it from there (no second
// shared-memory read of A) and releases it
enum { kCollFill = 1, kCollLastUse = 2 };
template <int COLL>
__device__ __forceinline__ void tc_mma_tf32_pair_c(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                   uint32_t accumulate) {
    if constexpr (COLL == kCollFill) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32.collector::a::fill [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32.collector::a::lastuse [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
            : "memory");
    }
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // arrive on this offset in both CTAs
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

#ifndef SDFGB_GEMM_AREUSE
#define SDFGB_GEMM_AREUSE 1  // A-collector reuse between the two A-hi MMAs of a K = 8 step
#endif
#ifndef SDFGB_GEMM_PAIR_GROUP
#define SDFGB_GEMM_PAIR_GROUP 8  // tile rows per rasterisation group (sweep: 4 / 8 / 16 / 32)
#endif
#ifndef SDFGB_GEMM_PAIR_STAGES
#define SDFGB_GEMM_PAIR_STAGES 4
#endif
#ifndef SDFGB_GEMM_PAIR_NACC
#define SDFGB_GEMM_PAIR_NACC 4
#endif
#ifndef SDFGB_GEMM_PAIR_MINB
#define SDFGB_GEMM_PAIR_MINB 1
#endif
constexpr int STAGES2 = SDFGB_GEMM_PAIR_STAGES;
constexpr int PNACC = SDFGB_GEMM_PAIR_NACC;       // TMEM accumulators of the pair kernel
constexpr int PTMEM_COLS = BN * PNACC;
constexpr int BHALF = BN / 2;                                // B rows each CTA stages
constexpr int BTILE2 = BHALF * BK * 4;                       // 8 KB
constexpr int STAGE2_BYTES = 2 * TILE_BYTES + 2 * BTILE2;    // 48 KB: Ahi, Alo, Bhi half, Blo half
constexpr int GEMM2_SMEM = STAGES2 * STAGE2_BYTES + 1024 + 256;

#ifndef SDFGB_BMN_LBO
#define SDFGB_BMN_LBO 4096  // bytes between 32-column MN atoms (one 32 x 32 TMA box)
#endif
#ifndef SDFGB_BMN_SBO
#define SDFGB_BMN_SBO 512  // bytes between 4-row K groups (128 B rows)
#endif
#ifndef SDFGB_BMN_KSTEP
#define SDFGB_BMN_KSTEP 1024  // descriptor start advance per K = 8 MMA
#endif
// BMN: B's hi / lo come MN-major straight from row-major [K][N] buffers (B itself
// and its lo part): TMA boxes of 32 N x 32 K, the MMA's B descriptor MN-major
template <bool BMN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, SDFGB_GEMM_PAIR_MINB)
gemm_3xtf32_pair_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                        const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                        float* __restrict__ C, int M, int N, int K) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
    uint64_t* empty = full + STAGES2;
    uint64_t* tmem_full = empty + STAGES2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = pair_rank();
    int m0, n0;  // this CTA's 128 rows; the pair's 128 columns
    {
        constexpr int G = SDFGB_GEMM_PAIR_GROUP / 2;  // pair rows per group
        const int tiles_m = (M + 2 * BM - 1) / (2 * BM), tiles_n = (N + BN - 1) / BN;
        const int pid = blockIdx.x / 2, group = G * tiles_n;
        const int first_m = (pid / group) * G;
        const int gm = min(tiles_m - first_m, G);
        const int in_group = pid % group;
        m0 = (first_m + in_group % gm) * 2 * BM + (int)rank * BM;
        n0 = (in_group / gm) * BN;
    }
    const int KB = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAlo)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBlo)) : "memory");
    }
    if (warp == 2) {  // the same warp in both CTAs
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(PTMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    pair_sync();  // the peer's barriers are initialised before any load signals them
#if SDFGB_GEMM_PDL
    // programmatic dependent launch: the set-up above (barriers, TMEM,
    // descriptor prefetch) overlapped the split pre-pass; its output is read
    // only from here on
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // producer, in both CTAs
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % STAGES2;
                const uint32_t ph = (kb / STAGES2) & 1;
                mbar_wait_wd(&empty[s], ph ^ 1);  // both CTAs' stage s consumed by the pair MMA
                uint8_t* st = smem + s * STAGE2_BYTES;
                if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE2_BYTES);  // both halves
                const uint32_t lbar = smem_u32(&full[s]) & 0xFEFFFFFFu;
                tma_load_2d_pair(st + 0 * TILE_BYTES, &mAhi, lbar, kb * BK, m0);
                tma_load_2d_pair(st + 1 * TILE_BYTES, &mAlo, lbar, kb * BK, m0);
                if constexpr (BMN) {  // two 32-column MN atoms per half
#pragma unroll
                    for (int h = 0; h < BHALF / 32; ++h) {
                        tma_load_2d_pair(st + 2 * TILE_BYTES + h * 32 * BK * 4, &mBhi, lbar,
                                         n0 + (int)rank * BHALF + 32 * h, kb * BK);
                        tma_load_2d_pair(st + 2 * TILE_BYTES + BTILE2 + h * 32 * BK * 4, &mBlo, lbar,
                                         n0 + (int)rank * BHALF + 32 * h, kb * BK);
                    }
                } else {
                    tma_load_2d_pair(st + 2 * TILE_BYTES, &mBhi, lbar, kb * BK, n0 + (int)rank * BHALF);
                    tma_load_2d_pair(st + 2 * TILE_BYTES + BTILE2, &mBlo, lbar, kb * BK, n0 + (int)rank * BHALF);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {  // the leader issues the pair's MMAs
            constexpr uint32_t idesc = idesc_tf32(2 * BM, BN) | (BMN ? (1u << 16) : 0u);  // bit 16: B MN-major
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % STAGES2;
                const uint32_t ph = (kb / STAGES2) & 1;
                mbar_wait_wd(&full[s], ph);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * STAGE2_BYTES);
                const uint32_t dacc = tmem_d + (uint32_t)((kb % PNACC) * BN);
                const uint32_t first = kb < PNACC;
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {
                    const uint32_t off = k * 32;
                    const uint64_t ahi = sw128_kmajor_desc(base + 0 * TILE_BYTES + off);
                    const uint64_t alo = sw128_kmajor_desc(base + 1 * TILE_BYTES + off);
                    // MN-major B: the k-th K=8 slice is the k-th 1 KB row group of every atom
                    const uint64_t bhi = BMN ? sw128_mnmajor_desc(base + 2 * TILE_BYTES + k * SDFGB_BMN_KSTEP,
                                                                  SDFGB_BMN_LBO, SDFGB_BMN_SBO)
                                             : sw128_kmajor_desc(base + 2 * TILE_BYTES + off);
                    const uint64_t blo = BMN ? sw128_mnmajor_desc(base + 2 * TILE_BYTES + BTILE2 + k * SDFGB_BMN_KSTEP,
                                                                  SDFGB_BMN_LBO, SDFGB_BMN_SBO)
                                             : sw128_kmajor_desc(base + 2 * TILE_BYTES + BTILE2 + off);
#if SDFGB_GEMM_AREUSE
                    // A hi feeds two MMAs from one shared-memory read
                    tc_mma_tf32_pair_c<kCollFill>(dacc, ahi, blo, idesc, !(first && k == 0));
                    tc_mma_tf32_pair_c<kCollLastUse>(dacc, ahi, bhi, idesc, 1u);
                    tc_mma_tf32_pair(dacc, alo, bhi, idesc, 1u);
#else
                    tc_mma_tf32_pair(dacc, alo, bhi, idesc, !(first && k == 0));
                    tc_mma_tf32_pair(dacc, ahi, blo, idesc, 1u);
                    tc_mma_tf32_pair(dacc, ahi, bhi, idesc, 1u);
#endif
                }
                tc_commit_pair(&empty[s]);
            }
            tc_commit_pair(tmem_full);
        }
    } else if (warp >= 4) {  // epilogue, in both CTAs: this CTA's 128 rows
        mbar_wait_wd(tmem_full, 0);
        tc_fence_after();
        const int rw = (warp & 3) * 32;
        const int row = m0 + rw + lane;
        const int nacc = KB < PNACC ? KB : PNACC;
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
            uint32_t r[16];
            tmem_ld16(tmem_d + ((uint32_t)rw << 16) + c, r);
            for (int q = 1; q < nacc; ++q) {
                uint32_t o[16];
                tmem_ld16(tmem_d + ((uint32_t)rw << 16) + q * BN + c, o);
#pragma unroll
                for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) + __uint_as_float(o[e]));
            }
            if (row < M) {
                float* dst = C + (int64_t)row * N + n0 + c;
                if (n0 + c + 16 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        reinterpret_cast<float4*>(dst)[q] =
                            make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                        __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        if (n0 + c + q < N) dst[q] = __uint_as_float(r[q]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    pair_sync();  // neither CTA leaves while the pair's MMAs / commits may touch it
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(PTMEM_COLS));
    }
}

// Long contractions: the same pipeline, but every CHUNK uses of an
// accumulator are folded into per-thread fp32 registers by 8 epilogue warps
// (2 per TMEM lane quarter) while the tensor core keeps going on the other
// three accumulators.  The tensor core's truncating accumulation then spans
// at most CHUNK k-blocks per accumulator whatever K is: max relative error
// 2.7e-6 at K = 16384 (one accumulation per accumulator: 4.4e-5, growing
// linearly with K).  Measured ~5 % slower at 4096^3 / 16384^3, so
// sdfgb_gemm_f32 selects it only for K > kFlushK.
constexpr int FLUSH_EPI_WARPS = 8;
constexpr int FLUSH_THREADS = 128 + 32 * FLUSH_EPI_WARPS;
constexpr int CHUNK = 8;        // uses of one accumulator (k-blocks) per chunk
constexpr int64_t kFlushK = 16384;

__global__ void __launch_bounds__(FLUSH_THREADS, 1)
gemm_3xtf32_flush_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                   const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                   float* __restrict__ C, int M, int N, int K) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;   // [NACC]: an accumulator's chunk is complete
    uint64_t* acc_empty = acc_full + NACC; // [NACC]: the epilogue has folded it into registers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // grouped rasterisation: consecutive CTAs cover SDFGB_GEMM_GROUP tile rows
    // x a few tile columns, so a wave of co-resident CTAs shares ~26 operand
    // panels instead of ~5 A + 148 B panels (row-major order re-read every B
    // panel from DRAM once per tile row: ~280 GB at 16384^3)
    int m0, n0;
    {
        const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
        const int pid = blockIdx.x, group = SDFGB_GEMM_GROUP * tiles_n;
        const int first_m = (pid / group) * SDFGB_GEMM_GROUP;
        const int gm = min(tiles_m - first_m, SDFGB_GEMM_GROUP);
        const int in_group = pid % group;
        m0 = (first_m + in_group % gm) * BM;
        n0 = (in_group / gm) * BN;
    }
    const int KB = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < NACC; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 32 * FLUSH_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAlo)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBlo)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                mbar_expect_tx(&full[s], STAGE_BYTES);
                tma_load_2d(st + 0 * TILE_BYTES, &mAhi, &full[s], kb * BK, m0);
                tma_load_2d(st + 1 * TILE_BYTES, &mAlo, &full[s], kb * BK, m0);
                tma_load_2d(st + 2 * TILE_BYTES, &mBhi, &full[s], kb * BK, n0);
                tma_load_2d(st + 3 * TILE_BYTES, &mBlo, &full[s], kb * BK, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(BM, BN);
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                // k-block kb -> accumulator a = kb % 4 (round robin: four
                // independent accumulation chains keep the tensor pipe full);
                // every CHUNK uses of an accumulator form a chunk that the
                // epilogue folds into registers before the accumulator's next
                // use, staggered across the four accumulators
                const int a = kb & (NACC - 1), u = kb / NACC, cu = u / CHUNK, j = u - cu * CHUNK;
                if (j == 0 && cu >= 1) {
                    mbar_wait(&acc_empty[a], (cu - 1) & 1);  // chunk cu-1 of this accumulator folded
                    tc_fence_after();
                }
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
                const uint32_t dacc = tmem_d + (uint32_t)(a * BN);
                const uint32_t first = j == 0;
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {
                    const uint32_t off = k * 32;  // 8 tf32 = 32 B along K inside the 128 B atom
                    const uint64_t ahi = sw128_kmajor_desc(base + 0 * TILE_BYTES + off);
                    const uint64_t alo = sw128_kmajor_desc(base + 1 * TILE_BYTES + off);
                    const uint64_t bhi = sw128_kmajor_desc(base + 2 * TILE_BYTES + off);
                    const uint64_t blo = sw128_kmajor_desc(base + 3 * TILE_BYTES + off);
                    tc_mma_tf32(dacc, alo, bhi, idesc, !(first && k == 0));
                    tc_mma_tf32(dacc, ahi, blo, idesc, 1u);
                    tc_mma_tf32(dacc, ahi, bhi, idesc, 1u);
                }
                tc_commit(&empty[s]);
                if (j == CHUNK - 1 || kb + NACC >= KB) tc_commit(&acc_full[a]);
            }
        }
    } else if (warp >= 4) {
        // Each thread owns one output row (its TMEM lane) and keeps the
        // row's running fp32 sum in registers: every finished accumulator
        // chunk is folded in with IEEE adds, so the tensor core's truncating
        // accumulation spans at most CHUNK k-blocks per accumulator whatever
        // K is (one long accumulation per accumulator biased the result by
        // ~1e-8 per k-block: 4.4e-5 relative at K = 16384).
        constexpr int HC = BN * 4 / FLUSH_EPI_WARPS;  // columns per epilogue warp
        const int rw = (warp & 3) * 32;
        const int h0 = ((warp - 4) >> 2) * HC;
        const int row = m0 + rw + lane;
        const int uses0 = (KB + NACC - 1) / NACC;  // uses of accumulator 0 (the most)
        const int nchunks = (uses0 + CHUNK - 1) / CHUNK;
        float sum[HC];
#pragma unroll
        for (int e = 0; e < HC; ++e) sum[e] = 0.f;
        for (int cu = 0; cu < nchunks; ++cu) {
#pragma unroll 1
            for (int a = 0; a < NACC; ++a) {  // the order the chunks complete in
                const int uses = (KB - a + NACC - 1) / NACC;
                if (cu * CHUNK >= uses) continue;
                mbar_wait_sleep(&acc_full[a], cu & 1, 512);
                tc_fence_after();
                const uint32_t t0 = tmem_d + ((uint32_t)rw << 16) + (uint32_t)(a * BN + h0);
#pragma unroll
                for (int cc = 0; cc < HC; cc += 16) {
                    uint32_t r[16];
                    tmem_ld16(t0 + cc, r);
#pragma unroll
                    for (int e = 0; e < 16; ++e) sum[cc + e] += __uint_as_float(r[e]);
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[a]);
            }
        }
#pragma unroll
        for (int cq = 0; cq < HC; cq += 16) {
            const int c = h0 + cq;
            uint32_t r[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(sum[cq + e]);
            if (row < M) {
                float* dst = C + (int64_t)row * N + n0 + c;
                if (n0 + c + 16 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        reinterpret_cast<float4*>(dst)[q] =
                            make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                        __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        if (n0 + c + q < N) dst[q] = __uint_as_float(r[q]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(TMEM_COLS));
    }
}

// ------------------------------------------------------------ SIMT GEMMs
// 64x64 tile, 256 threads, 4x4 per thread, each element accumulated over k in
// order.  float: FFMA (the cross-check of the tensor-core kernel).  double
// (native precision): separate IEEE multiply and add from 0 in k order --
// exactly the reference's MapReduceFusion loop `C += A*B` after init_C
// (library.py:461-554; its C is compiled without FMA contraction), so the
// result is bit-identical to the reference's generated code.
template <typename T>
__device__ __forceinline__ T mac(T acc, T a, T b);
template <>
__device__ __forceinline__ float mac<float>(float acc, float a, float b) { return fmaf(a, b, acc); }
template <>
__device__ __forceinline__ double mac<double>(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
}

template <typename T>
__global__ void __launch_bounds__(256)
gemm_simt_kernel(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                 int64_t M, int64_t N, int64_t K) {
    __shared__ T As[16][64 + 4];
    __shared__ T Bs[16][64 + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
    T acc[4][4] = {};
    for (int64_t k0 = 0; k0 < K; k0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            const int kk = e % 16, mm = e / 16;
            As[kk][mm] = (m0 + mm < M && k0 + kk < K) ? A[(m0 + mm) * K + k0 + kk] : T(0);
            const int nn = e % 64, kb = e / 64;
            Bs[kb][nn] = (n0 + nn < N && k0 + kb < K) ? B[(k0 + kb) * N + n0 + nn] : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = mac<T>(acc[i][j], As[kk][ty * 4 + i], Bs[kk][tx * 4 + j]);
        __syncthreads();
    }
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            const int64_t m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
            if (m < M && n < N) C[m * N + n] = acc[i][j];
        }
}

// ------------------------------------------------------------ host side
int make_kmajor_map(CUtensorMap* map, const float* base, int64_t rows, int64_t K, int box_rows = BM) {
    return encode_tiled_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, rows, K, BK, box_rows,
                           CU_TENSOR_MAP_SWIZZLE_128B);
}

// CTA-pair kernel by default (4096^3: 611 -> 594 us; 16384^3 on par);
// SDFGB_GEMM_PAIR=0 selects the one-CTA kernel
bool gemm_use_pair() {
#ifndef SDFGB_GEMM_PAIR_DEFAULT
#define SDFGB_GEMM_PAIR_DEFAULT 1
#endif
    static const bool on = [] {
        const char* e = getenv("SDFGB_GEMM_PAIR");
        return e ? atoi(e) != 0 : SDFGB_GEMM_PAIR_DEFAULT != 0;
    }();
    return on;
}

}  // namespace
}  // namespace sdfgb

extern "C" size_t sdfgb_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
    // Ahi, Alo (M x K) and Bt_hi, Bt_lo (N x K), each 256-byte aligned
    auto r = [](size_t b) { return (b + 255) / 256 * 256; };
    return 2 * r((size_t)M * K * 4) + 2 * r((size_t)N * K * 4);
}

namespace sdfgb {

// B (K x N, row-major) -> Bt_hi / Bt_lo (N x K, K-major): the 3xTF32 split of
// the right operand, done once per B (the host entry's row panels share it)
#ifndef SDFGB_GEMM_BMN
#define SDFGB_GEMM_BMN 1  // the pair kernel reads B's hi / lo MN-major (no transpose in the pre-pass)
#endif
// the pair kernel reads B MN-major (no transpose) when it runs and B / Blo are aligned
static bool gemm_b_mn(const float* B, const float* Blo, int64_t K, int64_t N) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(Blo)) & 15) == 0;
    return SDFGB_GEMM_BMN && K <= kFlushK && gemm_use_pair() && N % 4 == 0 && aligned;
}

GemmB gemm_b_operands(const float* B, float* Bhi, float* Blo, int64_t K, int64_t N) {
    return gemm_b_mn(B, Blo, K, N) ? GemmB{B, Blo, true} : GemmB{Bhi, Blo, false};
}

int gemm_split_b(const float* B, float* Bhi, float* Blo, int64_t K, int64_t N, cudaStream_t s, GemmB* out) {
    if (gemm_b_mn(B, Blo, K, N)) {
        // MN-major: B's hi is B itself (tensor-core truncation), only lo is written, untransposed
        SDFGB_TRY(launch_split(reinterpret_cast<const float4*>(B), reinterpret_cast<float4*>(Blo), K * N / 4, s));
        SDFGB_LAUNCHED("split_lo_kernel");
        *out = {B, Blo, true};
        return SDFGB_OK;
    }
    if (N % 4 == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0) {  // K % 4 == 0 already
        dim3 tg((unsigned)((N + 63) / 64), (unsigned)((K + 63) / 64));
        split_transpose64_kernel<<<tg, 256, 0, s>>>(B, Bhi, Blo, K, N);
        SDFGB_LAUNCHED("split_transpose64_kernel");
    } else {
        dim3 tg((unsigned)((N + 31) / 32), (unsigned)((K + 31) / 32));
        split_transpose_kernel<<<tg, dim3(32, 8), 0, s>>>(B, Bhi, Blo, K, N);
        SDFGB_LAUNCHED("split_transpose_kernel");
    }
    *out = {Bhi, Blo, false};
    return SDFGB_OK;
}

// C = A x B with B already split (gemm_split_b); Ahi / Alo hold M x K each
// The pair kernel with programmatic dependent launch (SDFGB_GEMM_PDL): its
// CTAs start while the split pre-pass drains (the kernel waits on it with
// griddepcontrol.wait before its first load).
template <typename K>
int launch_pair(K kern, unsigned grid, cudaStream_t s, const CUtensorMap& a, const CUtensorMap& b,
                const CUtensorMap& c, const CUtensorMap& d, float* C, int M, int N, int Kd) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = GEMM2_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = SDFGB_GEMM_PDL;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    return check_cuda(cudaLaunchKernelEx(&cfg, kern, a, b, c, d, C, M, N, Kd), "gemm pair launch");
}

int gemm_f32_presplit(const float* A, const GemmB& b, float* C, int64_t M, int64_t N, int64_t K, float* Ahi,
                      float* Alo, cudaStream_t s) {
    const float* Bhi = b.hi;
    const float* Blo = b.lo;
    CUtensorMap mAhi, mAlo, mBhi, mBlo;
    if (SDFGB_GEMM_RAW_AHI && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(Alo)) & 15) == 0) {
        SDFGB_TRY(launch_split(reinterpret_cast<const float4*>(A), reinterpret_cast<float4*>(Alo), M * K / 4, s));
        SDFGB_LAUNCHED("split_lo_kernel");
        SDFGB_TRY(make_kmajor_map(&mAhi, A, M, K));
    } else {
        split_rows_kernel<<<num_sms() * 8, 256, 0, s>>>(A, Ahi, Alo, M * K);
        SDFGB_LAUNCHED("split_rows_kernel");
        SDFGB_TRY(make_kmajor_map(&mAhi, Ahi, M, K));
    }
    SDFGB_TRY(make_kmajor_map(&mAlo, Alo, M, K));
    if (K <= kFlushK && gemm_use_pair()) {
        static std::once_flag attr2;
        static cudaError_t attr2_err = cudaSuccess;
        std::call_once(attr2, [] {
            attr2_err = cudaFuncSetAttribute(gemm_3xtf32_pair_kernel<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM2_SMEM);
            if (attr2_err == cudaSuccess)
                attr2_err = cudaFuncSetAttribute(gemm_3xtf32_pair_kernel<true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM2_SMEM);
        });
        SDFGB_CUDA(attr2_err);
        const int64_t pairs = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
        if (b.mn) {  // row-major [K][N] B operands, 32 x 32 boxes (one 128 B swizzle span of N)
            // MN-major tf32 operands take the "128 B swizzle, 32 B atomicity" smem layout
            // (CUTLASS: Layout_MN_SW128_32B_Atom, the only one it allows for them)
            constexpr CUtensorMapSwizzle sw = SDFGB_BMN_LAYOUT == 1 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                                                     : CU_TENSOR_MAP_SWIZZLE_128B;
            SDFGB_TRY(encode_tiled_2d(&mBhi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Bhi, K, N, 32, BK, sw));
            SDFGB_TRY(encode_tiled_2d(&mBlo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Blo, K, N, 32, BK, sw));
            SDFGB_TRY(launch_pair(gemm_3xtf32_pair_kernel<true>, (unsigned)(2 * pairs), s, mAhi, mAlo, mBhi, mBlo, C,
                                  (int)M, (int)N, (int)K));
        } else {
            SDFGB_TRY(make_kmajor_map(&mBhi, Bhi, N, K, BHALF));
            SDFGB_TRY(make_kmajor_map(&mBlo, Blo, N, K, BHALF));
            SDFGB_TRY(launch_pair(gemm_3xtf32_pair_kernel<false>, (unsigned)(2 * pairs), s, mAhi, mAlo, mBhi, mBlo, C,
                                  (int)M, (int)N, (int)K));
        }
        SDFGB_LAUNCHED("gemm_3xtf32_pair_kernel");
        return SDFGB_OK;
    }
    if (b.mn) return set_error(SDFGB_ERR_INVALID, "gemm: MN-major B needs the pair kernel");
    SDFGB_TRY(make_kmajor_map(&mBhi, Bhi, N, K));
    SDFGB_TRY(make_kmajor_map(&mBlo, Blo, N, K));
    static std::once_flag attr;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr, [] {
        attr_err = cudaFuncSetAttribute(gemm_3xtf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
        if (attr_err == cudaSuccess)
            attr_err = cudaFuncSetAttribute(gemm_3xtf32_flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            GEMM_SMEM);
    });
    SDFGB_CUDA(attr_err);
    dim3 grid((unsigned)(((N + BN - 1) / BN) * ((M + BM - 1) / BM)));
    if (K > kFlushK || getenv("SDFGB_GEMM_FLUSH")) {
        gemm_3xtf32_flush_kernel<<<grid, FLUSH_THREADS, GEMM_SMEM, s>>>(mAhi, mAlo, mBhi, mBlo, C, (int)M, (int)N,
                                                                         (int)K);
        SDFGB_LAUNCHED("gemm_3xtf32_flush_kernel");
    } else {
        gemm_3xtf32_kernel<<<grid, GEMM_THREADS, GEMM_SMEM, s>>>(mAhi, mAlo, mBhi, mBlo, C, (int)M, (int)N, (int)K);
        SDFGB_LAUNCHED("gemm_3xtf32_kernel");
    }
    return SDFGB_OK;
}

}  // namespace sdfgb

extern "C" int sdfgb_gemm_f32_ex(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                                 void* ws, size_t ws_bytes, int flags, void* stream) {
    using namespace sdfgb;
    if (M < 0 || N < 0 || K < 0 || (M * N > 0 && !C))
        return set_error(SDFGB_ERR_INVALID, "gemm: bad arguments");
    if (M == 0 || N == 0) return SDFGB_OK;
    cudaStream_t s = as_stream(stream);
    if (K == 0) {  // init_C state only: C = 0 (library.py:541-554)
        SDFGB_CUDA(cudaMemsetAsync(C, 0, (size_t)M * N * 4, s));
        return SDFGB_OK;
    }
    if (K % 4 != 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
        return set_error(SDFGB_ERR_INVALID, "gemm: K must be a multiple of 4 (TMA row stride)");
    if (!A || !B || !ws || ws_bytes < sdfgb_gemm_workspace_bytes(M, N, K))
        return set_error(SDFGB_ERR_WORKSPACE, "gemm: workspace too small");
    // workspace: B's split first (its place does not depend on M, so row
    // pieces of one product can share it), then A's
    auto r = [](size_t b) { return (b + 255) / 256 * 256; };
    uint8_t* w = static_cast<uint8_t*>(ws);
    float* Bhi = reinterpret_cast<float*>(w);
    float* Blo = reinterpret_cast<float*>(w + r((size_t)N * K * 4));
    float* Ahi = reinterpret_cast<float*>(w + 2 * r((size_t)N * K * 4));
    float* Alo = reinterpret_cast<float*>(w + 2 * r((size_t)N * K * 4) + r((size_t)M * K * 4));
    GemmB bops;
    if (flags & SDFGB_GEMM_B_SPLIT)
        bops = gemm_b_operands(B, Bhi, Blo, K, N);  // split by an earlier call with this B and workspace
    else
        SDFGB_TRY(gemm_split_b(B, Bhi, Blo, K, N, s, &bops));
    return gemm_f32_presplit(A, bops, C, M, N, K, Ahi, Alo, s);
}

extern "C" int sdfgb_gemm_f32(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                              void* ws, size_t ws_bytes, void* stream) {
    return sdfgb_gemm_f32_ex(A, B, C, M, N, K, ws, ws_bytes, 0, stream);
}

extern "C" int sdfgb_gemm_f32_simt(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                                   void* stream) {
    using namespace sdfgb;
    if (M < 0 || N < 0 || K < 0 || (M * N > 0 && (!A || !B || !C)))
        return set_error(SDFGB_ERR_INVALID, "gemm_simt: bad arguments");
    if (M == 0 || N == 0) return SDFGB_OK;
    dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
    gemm_simt_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(A, B, C, M, N, K);
    SDFGB_LAUNCHED("gemm_simt_kernel");
    return SDFGB_OK;
}

extern "C" int sdfgb_gemm_f64(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K,
                              void* stream) {
    using namespace sdfgb;
    if (M < 0 || N < 0 || K < 0 || (M * N > 0 && (!C || (K > 0 && (!A || !B)))))
        return set_error(SDFGB_ERR_INVALID, "gemm_f64: bad arguments");
    if (M == 0 || N == 0) return SDFGB_OK;
    dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
    gemm_simt_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(A, B, C, M, N, K);
    SDFGB_LAUNCHED("gemm_simt_kernel");
    return SDFGB_OK;
}
