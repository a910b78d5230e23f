// hist.cu -- K1: WCR-sum histogram with a dynamic subscript.
//
// Replaces the reference's per-instance subscript write ``h[k] = 1`` under a
// WCR-sum memlet (tasklets.py:297-300 -> interpreter.py:262-278 ->
// codegen.py:733-747 ``hist[k] += 1``) executed once per point of the map
// [0:H-1, 0:W-1].  Binning ``bi = v * S // D`` follows the C emission
// ``(int64_t)floor((double)(v*S) / (double)D)`` (tasklets.py:432-433, :480-481),
// computed here in double so it is bit-identical to the reference for every
// input (fp32 data widens exactly).
//
// B200 design (HBM-bound: 4 B/px read, 256 x 8 B written):
//   * streaming 128-bit loads (ld.global.nc.L1::no_allocate), 4 vectors in
//     flight per thread;
//   * shared-memory-privatised counters, R replicas (warp % R) so skewed
//     images do not serialise one address; a warp whose lanes all hit one
//     bin issues a single add of 32;
//   * 2-CTA thread-block clusters fold their smem histograms through DSMEM
//     into the leader CTA, which alone merges into global memory -> grid/2
//     x bins global atomics.  (8-CTA clusters halve those again but strand
//     SMs: clusters must fit in a GPC, and 16.9 -> 15.8 us measured.)
//   * programmatic dependent launch: the counter init and CTA launch overlap
//     the previous kernel's merge tail (15.8 -> 14.2 us on 4096^2 fp32;
//     sweep in tools/sweep.sh).
#include <algorithm>
#include <cmath>
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sdfgb {
namespace {

#ifndef SDFGB_H_BLOCK
#define SDFGB_H_BLOCK 1024  // one CTA per SM: 13.3 -> 13.0 us at 4096^2 (profiles/r2_hist_variants.txt)
#endif
#ifndef SDFGB_H_UNROLL
#define SDFGB_H_UNROLL 4
#endif
#ifndef SDFGB_H_CLUSTER
#define SDFGB_H_CLUSTER 2
#endif
#ifndef SDFGB_H_PDL
#define SDFGB_H_PDL 1
#endif
constexpr int kHistBlock = SDFGB_H_BLOCK;
constexpr int kHistUnroll = SDFGB_H_UNROLL;
constexpr int kHistCluster = SDFGB_H_CLUSTER;
constexpr int kMaxSmemBins = 12288;  // 48 KB of uint32 counters per replica set

enum BinMode { kScaled = 0, kIdentity = 1, kPow2 = 2 };

// Bin of one element, clamped: an out-of-range element (NaN included) maps to
// the extra "trash" counter at index `bins`, so the update needs no branch and
// the trash counters are exactly the out-of-bounds count.
template <typename T, int MODE>
__device__ __forceinline__ uint32_t bin_clamped(T v, double scale, double div, bool has_div, float scale_f,
                                                uint32_t bins) {
    if constexpr (MODE == kIdentity) {
        const uint64_t k = (uint64_t)(int64_t)v;
        return k < bins ? (uint32_t)k : bins;
    } else if constexpr (MODE == kPow2) {
        // fp32 input, scale = 2^k (k >= 0), div = 1: v * scale is exact, so the
        // floor can be taken in fp32 and equals the reference's floor in double.
        // fma_rd(v, scale, 2^23) = floor(v*scale) + 2^23 exactly for
        // 0 <= v*scale < 2^23, so its bit pattern minus 0x4B000000 is the bin;
        // negative, >= 2^23, inf and NaN inputs all land above `bins` as
        // unsigned.  SASS: FFMA.RM + VIADDMNMX.U32.
        const uint32_t b = (uint32_t)__float_as_int(__fmaf_rd((float)v, scale_f, 8388608.0f)) - 0x4B000000u;
        return min(b, bins);
    } else {
        double q = (double)v * scale;
        if (has_div) q = q / div;
        q = floor(q);
        return (q >= 0.0 && q < (double)bins) ? (uint32_t)q : bins;  // NaN -> trash
    }
}

__device__ __forceinline__ void smem_inc(uint32_t addr) {
    // unused-result shared add of 1: ptxas emits ATOMS.POPC.INC (warp-aggregated)
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}

// Where a CTA's counts go: one hist/oob pair (the one-GPU entries), or every
// rank's pair mapped into this process (peer memory over NVLink): the
// compute step and the all-reduce of the multi-GPU histogram in one kernel,
// each cluster leader adding its bins straight into every rank's histogram.
constexpr int kMaxPeers = 8;
struct HistOut {
    unsigned long long* hist[kMaxPeers];
    unsigned long long* oob[kMaxPeers];
    int n;  // destinations (1 = local only)
};

template <typename T, int MODE>
__global__ void __cluster_dims__(kHistCluster, 1, 1) __launch_bounds__(kHistBlock)
hist_smem_kernel(const T* __restrict__ in, int64_t n, int64_t head, double scale, double div,
                 int64_t bins64, int reps, const HistOut out) {
    extern __shared__ uint32_t sh[];
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::n;
    const bool has_div = div != 1.0;
    const float scale_f = (float)scale;
    const uint32_t bins = (uint32_t)bins64;
    const uint32_t row = bins + 1;  // + trash counter
    const int tid = threadIdx.x;
    const int warp = tid >> 5;

    for (uint32_t k = tid; k < (uint32_t)reps * row; k += blockDim.x) sh[k] = 0u;
    // programmatic dependent launch: everything above overlaps the previous
    // kernel's tail; the image and the counters are touched only after it
    // has completed and flushed (no-op without the launch attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();

    const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(sh) + (uint32_t)(warp % reps) * row * 4u;
    auto bump = [&](T v) { smem_inc(hbase + 4u * bin_clamped<T, MODE>(v, scale, div, has_div, scale_f, bins)); };

    // misaligned head (< VN elements) and ragged tail: block 0, scalar
    const int64_t nvec = (n - head) / VN;
    const int64_t tail0 = head + nvec * VN;
    if (blockIdx.x == 0) {
        for (int64_t p = tid; p < head; p += blockDim.x) bump(in[p]);
        for (int64_t p = tail0 + tid; p < n; p += blockDim.x) bump(in[p]);
    }

    const V* vin = reinterpret_cast<const V*>(in + head);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + tid;
    // software pipeline: the next kHistUnroll vectors are in flight while the
    // current ones are binned
    V cur[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u)
        cur[u] = (i + u * stride < nvec) ? ldg_stream(vin + i + u * stride) : V{};
    for (; i < nvec; i += kHistUnroll * stride) {
        V nxt[kHistUnroll];
        const int64_t j = i + kHistUnroll * stride;
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u)
            nxt[u] = (j + u * stride < nvec) ? ldg_stream(vin + j + u * stride) : V{};
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u)
            if (i + u * stride < nvec) {
#pragma unroll
                for (int c = 0; c < VN; ++c) bump(vget<V, T>(cur[u], c));
            }
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) cur[u] = nxt[u];
    }
    __syncthreads();
    // let the next kernel in the stream start launching its CTAs
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // fold replicas into replica 0 (trash included)
    for (uint32_t k = tid; k < row; k += blockDim.x) {
        uint32_t s = 0;
        for (int r = 0; r < reps; ++r) s += sh[r * row + k];
        sh[k] = s;
    }
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (cluster.block_rank() != 0) {
        uint32_t* lead = cluster.map_shared_rank(sh, 0);
        for (uint32_t k = tid; k < row; k += blockDim.x) {
            const uint32_t c = sh[k];
            if (c) atomicAdd(&lead[k], c);
        }
    }
    cluster.sync();
    if (cluster.block_rank() == 0) {
        if (out.n == 1) {
            for (uint32_t k = tid; k < row; k += blockDim.x) {
                const uint32_t c = sh[k];
                if (c) atomicAdd(k < bins ? &out.hist[0][k] : out.oob[0], (unsigned long long)c);
            }
        } else {
            // system-scope adds into every rank's bins; clusters start at
            // different ranks so the NVLink traffic spreads over the peers
            const int first = (int)(blockIdx.x / kHistCluster) % out.n;
            for (int q = 0; q < out.n; ++q) {
                const int r = (first + q) % out.n;
                for (uint32_t k = tid; k < row; k += blockDim.x) {
                    const uint32_t c = sh[k];
                    if (c) atomicAdd_system(k < bins ? &out.hist[r][k] : out.oob[r], (unsigned long long)c);
                }
            }
        }
    }
}

// Bins beyond the shared-memory budget: direct global WCR (still on device).
template <typename T, int MODE>
__global__ void __launch_bounds__(256)
hist_global_kernel(const T* __restrict__ in, int64_t n, double scale, double div, int64_t bins,
                   unsigned long long* __restrict__ hist, unsigned long long* __restrict__ oob) {
    const bool has_div = div != 1.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = bin_clamped<T, MODE>(in[p], scale, div, has_div, (float)scale, (uint32_t)bins);
        atomicAdd(b < bins ? &hist[b] : oob, 1ull);
    }
}

template <typename T, int MODE>
int launch_hist(const T* img, int64_t n, double scale, double div, int64_t* hist, int64_t bins,
                uint64_t* oob, void* stream, const HistOut* peers = nullptr) {
    if (n < 0 || bins <= 0 || (n > 0 && !img) || (!peers && (!hist || !oob)))
        return set_error(SDFGB_ERR_INVALID, "hist: bad arguments (n=%lld bins=%lld)",
                         (long long)n, (long long)bins);
    if (n == 0) return SDFGB_OK;
    cudaStream_t s = as_stream(stream);
    HistOut out = {};
    if (peers) {
        out = *peers;
    } else {
        out.hist[0] = reinterpret_cast<unsigned long long*>(hist);
        out.oob[0] = reinterpret_cast<unsigned long long*>(oob);
        out.n = 1;
    }
    auto* H = out.hist[0];
    auto* O = out.oob[0];
    if (bins + 1 > kMaxSmemBins || bins >= (1ll << 31)) {
        if (out.n != 1)
            return set_error(SDFGB_ERR_INVALID, "hist_p2p: %lld bins exceed the shared-memory kernel",
                             (long long)bins);
        int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
        hist_global_kernel<T, MODE><<<blocks, 256, 0, s>>>(img, n, scale, div, bins, H, O);
        SDFGB_LAUNCHED("hist_global_kernel");
        return SDFGB_OK;
    }
    constexpr int VN = Vec16<T>::n;
    int reps = (int)std::max<int64_t>(1, std::min<int64_t>(8, kMaxSmemBins / (bins + 1)));
    size_t smem = (size_t)reps * (bins + 1) * sizeof(uint32_t);
    auto kern = hist_smem_kernel<T, MODE>;
    if (smem > 48 * 1024)
        SDFGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    uintptr_t addr = reinterpret_cast<uintptr_t>(img);
    int64_t head = (int64_t)(((16 - (addr & 15)) & 15) / sizeof(T));
    if (head > n) head = n;
    int64_t nvec = (n - head) / VN;
    int64_t want = (nvec + (int64_t)kHistBlock * kHistUnroll - 1) / ((int64_t)kHistBlock * kHistUnroll);
    // one wave of co-resident clusters (a second partial wave would double the tail)
    static int clusters[3][2] = {};
    int& nc = clusters[MODE][sizeof(T) == 8];
    if (nc == 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kHistCluster * 64);
        cfg.blockDim = dim3(kHistBlock);
        cfg.dynamicSmemBytes = smem;
        if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc <= 0) {
            cudaGetLastError();
            int per_sm = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHistBlock, smem);
            nc = std::max(1, per_sm * num_sms() / kHistCluster * 7 / 8);
        }
    }
    int64_t cap = (int64_t)nc * kHistCluster;
    int64_t blocks = std::max<int64_t>(1, std::min(want, cap));
    blocks = (blocks + kHistCluster - 1) / kHistCluster * kHistCluster;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(kHistBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = SDFGB_H_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SDFGB_CUDA(cudaLaunchKernelEx(&cfg, kern, img, n, head, scale, div, bins, reps, out));
    SDFGB_LAUNCHED("hist_smem_kernel");
    return SDFGB_OK;
}

}  // namespace
}  // namespace sdfgb

namespace {
// scale = 2^k with k >= 0, div == 1, and bins < 2^23: the fp32 fast path is exact
bool pow2_exact(double scale, double div, int64_t bins) {
    if (div != 1.0 || !(scale >= 1.0) || scale > 1073741824.0 || bins >= (1 << 23)) return false;
    int e;
    return frexp(scale, &e) == 0.5;
}
}  // namespace

extern "C" int sdfgb_hist_f32_p2p(const float* img, int64_t n, double scale, double div,
                                  int64_t* const* peer_hist, uint64_t* const* peer_oob, int npeers,
                                  int64_t bins, void* stream) {
    if (npeers < 1 || npeers > sdfgb::kMaxPeers || !peer_hist || !peer_oob)
        return sdfgb::set_error(SDFGB_ERR_INVALID, "hist_p2p: 1..%d destinations", sdfgb::kMaxPeers);
    sdfgb::HistOut out = {};
    for (int r = 0; r < npeers; ++r) {
        if (!peer_hist[r] || !peer_oob[r]) return sdfgb::set_error(SDFGB_ERR_INVALID, "hist_p2p: null destination");
        out.hist[r] = reinterpret_cast<unsigned long long*>(peer_hist[r]);
        out.oob[r] = reinterpret_cast<unsigned long long*>(peer_oob[r]);
    }
    out.n = npeers;
    if (pow2_exact(scale, div, bins))
        return sdfgb::launch_hist<float, sdfgb::kPow2>(img, n, scale, div, nullptr, bins, nullptr, stream, &out);
    return sdfgb::launch_hist<float, sdfgb::kScaled>(img, n, scale, div, nullptr, bins, nullptr, stream, &out);
}

extern "C" int sdfgb_hist_f32(const float* img, int64_t n, double scale, double div,
                              int64_t* hist, int64_t bins, uint64_t* oob, void* stream) {
    if (pow2_exact(scale, div, bins))
        return sdfgb::launch_hist<float, sdfgb::kPow2>(img, n, scale, div, hist, bins, oob, stream);
    return sdfgb::launch_hist<float, sdfgb::kScaled>(img, n, scale, div, hist, bins, oob, stream);
}
extern "C" int sdfgb_hist_f64(const double* img, int64_t n, double scale, double div,
                              int64_t* hist, int64_t bins, uint64_t* oob, void* stream) {
    return sdfgb::launch_hist<double, sdfgb::kScaled>(img, n, scale, div, hist, bins, oob, stream);
}
extern "C" int sdfgb_hist_i64(const int64_t* img, int64_t n, int64_t* hist, int64_t bins,
                              uint64_t* oob, void* stream) {
    return sdfgb::launch_hist<int64_t, sdfgb::kIdentity>(img, n, 1.0, 1.0, hist, bins, oob, stream);
}
