// topk_rx.cu -- K3 (standalone Top-k over scores in memory) on the fused step's
// fixed-radix select (select_radix.cuh).
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores, ties to
// the LOWER index, returned in ascending index order.  One thread-block cluster of
// C <= 16 CTAs (512 threads) per row; CTA r loads its slice of the row ONCE into
// shared-memory keys (order-preserving u32, warp-run layout of select.cuh),
// counting each key into the 12-bit digit histogram as it goes; then the two-barrier
// radix threshold and the emit pass of select_radix.cuh write the ascending
// selection.  Versus topk2.cu (register keys, adaptive 512-bin histograms over the
// (min, max) range, four cluster barriers) this needs two barriers and two passes
// over the keys; candidate overflow takes the same exact MSD radix fallback.
// Rows up to 16 x 16384 tokens.  Opt-in (FIER_TOPK=rx): at 112 registers x 512
// threads one CTA fits per SM, so C3's 256 CTAs run in two waves (55 us vs 25.6 us
// for topk2's register keys at two CTAs per SM; C4 241 vs 151 us) -- the radix
// select pays off inside the fused step, where the keys never leave the chip.
#include <cstdlib>
#include <string>

#include "select_radix.cuh"

namespace fier_cuda {

constexpr int kTrThreads = 512;
constexpr int kTrMaxKpt = 32;  // slice <= 16384 keys (64 KB of shared-memory keys)

__device__ __noinline__ void topk_rx_fallback(cg::cluster_group& cluster, const SmemKeys& keys, int k, RxShared& S,
                                              int32_t* out, int s0, int wbase) {
    const int lane = threadIdx.x & 31;
    const T2Threshold th = t2_radix_select<kTrThreads>(cluster, keys, k, S);
    uint32_t base = 0, count = 0;
    t2_compact<kTrThreads>(cluster, keys, th, S, &base, &count,
                           [&](uint32_t slot, int j) { out[slot] = s0 + wbase + 32 * j + lane; });
}

__global__ void __launch_bounds__(kTrThreads, 1) topk_rx_kernel(const float* __restrict__ scores, int tokens,
                                                                int64_t ld, int k, int kpt,
                                                                int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int slice = kTrThreads * kpt;
    const int s0 = rank * slice;
    const int wbase = warp * 32 * kpt;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    RxShared& S = *reinterpret_cast<RxShared*>(smem_raw);
    RxPublished& P = *reinterpret_cast<RxPublished*>(smem_raw + (sizeof(RxShared) + 15) / 16 * 16);
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(smem_raw + (sizeof(RxShared) + 15) / 16 * 16 +
                                                   (sizeof(RxPublished) + 15) / 16 * 16);
    rx_clear<kTrThreads>(S);
    __syncthreads();
    // ---- keys of this CTA's slice: one coalesced pass, 8 loads in flight per thread ----
    const float* srow = scores + (int64_t)row * ld;
    uint32_t* run = keys_s + wbase;
    for (int j0 = 0; j0 < kpt; j0 += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int t = s0 + wbase + 32 * (j0 + u) + lane;
            v[u] = (j0 + u < kpt && t < tokens) ? __ldg(srow + t) : __int_as_float(0x7fffffff);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (j0 + u < kpt) {
                const uint32_t key = isnan(v[u]) ? 0u : float_key(v[u]);  // NaN / past the end: empty
                run[32 * (j0 + u) + lane] = key;
                rx_count(S, key);
            }
        }
    }
    const SmemKeys keys{run, kpt};
    int32_t* out = sel + (int64_t)row * k;
    const RxResult R = rx_threshold<kTrThreads>(cluster, keys, s0, wbase, slice, k, S, P);
    if (!R.fallback) {
        // peers may still read this CTA's candidate list: arrive now, wait before exiting
        asm volatile("barrier.cluster.arrive.release;" ::: "memory");
        rx_emit<kTrThreads>(keys, R, s0, wbase, S, [&](uint32_t slot, int j) { out[slot] = s0 + wbase + 32 * j + lane; });
        asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
    } else {
        topk_rx_fallback(cluster, keys, k, S, out, s0, wbase);
    }
}

static size_t topk_rx_smem(int kpt) {
    return (sizeof(RxShared) + 15) / 16 * 16 + (sizeof(RxPublished) + 15) / 16 * 16 +
           (size_t)kTrThreads * kpt * 4;
}

static bool topk_rx_enabled() {  // FIER_TOPK=rx (A/B measurements)
    static const bool v = [] {
        const char* e = getenv("FIER_TOPK");
        return e && std::string(e) == "rx";
    }();
    return v;
}

// Returns -1 if the row is too long for this kernel.
int topk_rx_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st) {
    if (!topk_rx_enabled() || rows > 65535) return -1;
    int c = 1;
    while (c < kT2MaxCluster && ceil_div(tokens, c) > (int64_t)kTrThreads * kTrMaxKpt) c *= 2;
    if (ceil_div(tokens, c) > (int64_t)kTrThreads * kTrMaxKpt) return -1;
    // one CTA per SM: grow the cluster while the grid stays within one wave
    while (c < kT2MaxCluster && (int64_t)rows * c * 2 <= num_sms() && ceil_div(tokens, 2 * c) >= 2 * kTrThreads) c *= 2;
    const int kpt = (int)ceil_div(ceil_div(tokens, c), kTrThreads);
    const int cluster = (int)ceil_div(tokens, (int64_t)kTrThreads * kpt);
    const size_t smem = topk_rx_smem(kpt);
    static const bool attr = [] {
        cudaFuncSetAttribute(topk_rx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)topk_rx_smem(kTrMaxKpt));
        cudaFuncSetAttribute(topk_rx_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(kTrThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cluster;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, topk_rx_kernel, scores, tokens, ld, k, kpt, sel);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

}  // namespace fier_cuda
