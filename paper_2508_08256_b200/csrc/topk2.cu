// topk2.cu -- K3 (register path): per-row Top-k with one wide histogram pass.
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores, ties
// to the LOWER index, returned in ascending index order.  The algorithm (one
// thread-block cluster per row, keys in registers, one 512-bin histogram,
// candidate refinement, exact rank, ballot compaction) lives in select.cuh and
// is shared with the fused decode step (step_fused.cu); this kernel loads the
// row's scores from memory and writes the selection to memory.
#include <cstdlib>

#include "select.cuh"

namespace fier_cuda {

template <int KPT>
__global__ void __launch_bounds__(kT2Threads, 2) topk2_kernel(const float* __restrict__ scores, int tokens,
                                                              int64_t ld, int k, int slice,
                                                              int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* srow = scores + (int64_t)row * ld;
    const int s0 = rank * slice;
    const int cnt = max(0, min(s0 + slice, tokens) - s0);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    T2Shared& S = *reinterpret_cast<T2Shared*>(smem_raw);

    // every CTA of the cluster must be running before anyone stores into its smem
    asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
    const int wbase = warp * 32 * KPT;
    uint32_t key[KPT];
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const int p = wbase + 32 * j + lane;
        const float v = p < cnt ? srow[s0 + p] : __int_as_float(0x7fffffff);
        // 1: a NaN score (ranks lowest, score_key), 0: an empty slot past the row end.  Kept
        // branch-free around the load: with the row-end test first the compiler serialised
        // the KPT loads (C4 Top-k 151 -> 251 us).
        key[j] = isnan(v) ? (p < cnt ? 1u : 0u) : float_key(v);
        if (isfinite(v)) {
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
    }
    const RegKeys<KPT> keys{key};
    const T2Threshold th = t2_threshold<kT2Threads>(cluster, keys, mn, mx, s0, wbase, k, S);
    int32_t* out = sel + (int64_t)row * k;
    uint32_t base, count;
    t2_compact<kT2Threads>(cluster, keys, th, S, &base, &count,
                    [&](uint32_t slot, int j) { out[slot] = s0 + wbase + 32 * j + lane; });
}

// Long slices (> 16 keys per thread): the keys live in shared memory (64 KB next to the
// 46 KB T2Shared: still two CTAs per SM) instead of 32 registers per thread, which at the
// 64-register cap of two 512-thread CTAs per SM spilled to local memory.
__global__ void __launch_bounds__(kT2Threads, 2) topk2s_kernel(const float* __restrict__ scores, int tokens,
                                                               int64_t ld, int k, int slice, int kpt,
                                                               int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* srow = scores + (int64_t)row * ld;
    const int s0 = rank * slice;
    const int cnt = max(0, min(s0 + slice, tokens) - s0);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    T2Shared& S = *reinterpret_cast<T2Shared*>(smem_raw);
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(smem_raw + (sizeof(T2Shared) + 15) / 16 * 16);

    asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
    const int wbase = warp * 32 * kpt;
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll 8
    for (int j = 0; j < kpt; ++j) {
        const int p = wbase + 32 * j + lane;
        const float v = p < cnt ? srow[s0 + p] : __int_as_float(0x7fffffff);
        keys_s[p] = isnan(v) ? (p < cnt ? 1u : 0u) : float_key(v);  // 1: NaN score, 0: empty slot
        if (isfinite(v)) {
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
    }
    const SmemKeys keys{keys_s + wbase, kpt};  // read after t2_threshold's first CTA barrier
    const T2Threshold th = t2_threshold<kT2Threads>(cluster, keys, mn, mx, s0, wbase, k, S);
    int32_t* out = sel + (int64_t)row * k;
    uint32_t base, count;
    t2_compact<kT2Threads>(cluster, keys, th, S, &base, &count,
                           [&](uint32_t slot, int j) { out[slot] = s0 + wbase + 32 * j + lane; });
}

static int launch_t2s(int cluster, int rows, cudaStream_t st, const float* scores, int tokens, int64_t ld, int k,
                      int kpt, int32_t* sel) {
    const size_t smem = (sizeof(T2Shared) + 15) / 16 * 16 + (size_t)kT2Threads * kpt * 4;
    static bool attr = [&] {
        cudaFuncSetAttribute(topk2s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((sizeof(T2Shared) + 15) / 16 * 16 + kT2Threads * 32 * 4));
        cudaFuncSetAttribute(topk2s_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(kT2Threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cluster;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, topk2s_kernel, scores, tokens, ld, k, kpt * kT2Threads, kpt, sel);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

template <int KPT>
static int launch_t2(int cluster, int rows, cudaStream_t st, const float* scores, int tokens, int64_t ld, int k,
                     int slice, int32_t* sel) {
    auto kern = topk2_kernel<KPT>;
    const size_t smem = sizeof(T2Shared);
    static bool attr = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(kT2Threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cluster;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, scores, tokens, ld, k, slice, sel);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

// Rows up to kT2MaxCluster * 512 * 32 keys.  Returns -1 if the row is too long.
int topk2_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st) {
    int c = 1;
    // grow the cluster until the grid covers the chip (or slices reach 8 keys per thread),
    // then until the slice fits the 32 registers per thread
    constexpr int max_c = 4;
    while (c < max_c && (int64_t)rows * c < 2 * num_sms() && ceil_div(tokens, c) > 8 * kT2Threads) c *= 2;
    while (c < kT2MaxCluster && ceil_div(tokens, c) > 32 * kT2Threads) c *= 2;
    const int64_t slice = ceil_div(tokens, c);
    if (slice > 32 * kT2Threads) return -1;
    const int kpt = (int)ceil_div(slice, kT2Threads);
    if (kpt <= 1) return launch_t2<1>(c, rows, st, scores, tokens, ld, k, kT2Threads, sel);
    if (kpt <= 2) return launch_t2<2>(c, rows, st, scores, tokens, ld, k, 2 * kT2Threads, sel);
    if (kpt <= 4) return launch_t2<4>(c, rows, st, scores, tokens, ld, k, 4 * kT2Threads, sel);
    if (kpt <= 8) return launch_t2<8>(c, rows, st, scores, tokens, ld, k, 8 * kT2Threads, sel);
    if (kpt <= 16) return launch_t2<16>(c, rows, st, scores, tokens, ld, k, 16 * kT2Threads, sel);
    return launch_t2s(c, rows, st, scores, tokens, ld, k, 32, sel);
}

}  // namespace fier_cuda
