// topk.cu -- K3: per-head Top-k token selector (radix select, exact tie rule).
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores,
// ties to the LOWER index, returned in ascending index order.
//
// One thread-block cluster (C CTAs, C <= 8) per score row; CTA r owns the
// contiguous slice [r*S, (r+1)*S) of the row, caches its order-preserving u32
// keys in shared memory, and the cluster runs three radix passes (11/11/10
// bits) over them.  Each pass builds a shared-memory histogram of the keys
// still matching the resolved prefix; the cluster sums the C histograms over
// distributed shared memory and every CTA finds the same digit (deterministic,
// no atomics across CTAs).  After the passes the exact threshold key T and
// the number r of T-valued keys to keep are known.  Compaction is a pure
// function of index order: a key at position i is kept iff key > T or
// (key == T and #(T-valued keys before i) < r), and its output slot is
// #(> T before i) + min(#(== T before i), r) -- warp ballots + a block scan
// + a cluster prefix over the CTA totals, so the output is ascending without
// any sort.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace fier_cuda {

constexpr int kTkThreads = 1024;
constexpr int kTkBins = 2048;
constexpr int kTkMaxCached = 32768;  // keys per CTA kept in shared memory
constexpr int kTkMisc = 160;  // scan scratch [0,64), results [64,72), warp counts [72,136)

// Block-wide exclusive scan of one u32 per thread; returns the exclusive
// prefix and writes the block total to *total (all threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t w = lane < nw ? scratch[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        scratch[32 + lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    const uint32_t warp_excl = warp ? scratch[32 + warp - 1] : 0u;
    *total = scratch[32 + (blockDim.x >> 5) - 1];
    const uint32_t r = warp_excl + x - v;
    __syncthreads();
    return r;
}

template <bool CACHED>
__global__ void __launch_bounds__(kTkThreads, 1)
    topk_kernel(const float* __restrict__ scores, int tokens, int64_t ld, int k, int slice,
                int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* srow = scores + (int64_t)row * ld;
    const int s0 = rank * slice;
    const int cnt = max(0, min(s0 + slice, tokens) - s0);

    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* hist0 = smem;
    uint32_t* hist1 = smem + kTkBins;
    uint32_t* tot = smem + 2 * kTkBins;
    uint32_t* misc = smem + 3 * kTkBins;  // [0..63] scan scratch, [64..] results
    uint32_t* keys = misc + kTkMisc;

    uint32_t prefix = 0, pmask = 0;
    uint32_t krem = (uint32_t)k;

#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
        const int bins = pass == 2 ? 1024 : 2048;
        uint32_t* hist = (pass & 1) ? hist1 : hist0;
        for (int i = tid; i < bins; i += kTkThreads) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < cnt; i += kTkThreads) {
            uint32_t key;
            if (CACHED && pass > 0) {
                key = keys[i];
            } else {
                key = float_key(srow[s0 + i]);
                if (CACHED) keys[i] = key;
            }
            if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & (bins - 1)], 1u);
        }
        cluster.sync();
        for (int i = tid; i < bins; i += kTkThreads) {
            uint32_t acc = 0;
            for (int r = 0; r < nct; ++r) acc += cluster.map_shared_rank(hist, r)[i];
            tot[i] = acc;
        }
        __syncthreads();
        // Digit search, descending: thread t owns descending positions
        // [t*per, (t+1)*per).  Find the bin where the running count from the
        // top first reaches krem.
        const int per = bins / kTkThreads;
        uint32_t local = 0;
        for (int j = 0; j < per; ++j) local += tot[bins - 1 - (tid * per + j)];
        uint32_t total;
        uint32_t above = block_excl_scan(local, misc, &total);
        for (int j = 0; j < per; ++j) {
            const int bin = bins - 1 - (tid * per + j);
            const uint32_t c = tot[bin];
            if (above < krem && krem <= above + c) {
                misc[64] = (uint32_t)bin;
                misc[65] = above;
            }
            above += c;
        }
        __syncthreads();
        const uint32_t bin = misc[64];
        krem -= misc[65];
        prefix |= bin << shift;
        pmask |= (uint32_t)(bins - 1) << shift;
        __syncthreads();
    }
    const uint32_t T = prefix;  // exact threshold key; keep krem keys equal to T

    // ---- compaction in index order ----
    // warp w owns [w*per_w, min((w+1)*per_w, cnt)), per_w a multiple of 32
    const int per_w = (int)(((cnt + 32 * 32 - 1) / (32 * 32)) * 32);
    const int w0 = warp * per_w, w1 = min(w0 + per_w, cnt);
    uint32_t gt = 0, eq = 0;
    for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        uint32_t key = 0;
        if (i < w1) key = CACHED ? keys[i] : float_key(srow[s0 + i]);
        gt += __popc(__ballot_sync(0xffffffffu, key > T));
        eq += __popc(__ballot_sync(0xffffffffu, key == T));
    }
    uint32_t* wgt = misc + 72;        // [32]
    uint32_t* weq = misc + 72 + 32;   // [32]
    if (lane == 0) {
        wgt[warp] = gt;
        weq[warp] = eq;
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t a = wgt[lane], e = weq[lane];
        uint32_t ia = a, ie = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
            const uint32_t ye = __shfl_up_sync(0xffffffffu, ie, o);
            if (lane >= o) {
                ia += ya;
                ie += ye;
            }
        }
        wgt[lane] = ia - a;  // exclusive
        weq[lane] = ie - e;
        if (lane == 31) {
            misc[66] = ia;  // CTA total > T
            misc[67] = ie;  // CTA total == T
        }
    }
    cluster.sync();
    uint32_t cta_gt = 0, cta_eq = 0;
    for (int r = 0; r < rank; ++r) {
        const uint32_t* m = cluster.map_shared_rank(misc, r);
        cta_gt += m[66];
        cta_eq += m[67];
    }
    uint32_t gt_before = cta_gt + wgt[warp];
    uint32_t eq_before = cta_eq + weq[warp];
    int32_t* out = sel + (int64_t)row * k;
    const uint32_t lower = (1u << lane) - 1u;
    for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        uint32_t key = 0;
        if (i < w1) key = CACHED ? keys[i] : float_key(srow[s0 + i]);
        const bool g = key > T, e = key == T;
        const uint32_t mg = __ballot_sync(0xffffffffu, g);
        const uint32_t me = __ballot_sync(0xffffffffu, e);
        const uint32_t my_gt = gt_before + __popc(mg & lower);
        const uint32_t my_eq = eq_before + __popc(me & lower);
        if (g || (e && my_eq < krem)) out[my_gt + min(my_eq, krem)] = s0 + i;
        gt_before += __popc(mg);
        eq_before += __popc(me);
    }
    cluster.sync();  // keep misc alive until every CTA has read it
}

struct TopkPlan {
    int cluster;
    int slice;
    bool cached;
    size_t smem;
};

static TopkPlan plan_topk(int rows, int tokens) {
    TopkPlan p;
    int c = 1;
    while (c < 8 && ((int64_t)rows * c < 2 * 148 || ceil_div(tokens, c) > kTkMaxCached)) c *= 2;
    while (c > 1 && tokens / c < 2048) c /= 2;
    p.cluster = c;
    p.slice = (int)(ceil_div(ceil_div(tokens, c), 32) * 32);
    p.cached = p.slice <= kTkMaxCached;
    p.smem = (size_t)(3 * kTkBins + kTkMisc) * 4 + (p.cached ? (size_t)p.slice * 4 : 0);
    return p;
}

size_t topk_workspace(int rows, int tokens, int k) {
    (void)rows;
    (void)tokens;
    (void)k;
    return 0;
}

template <bool CACHED>
static int launch_topk_impl(const TopkPlan& p, const float* scores, int rows, int tokens,
                            int64_t ld, int k, int32_t* sel, cudaStream_t st) {
    auto kern = topk_kernel<CACHED>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.cluster, rows, 1);
    cfg.blockDim = dim3(kTkThreads, 1, 1);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, scores, tokens, ld, k, p.slice, sel);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

int topk_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel,
                  cudaStream_t st) {
    const TopkPlan p = plan_topk(rows, tokens);
    if (p.cached) return launch_topk_impl<true>(p, scores, rows, tokens, ld, k, sel, st);
    return launch_topk_impl<false>(p, scores, rows, tokens, ld, k, sel, st);
}

}  // namespace fier_cuda
