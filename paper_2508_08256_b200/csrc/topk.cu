// topk.cu -- K3 dispatch: per-head Top-k token selector.
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores,
// ties to the LOWER index, returned in ascending index order.
//
//   many short rows              topk_global.cu  tr_row_kernel: one small CTA per row (C4)
//   millions of keys (workspace) topk_global.cu  wide grid, per-row radix state in global memory
//   rows <= 16 * 512 * 32 keys   topk2.cu      one thread-block cluster per row
//   longer rows (C5, 1M tokens)  topk_long.cu  three streaming passes around a radix threshold
//   anything else                topk_stream_kernel below (exact smem radix select)
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace fier_cuda {

constexpr int kTkRadixBins = 2048;
constexpr int kTkMaxCluster = 8;

// Rows neither topk2 nor topk_long covers: an smem-radix kernel streaming keys from
// global memory each pass (correct for any length; not a fast path).
__global__ void __launch_bounds__(1024, 1)
    topk_stream_kernel(const float* __restrict__ scores, int tokens, int64_t ld, int k, int slice,
                       int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* srow = scores + (int64_t)row * ld;
    const int s0 = rank * slice;
    const int cnt = max(0, min(s0 + slice, tokens) - s0);
    __shared__ uint32_t hist[2][kTkRadixBins];
    __shared__ uint32_t tot[kTkRadixBins];
    __shared__ uint32_t misc[160];
    uint32_t prefix = 0, pmask = 0, krem = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
        const int bins = pass == 2 ? 1024 : 2048;
        uint32_t* h = hist[pass & 1];
        for (int i = tid; i < bins; i += 1024) h[i] = 0;
        __syncthreads();
        for (int i = tid; i < cnt; i += 1024) {
            const uint32_t key = score_key(srow[s0 + i]);
            if ((key & pmask) == prefix) atomicAdd(&h[(key >> shift) & (bins - 1)], 1u);
        }
        cluster.sync();
        for (int i = tid; i < bins; i += 1024) {
            uint32_t a = 0;
            for (int r = 0; r < nct; ++r) a += cluster.map_shared_rank(h, r)[i];
            tot[i] = a;
        }
        __syncthreads();
        if (warp == 0) {
            const int per = bins / 32;
            uint32_t loc = 0;
            for (int j = 0; j < per; ++j) loc += tot[bins - 1 - (lane * per + j)];
            uint32_t inc = loc;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            uint32_t ab = inc - loc;
            for (int j = 0; j < per; ++j) {
                const int bin = bins - 1 - (lane * per + j);
                const uint32_t c = tot[bin];
                if (ab < krem && krem <= ab + c) {
                    misc[64] = (uint32_t)bin;
                    misc[65] = ab;
                }
                ab += c;
            }
        }
        __syncthreads();
        krem -= misc[65];
        prefix |= misc[64] << shift;
        pmask |= (uint32_t)(bins - 1) << shift;
        __syncthreads();
    }
    const uint32_t T = prefix;
    const int per_w = (int)(((cnt + 32 * 32 - 1) / (32 * 32)) * 32);
    const int w0 = warp * per_w, w1 = min(w0 + per_w, cnt);
    uint32_t gt = 0, eq = 0;
    for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const uint32_t key = i < w1 ? score_key(srow[s0 + i]) : 0u;
        gt += __popc(__ballot_sync(0xffffffffu, key > T));
        eq += __popc(__ballot_sync(0xffffffffu, key == T));
    }
    uint32_t* wgt = misc + 72;
    uint32_t* weq = misc + 104;
    if (lane == 0) {
        wgt[warp] = gt;
        weq[warp] = eq;
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t a = wgt[lane], e = weq[lane];
        uint32_t ia = a, ie = e;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
            const uint32_t ye = __shfl_up_sync(0xffffffffu, ie, o);
            if (lane >= o) {
                ia += ya;
                ie += ye;
            }
        }
        wgt[lane] = ia - a;
        weq[lane] = ie - e;
        if (lane == 31) {
            misc[66] = ia;
            misc[67] = ie;
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
        const uint32_t key = i < w1 ? score_key(srow[s0 + i]) : 0u;
        const bool g = key > T, e = key == T;
        const uint32_t mg = __ballot_sync(0xffffffffu, g);
        const uint32_t me = __ballot_sync(0xffffffffu, e);
        const uint32_t my_gt = gt_before + __popc(mg & lower);
        const uint32_t my_eq = eq_before + __popc(me & lower);
        if (g || (e && my_eq < krem)) out[my_gt + min(my_eq, krem)] = s0 + i;
        gt_before += __popc(mg);
        eq_before += __popc(me);
    }
    cluster.sync();
}

size_t topk_global_workspace(int rows, int tokens, int k);
int topk_global_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel,
                         void* workspace, size_t workspace_bytes, cudaStream_t st);

// Workspace of the wide-grid path (topk_global.cu); 0 where it does not apply.
size_t topk_workspace(int rows, int tokens, int k) { return topk_global_workspace(rows, tokens, k); }

template <typename Kern, typename... Args>
static int launch_cluster(Kern kern, int cluster, int rows, int threads, size_t smem, cudaStream_t st,
                          Args... args) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

int topk2_dispatch(const float*, int, int, int64_t, int, int32_t*, cudaStream_t);
int topk_long_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st);

int topk_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st);

// With a workspace of topk_workspace() bytes, rows holding millions of keys take the
// wide-grid radix select (topk_global.cu); otherwise the cluster paths below.
int topk_dispatch_ws(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, void* workspace,
                     size_t workspace_bytes, cudaStream_t st) {
    if ((ld & 3) == 0 && (reinterpret_cast<uintptr_t>(scores) & 15) == 0) {
        const int rc = topk_global_dispatch(scores, rows, tokens, ld, k, sel, workspace, workspace_bytes, st);
        if (rc >= 0) return rc;
    }
    return topk_dispatch(scores, rows, tokens, ld, k, sel, st);
}

int topk_rows_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st);

int topk_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel,
                  cudaStream_t st) {
    int rc = topk_rows_dispatch(scores, rows, tokens, ld, k, sel, st);  // many short rows (C4): a CTA per row
    if (rc >= 0) return rc;
    rc = topk2_dispatch(scores, rows, tokens, ld, k, sel, st);
    if (rc >= 0) return rc;
    rc = topk_long_dispatch(scores, rows, tokens, ld, k, sel, st);  // rows too long for the on-chip path (C5)
    if (rc >= 0) return rc;
    int c = 1;
    while (c < kTkMaxCluster && (int64_t)rows * c < 2 * num_sms()) c *= 2;
    const int64_t slice = ceil_div(tokens, c);
    const int sl = (int)(ceil_div(slice, 32) * 32);
    return launch_cluster(topk_stream_kernel, c, rows, 1024, 0, st, scores, tokens, ld, k, sl, sel);
}

}  // namespace fier_cuda
