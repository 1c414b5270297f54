// shard.cu -- X1: the sequence-sharded decode step's exchange kernels.
//
// A long context is split into P contiguous token ranges [start_r, end_r) whose
// boundaries are multiples of g, so each shard's packed index is bit-identical
// to the matching slice of the global quantize() (groups never straddle a
// shard, quant1bit.hpp:5-9, 84).  Scores are per token, so a shard's scores
// equal the global ones.  The global Top-n (topk_oracle, core.hpp:134-148:
// score desc, lower index first, ascending output) is recovered from the
// per-shard Top-n candidate lists:
//
//   1. candidates   each shard keeps its local Top-min(n, l_r) (exact, same
//                   tie rule) as (score, global index) padded to n with
//                   (-inf, -1)                              fier_shard_candidates
//   2. exchange     all-gather of the P candidate lists (NCCL, host side)
//   3. merge        the P lists laid side by side are in global-index order
//                   (shard-major, ascending within a shard), so K3 on that
//                   row with k = n applies the reference tie rule globally;
//                   positions are mapped back to global indices, and each
//                   shard takes its own contiguous run    fier_shard_merge
//   4. attention    K4 on the ragged local run -> (o_r, lse_r)
//   5. exchange     all-gather of the partials
//   6. LSE merge    o = sum_r o_r 2^(lse_r - M) / sum_r 2^(lse_r - M)  fier_lse_merge
//
// Global Top-n is a subset of the union of the local Top-n lists (an element
// beaten by n others inside its own shard is beaten globally), so the merge is
// exact, ties included.
#include <cfloat>
#include <climits>

#include "common.cuh"

namespace fier_cuda {

int topk_dispatch(const float*, int, int, int64_t, int, int32_t*, cudaStream_t);

__global__ void shard_candidates_kernel(const float* __restrict__ scores, int64_t ld, const int32_t* __restrict__ sel,
                                        int k, int nc, int start, float* __restrict__ cs, int32_t* __restrict__ ci) {
    const int row = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nc) return;
    float v = -INFINITY;
    int32_t gi = -1;
    if (i < k) {
        const int32_t t = sel[(int64_t)row * k + i];
        v = scores[(int64_t)row * ld + t];
        gi = start + t;
    }
    cs[(int64_t)row * nc + i] = v;
    ci[(int64_t)row * nc + i] = gi;
}

// [P][rows][nc] -> [rows][P*nc]
__global__ void shard_transpose_kernel(const float* __restrict__ cs, int P, int rows, int nc, float* __restrict__ dst) {
    const int row = blockIdx.y;
    const int64_t w = (int64_t)P * nc;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < w; j += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(j / nc), i = (int)(j % nc);
        dst[row * w + j] = cs[((int64_t)p * rows + row) * nc + i];
    }
}

__device__ __forceinline__ int lower_bound(const int32_t* a, int n, int32_t key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void shard_split_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ ci, int P, int rows,
                                   int nc, int n, int rank, int start, int32_t* __restrict__ sel_global,
                                   int32_t* __restrict__ sel_local, int32_t* __restrict__ counts) {
    const int row = blockIdx.x;
    const int32_t* pr = pos + (int64_t)row * n;
    __shared__ int s_lo, s_hi;
    if (threadIdx.x == 0) {
        s_lo = lower_bound(pr, n, rank * nc);
        s_hi = lower_bound(pr, n, (rank + 1) * nc);
        if (counts) counts[row] = s_hi - s_lo;
    }
    __syncthreads();
    const int lo = s_lo, hi = s_hi;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int32_t ps = pr[i];
        const int p = ps / nc;
        const int32_t gi = ci[((int64_t)p * rows + row) * nc + (ps - p * nc)];
        if (sel_global) sel_global[(int64_t)row * n + i] = gi;
        if (sel_local && i >= lo && i < hi) sel_local[(int64_t)row * n + (i - lo)] = gi - start;
    }
}

// lse in the log2 domain of K4 (lse = m + log2 l over scale*log2(e) logits)
__global__ void lse_merge_kernel(const float* __restrict__ outs, const float* __restrict__ lses, int P, int rows,
                                 int d, float* __restrict__ out, float* __restrict__ lse_out) {
    const int row = blockIdx.x;
    float M = -INFINITY;
    for (int p = 0; p < P; ++p) M = fmaxf(M, lses[(int64_t)p * rows + row]);
    float L = 0.f;
    for (int p = 0; p < P; ++p) {
        const float x = lses[(int64_t)p * rows + row];
        if (x != -INFINITY) L += exp2f(x - M);
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    if (lse_out && threadIdx.x == 0) lse_out[row] = L > 0.f ? M + __log2f(L) : -INFINITY;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float o = 0.f;
        for (int p = 0; p < P; ++p) {
            const float x = lses[(int64_t)p * rows + row];
            if (x != -INFINITY) o = fmaf(outs[((int64_t)p * rows + row) * d + c], exp2f(x - M), o);
        }
        out[(int64_t)row * d + c] = o * inv;
    }
}

}  // namespace fier_cuda

using namespace fier_cuda;

extern "C" {

int fier_shard_bounds(int64_t tokens, int32_t shards, int32_t group, int32_t rank, int64_t* start, int64_t* end) {
    FIER_REQUIRE(tokens >= 1 && shards >= 1 && group >= 1, "fier_shard_bounds: invalid arguments");
    FIER_REQUIRE(rank >= 0 && rank < shards, "fier_shard_bounds: rank out of range");
    // whole groups, spread as evenly as possible (the first G % P shards get one more)
    const int64_t G = ceil_div(tokens, group);
    const int64_t base = G / shards, extra = G % shards;
    const int64_t g0 = rank * base + (rank < extra ? rank : extra);
    const int64_t g1 = g0 + base + (rank < extra ? 1 : 0);
    *start = g0 * group < tokens ? g0 * group : tokens;
    *end = g1 * group < tokens ? g1 * group : tokens;
    return FIER_OK;
}

int fier_shard_candidates(const float* scores, int32_t rows, int64_t ld, const int32_t* sel, int32_t k, int32_t nc,
                          int32_t start, float* cand_scores, int32_t* cand_idx, void* stream) {
    FIER_REQUIRE(rows >= 1 && rows <= 65535 && nc >= 1 && k >= 0 && k <= nc, "fier_shard_candidates: invalid sizes");
    FIER_REQUIRE(cand_scores && cand_idx && (k == 0 || (scores && sel)), "fier_shard_candidates: null buffer");
    dim3 grid((unsigned)ceil_div(nc, 256), rows);
    shard_candidates_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(scores, ld, sel, k, nc, start,
                                                                                 cand_scores, cand_idx);
    return check_launch("fier_shard_candidates");
}

size_t fier_shard_merge_workspace(int32_t shards, int32_t rows, int32_t nc, int32_t n) {
    return (((size_t)shards * rows * nc * sizeof(float) + 255) & ~(size_t)255) + (size_t)rows * n * sizeof(int32_t);
}

int fier_shard_merge(const float* cand_scores, const int32_t* cand_idx, int32_t shards, int32_t rows, int32_t nc,
                     int32_t n, int32_t rank, int32_t start, int32_t* sel_global, int32_t* sel_local, int32_t* counts,
                     void* workspace, size_t workspace_bytes, void* stream) {
    FIER_REQUIRE(shards >= 1 && rows >= 1 && rows <= 65535 && nc >= 1, "fier_shard_merge: invalid sizes");
    FIER_REQUIRE((int64_t)shards * nc <= INT_MAX, "fier_shard_merge: candidate row too long");
    FIER_REQUIRE(n >= 1 && n <= nc, "topk_oracle: k out of range");
    FIER_REQUIRE(rank >= 0 && rank < shards, "fier_shard_merge: rank out of range");
    FIER_REQUIRE(cand_scores && cand_idx, "fier_shard_merge: null buffer");
    FIER_REQUIRE(workspace && workspace_bytes >= fier_shard_merge_workspace(shards, rows, nc, n),
                 "fier_shard_merge: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    float* flat = static_cast<float*>(workspace);
    int32_t* pos = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(workspace) +
                                              (((size_t)shards * rows * nc * sizeof(float) + 255) & ~(size_t)255));
    const int64_t w = (int64_t)shards * nc;
    dim3 tg((unsigned)std::min<int64_t>(ceil_div(w, 256), 1024), rows);
    shard_transpose_kernel<<<tg, 256, 0, st>>>(cand_scores, shards, rows, nc, flat);
    if (int rc = check_launch("fier_shard_merge")) return rc;
    if (int rc = topk_dispatch(flat, rows, (int)w, w, n, pos, st)) return rc;
    shard_split_kernel<<<rows, 256, 0, st>>>(pos, cand_idx, shards, rows, nc, n, rank, start, sel_global, sel_local,
                                             counts);
    return check_launch("fier_shard_merge");
}

int fier_lse_merge(const float* outs, const float* lses, int32_t shards, int32_t rows, int32_t dim, float* out,
                   float* lse, void* stream) {
    FIER_REQUIRE(shards >= 1 && rows >= 1 && dim >= 1, "fier_lse_merge: invalid sizes");
    FIER_REQUIRE(outs && lses && out, "fier_lse_merge: null buffer");
    lse_merge_kernel<<<rows, 128, 0, static_cast<cudaStream_t>(stream)>>>(outs, lses, shards, rows, dim, out, lse);
    return check_launch("fier_lse_merge");
}

}  // extern "C"
