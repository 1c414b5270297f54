// quest.cu -- Quest page retrieval on the GPU: page min/max
// summaries, Quest page scores, quantized-Quest page scores from the Fier scorer (K2),
// and the page fill that turns ranked pages into a token selection.
//
// Reference (baselines.hpp):
//   build_page_summaries :34-56   per page, channel-wise min / max of its members
//   quest_page_scores    :60-79   sum_j (or max_j) of max(q_j kmax_j, q_j kmin_j)
//   select_by_page_scores :85-111 rank pages (score desc, index asc), whole pages while
//                                 they fit, then the next page's lowest indices; ascending
//   quest_select_quantized :120-140 page score = mean of the members' approx_scores
// The page scores are evaluated in fp64 (products of fp32-exact inputs are exact) and
// stored as fp32; the ranking is then exact on those fp32 scores: the top pages come
// from K3 (topk_oracle's tie rule IS the page order), and one CTA per row ranks them,
// walks the fill and writes the tokens in index order.
#include <algorithm>
#include <cstdint>
#include <string>

#include "common.cuh"

namespace fier_cuda {

int topk_dispatch(const float*, int, int, int64_t, int, int32_t*, cudaStream_t);

constexpr int kQsPages = 8;         // pages per summaries block
constexpr int kPfMaxPages = 8192;   // pages ranked by one page-fill CTA
constexpr int kPfThreads = 512;

// K [B*Hkv][cap][d] -> kmax / kmin [B*Hkv][P][d] (fp32, exact)
template <typename T>
__global__ void quest_summaries_kernel(const T* __restrict__ K, int cap, int d, int tokens, int L, int P,
                                       float* __restrict__ kmax, float* __restrict__ kmin) {
    const int64_t row = blockIdx.y;
    const T* Kr = K + row * cap * (int64_t)d;
    for (int pp = 0; pp < kQsPages; ++pp) {
        const int p = blockIdx.x * kQsPages + pp;
        if (p >= P) break;
        const int t0 = p * L, t1 = min(t0 + L, tokens);
        for (int j = threadIdx.x; j < d; j += blockDim.x) {
            float mn = to_f32(Kr[(int64_t)t0 * d + j]), mx = mn;
            for (int t = t0 + 1; t < t1; ++t) {
                const float v = to_f32(Kr[(int64_t)t * d + j]);
                mn = v < mn ? v : mn;  // std::min / std::max (first seen on ties, -0 vs +0)
                mx = mx < v ? v : mx;
            }
            kmax[(row * P + p) * d + j] = mx;
            kmin[(row * P + p) * d + j] = mn;
        }
    }
}

// one warp per (q row, page): fp64 terms, warp reduction
template <typename T>
__global__ void quest_scores_kernel(const T* __restrict__ q, const float* __restrict__ kmax,
                                    const float* __restrict__ kmin, int Hq, int hpg, int d, int P, int sum,
                                    float* __restrict__ out, int64_t pld) {
    const int lane = threadIdx.x & 31;
    const int page = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int qrow = blockIdx.y;  // b * Hq + h
    if (page >= P) return;
    const int64_t kvrow = (int64_t)(qrow / Hq) * (Hq / hpg) + (qrow % Hq) / hpg;
    const float* mx = kmax + (kvrow * P + page) * d;
    const float* mn = kmin + (kvrow * P + page) * d;
    const T* qr = q + (int64_t)qrow * d;
    double acc = 0.0, best = -INFINITY;
    for (int j = lane; j < d; j += 32) {
        const double qj = (double)to_f32(qr[j]);
        const double hi = qj * (double)mx[j], lo = qj * (double)mn[j];
        const double term = hi < lo ? lo : hi;
        acc += term;
        best = best < term ? term : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    }
    if (lane == 0) out[(int64_t)qrow * pld + page] = (float)(sum ? acc : best);
}

// quantized Quest: page mean of the estimated scores (token order, fp64)
__global__ void page_mean_kernel(const float* __restrict__ scores, int64_t ld, int tokens, int L, int P,
                                 float* __restrict__ out, int64_t pld) {
    const int row = blockIdx.y;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
        const int t0 = p * L, t1 = min(t0 + L, tokens);
        double acc = 0.0;
        for (int t = t0; t < t1; ++t) acc += (double)scores[(int64_t)row * ld + t];
        out[(int64_t)row * pld + p] = (float)(acc / (double)(t1 - t0));
    }
}

// Block-wide exclusive scan of one value per thread slot (kPfThreads threads).
__device__ __forceinline__ int pf_scan(int v, int* wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < kPfThreads / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kPfThreads / 32) wsum[lane] = w;  // inclusive
    }
    __syncthreads();
    const int r = (warp ? wsum[warp - 1] : 0) + x - v;
    __syncthreads();
    return r;
}

// One CTA per row: the kp top pages (ascending page index, from K3) -> rank by (score
// desc, index asc) -> fill -> tokens ascending.
__global__ void __launch_bounds__(kPfThreads) page_fill_kernel(const float* __restrict__ ps, int64_t pld,
                                                               const int32_t* __restrict__ top, int kp, int tokens,
                                                               int L, int n, int32_t* __restrict__ sel) {
    extern __shared__ uint8_t smem_raw[];
    float* sc = reinterpret_cast<float*>(smem_raw);        // [kp] scores (page-index order)
    int* pg = reinterpret_cast<int*>(sc + kp);              // [kp] page ids
    int* by_rank = pg + kp;                                 // [kp] size of the page at rank r
    int* rank_of = by_rank + kp;                            // [kp]
    __shared__ int wsum[kPfThreads / 32];
    __shared__ int carry;
    const int row = blockIdx.x;
    for (int i = threadIdx.x; i < kp; i += kPfThreads) {
        const int p = top[(int64_t)row * kp + i];
        pg[i] = p;
        sc[i] = ps[(int64_t)row * pld + p];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kp; i += kPfThreads) {  // rank = pages ordered before page i
        const float s = sc[i];
        int r = 0;
        for (int j = 0; j < kp; ++j) r += (sc[j] > s) || (sc[j] == s && j < i);  // pg ascending in j
        rank_of[i] = r;
        by_rank[r] = min(L, tokens - pg[i] * L);
    }
    __syncthreads();
    // prefix of page sizes in rank order (in place: by_rank[r] <- tokens before rank r)
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < kp; base += kPfThreads) {
        const int i = base + threadIdx.x;
        const int v = i < kp ? by_rank[i] : 0;
        const int ex = pf_scan(v, wsum);
        const int c = carry;
        if (i < kp) by_rank[i] = c + ex;
        __syncthreads();
        if (threadIdx.x == kPfThreads - 1) carry = c + ex + v;
        __syncthreads();
    }
    // taken count per page (index order) -> output offsets -> tokens
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < kp; base += kPfThreads) {
        const int i = base + threadIdx.x;
        int take = 0;
        if (i < kp) {
            const int before = by_rank[rank_of[i]];
            take = max(0, min(min(L, tokens - pg[i] * L), n - before));
        }
        const int ex = pf_scan(take, wsum);
        const int c = carry;
        for (int t = 0; t < take; ++t) sel[(int64_t)row * n + c + ex + t] = pg[i] * L + t;
        __syncthreads();
        if (threadIdx.x == kPfThreads - 1) carry = c + ex + take;
        __syncthreads();
    }
}

static int pages_needed(int tokens, int L, int n) {
    const int P = (int)ceil_div(tokens, L);
    return min(P, n / L + 2);  // n/L whole pages + the partial one + the short last page
}

static int launched(const char* what) {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FIER_OK : fail(FIER_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace fier_cuda

using namespace fier_cuda;

extern "C" {

int fier_quest_summaries(const fier_shape* s, const void* K, int32_t tokens, int32_t page_size, float* kmax,
                         float* kmin, void* stream) {
    FIER_REQUIRE(s && K && kmax && kmin, "build_page_summaries: null buffer");
    FIER_REQUIRE(page_size >= 1, "build_page_summaries: page size must be >= 1");
    FIER_REQUIRE(tokens >= 1 && tokens <= s->capacity && s->dim >= 1 && s->batch >= 1 && s->kv_heads >= 1,
                 "build_page_summaries: empty key cache");
    const int P = (int)ceil_div(tokens, page_size), rows = s->batch * s->kv_heads;
    FIER_REQUIRE(rows <= 65535, "build_page_summaries: too many rows");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const dim3 grid((unsigned)ceil_div(P, kQsPages), (unsigned)rows);
    const int threads = min(256, (int)ceil_div(s->dim, 32) * 32);
    if (s->dtype == FIER_BF16)
        quest_summaries_kernel<__nv_bfloat16><<<grid, threads, 0, st>>>(
            static_cast<const __nv_bfloat16*>(K), s->capacity, s->dim, tokens, page_size, P, kmax, kmin);
    else if (s->dtype == FIER_F16)
        quest_summaries_kernel<__half><<<grid, threads, 0, st>>>(static_cast<const __half*>(K), s->capacity, s->dim,
                                                                 tokens, page_size, P, kmax, kmin);
    else
        quest_summaries_kernel<float><<<grid, threads, 0, st>>>(static_cast<const float*>(K), s->capacity, s->dim,
                                                                tokens, page_size, P, kmax, kmin);
    return launched("build_page_summaries");
}

int fier_quest_page_scores(const fier_shape* s, const void* q, const float* kmax, const float* kmin, int32_t tokens,
                           int32_t page_size, int32_t variant, float* page_scores, int64_t pld, void* stream) {
    FIER_REQUIRE(s && q && kmax && kmin && page_scores, "quest_page_scores: null buffer");
    FIER_REQUIRE(page_size >= 1 && tokens >= 1, "quest_page_scores: bad geometry");
    FIER_REQUIRE(s->kv_heads >= 1 && s->q_heads % s->kv_heads == 0, "quest_page_scores: heads do not match");
    const int P = (int)ceil_div(tokens, page_size);
    FIER_REQUIRE(pld >= P, "quest_page_scores: page score stride shorter than the page count");
    const int rows = s->batch * s->q_heads, hpg = s->q_heads / s->kv_heads;
    FIER_REQUIRE(rows <= 65535, "quest_page_scores: too many rows");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const dim3 grid((unsigned)ceil_div(P, 8), (unsigned)rows);
    const int sum = variant != 0;
    if (s->dtype == FIER_BF16)
        quest_scores_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(q), kmax, kmin,
                                                                 s->q_heads, hpg, s->dim, P, sum, page_scores, pld);
    else if (s->dtype == FIER_F16)
        quest_scores_kernel<__half><<<grid, 256, 0, st>>>(static_cast<const __half*>(q), kmax, kmin, s->q_heads, hpg,
                                                          s->dim, P, sum, page_scores, pld);
    else
        quest_scores_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(q), kmax, kmin, s->q_heads, hpg,
                                                         s->dim, P, sum, page_scores, pld);
    return launched("quest_page_scores");
}

int fier_page_mean(const float* scores, int32_t rows, int32_t tokens, int64_t ld, int32_t page_size,
                   float* page_scores, int64_t pld, void* stream) {
    FIER_REQUIRE(scores && page_scores, "quest_select_quantized: null buffer");
    FIER_REQUIRE(page_size >= 1, "quest_select_quantized: page size must be >= 1");
    FIER_REQUIRE(rows >= 1 && rows <= 65535 && tokens >= 1 && ld >= tokens, "quest_select_quantized: bad geometry");
    const int P = (int)ceil_div(tokens, page_size);
    FIER_REQUIRE(pld >= P, "quest_select_quantized: page score stride shorter than the page count");
    const dim3 grid((unsigned)std::min<int64_t>(ceil_div(P, 128), 1024), (unsigned)rows);
    page_mean_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(scores, ld, tokens, page_size, P,
                                                                         page_scores, pld);
    return launched("quest_select_quantized");
}

size_t fier_page_select_workspace(int32_t rows, int32_t tokens, int32_t page_size, int32_t n) {
    if (rows < 1 || tokens < 1 || page_size < 1 || n < 1) return 0;
    return (size_t)rows * pages_needed(tokens, page_size, n) * sizeof(int32_t);
}

int fier_page_select(const float* page_scores, int32_t rows, int32_t tokens, int64_t pld, int32_t page_size,
                     int32_t n, int32_t* sel, void* workspace, size_t workspace_bytes, void* stream) {
    FIER_REQUIRE(page_scores && sel, "page selection: null buffer");
    FIER_REQUIRE(page_size >= 1, "page selection: page size must be >= 1");
    FIER_REQUIRE(n >= 1 && n <= tokens, "page selection: budget out of range");
    FIER_REQUIRE(rows >= 1 && rows <= 65535, "page selection: rows out of range");
    const int P = (int)ceil_div(tokens, page_size);
    FIER_REQUIRE(pld >= P, "page selection: page score stride shorter than the page count");
    const int kp = pages_needed(tokens, page_size, n);
    FIER_REQUIRE(kp <= kPfMaxPages, "page selection: more than 8192 pages to rank per row");
    const size_t need = fier_page_select_workspace(rows, tokens, page_size, n);
    FIER_REQUIRE(workspace && workspace_bytes >= need, "page selection: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t* top = static_cast<int32_t*>(workspace);
    if (int rc = topk_dispatch(page_scores, rows, P, pld, kp, top, st)) return rc;
    const size_t smem = (size_t)kp * 16;
    if (smem > 48 * 1024) {
        static bool attr = [] {
            cudaFuncSetAttribute(page_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPfMaxPages * 16);
            return true;
        }();
        (void)attr;
    }
    page_fill_kernel<<<rows, kPfThreads, smem, st>>>(page_scores, pld, top, kp, tokens, page_size, n, sel);
    return launched("page selection");
}

}  // extern "C"
