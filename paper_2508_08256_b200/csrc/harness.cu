// harness.cu -- the GPU side of the recall / margin sweep: the
// per-query diagnostics the reference's evaluation harness computes on the CPU, at
// long context on the device.
//
// Reference (evalharness.hpp / core.hpp):
//   exact_scores        core.hpp:98-112        q . k_i in fp64 (optionally / sqrt(d))
//   margin_and_errors   evalharness.hpp:63-83  m = s_(k) - s_(k+1) of the exact scores
//                                              (descending), and over i of err = exact - est:
//                                              max |err|, sum err^2, sum max(0, m/2 - err),
//                                              sum max(0, |err| - m/2)
//   overlap_fraction    evalharness.hpp:40-48  |sel n oracle| / oracle budget (sorted lists)
//   relative_l2_error   core.hpp:181-190
// The order statistics s_(k), s_(k+1) come from K3 (topk over the exact scores, k + 1):
// the smallest selected value is s_(k+1), the second smallest s_(k) (ties by value).
#include <algorithm>
#include <cstdint>
#include <string>

#include "common.cuh"

namespace fier_cuda {

int topk_dispatch(const float*, int, int, int64_t, int, int32_t*, cudaStream_t);

// one warp per token, fp64 products of fp32-exact inputs; rows = B*Hq, GQA kv head h/hpg
template <typename T>
__global__ void exact_scores_kernel(const T* __restrict__ q, const T* __restrict__ K, int Hq, int hpg, int cap,
                                    int d, int tokens, double inv, double* __restrict__ out,
                                    float* __restrict__ out32, int64_t ld) {
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int qrow = blockIdx.y;
    if (t >= tokens) return;
    const int64_t kvrow = (int64_t)(qrow / Hq) * (Hq / hpg) + (qrow % Hq) / hpg;
    const T* k = K + (kvrow * cap + t) * d;
    const T* qr = q + (int64_t)qrow * d;
    double acc = 0.0;
    for (int j = lane; j < d; j += 32) acc += (double)to_f32(qr[j]) * (double)to_f32(k[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        out[(int64_t)qrow * ld + t] = acc * inv;
        if (out32) out32[(int64_t)qrow * ld + t] = (float)(acc * inv);
    }
}

// fp64 keys and query (the reference's own types): one thread per token, the reference's
// sequential channel order with unfused multiply and add (core.hpp:105-109), so the
// scores are the reference's bit for bit
__global__ void exact_scores_f64_kernel(const double* __restrict__ q, const double* __restrict__ K, int Hq, int hpg,
                                        int cap, int d, int tokens, double inv, double* __restrict__ out,
                                        float* __restrict__ out32, int64_t ld) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int qrow = blockIdx.y;
    if (t >= tokens) return;
    const int64_t kvrow = (int64_t)(qrow / Hq) * (Hq / hpg) + (qrow % Hq) / hpg;
    const double* k = K + (kvrow * cap + t) * d;
    const double* qr = q + (int64_t)qrow * d;
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc = __dadd_rn(acc, __dmul_rn(qr[j], k[j]));
    const double v = __dmul_rn(acc, inv);
    out[(int64_t)qrow * ld + t] = v;
    if (out32) out32[(int64_t)qrow * ld + t] = (float)v;
}

// per row: margin from the k+1 largest (sel), then the four error sums (block reduction)
__global__ void margin_errors_kernel(const double* __restrict__ exact, const float* __restrict__ est, int64_t ld,
                                     int tokens, const int32_t* __restrict__ top, int k1,
                                     double* __restrict__ rep) {
    __shared__ double red[4][32];
    __shared__ double sm[2];
    const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* ex = exact + (int64_t)row * ld;
    if (warp == 0) {  // two smallest values among the k+1 largest
        double a = INFINITY, b = INFINITY;  // a <= b
        for (int i = lane; i < k1; i += 32) {
            const double v = ex[top[(int64_t)row * k1 + i]];
            if (v < a) {
                b = a;
                a = v;
            } else if (v < b) {
                b = v;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double a2 = __shfl_xor_sync(0xffffffffu, a, o), b2 = __shfl_xor_sync(0xffffffffu, b, o);
            const double lo = fmin(a, a2), hi = fmin(fmax(a, a2), fmin(b, b2));
            a = lo;
            b = hi;
        }
        if (lane == 0) {
            sm[0] = b - a;  // s_(k) - s_(k+1)
        }
    }
    __syncthreads();
    const double m = sm[0], half_m = m * 0.5;
    double mx = 0.0, l2 = 0.0, h1 = 0.0, h2 = 0.0;
    for (int i = tid; i < tokens; i += blockDim.x) {
        const double err = ex[i] - (double)est[(int64_t)row * ld + i];
        mx = fmax(mx, fabs(err));
        l2 += err * err;
        h1 += fmax(0.0, half_m - err);
        h2 += fmax(0.0, fabs(err) - half_m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        l2 += __shfl_xor_sync(0xffffffffu, l2, o);
        h1 += __shfl_xor_sync(0xffffffffu, h1, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
    }
    if (lane == 0) {
        red[0][warp] = mx;
        red[1][warp] = l2;
        red[2][warp] = h1;
        red[3][warp] = h2;
    }
    __syncthreads();
    if (tid == 0) {
        double r[4] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            r[0] = fmax(r[0], red[0][w]);
            r[1] += red[1][w];
            r[2] += red[2][w];
            r[3] += red[3][w];
        }
        double* o = rep + (int64_t)row * 5;
        o[0] = m;
        o[1] = r[0];
        o[2] = r[1];
        o[3] = r[2];
        o[4] = r[3];
    }
}

// per row: |sel n oracle| / n_oracle for ascending lists (merge by binary search)
__global__ void overlap_kernel(const int32_t* __restrict__ sel, int n, const int32_t* __restrict__ oracle, int no,
                               double* __restrict__ out) {
    __shared__ int cnt;
    const int row = blockIdx.x;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int32_t* o = oracle + (int64_t)row * no;
    int hit = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int32_t v = sel[(int64_t)row * n + i];
        int lo = 0, hi = no;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (o[mid] < v) lo = mid + 1; else hi = mid;
        }
        hit += lo < no && o[lo] == v;
    }
    atomicAdd(&cnt, hit);
    __syncthreads();
    if (threadIdx.x == 0) out[row] = (double)cnt / (double)no;
}

static int launched(const char* what) {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FIER_OK : fail(FIER_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace fier_cuda

using namespace fier_cuda;

extern "C" {

int fier_exact_scores(const fier_shape* s, const void* q, const void* K, int32_t tokens, int32_t scaled,
                      double* scores, float* scores32, int64_t ld, void* stream) {
    FIER_REQUIRE(s && q && K && scores, "exact_scores: null buffer");
    FIER_REQUIRE(s->kv_heads >= 1 && s->q_heads % s->kv_heads == 0 && s->dim >= 1,
                 "exact_scores: query length does not match key dim");
    FIER_REQUIRE(tokens >= 1 && tokens <= s->capacity && ld >= tokens, "exact_scores: bad geometry");
    const int rows = s->batch * s->q_heads, hpg = s->q_heads / s->kv_heads;
    FIER_REQUIRE(rows <= 65535, "exact_scores: too many rows");
    const double inv = scaled ? 1.0 / std::sqrt((double)s->dim) : 1.0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const dim3 grid((unsigned)ceil_div(tokens, 8), (unsigned)rows);
    if (s->dtype == FIER_F64)
        exact_scores_f64_kernel<<<dim3((unsigned)ceil_div(tokens, 128), (unsigned)rows), 128, 0, st>>>(
            static_cast<const double*>(q), static_cast<const double*>(K), s->q_heads, hpg, s->capacity, s->dim,
            tokens, inv, scores, scores32, ld);
    else if (s->dtype == FIER_BF16)
        exact_scores_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(q),
                                                                 static_cast<const __nv_bfloat16*>(K), s->q_heads, hpg,
                                                                 s->capacity, s->dim, tokens, inv, scores, scores32, ld);
    else if (s->dtype == FIER_F16)
        exact_scores_kernel<__half><<<grid, 256, 0, st>>>(static_cast<const __half*>(q), static_cast<const __half*>(K),
                                                          s->q_heads, hpg, s->capacity, s->dim, tokens, inv, scores,
                                                          scores32, ld);
    else
        exact_scores_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(q), static_cast<const float*>(K),
                                                         s->q_heads, hpg, s->capacity, s->dim, tokens, inv, scores,
                                                         scores32, ld);
    return launched("exact_scores");
}

size_t fier_margin_errors_workspace(int32_t rows, int32_t k) {
    return rows >= 1 && k >= 1 ? (size_t)rows * (k + 1) * sizeof(int32_t) : 0;
}

int fier_margin_errors(const double* exact, const float* exact32, const float* est, int32_t rows, int32_t tokens,
                       int64_t ld, int32_t k, double* report, void* workspace, size_t workspace_bytes, void* stream) {
    FIER_REQUIRE(exact && exact32 && est && report, "margin_and_errors: null buffer");
    FIER_REQUIRE(k >= 1 && k < tokens, "margin_and_errors: need 1 <= k < l");
    FIER_REQUIRE(rows >= 1 && rows <= 65535 && ld >= tokens, "margin_and_errors: bad geometry");
    FIER_REQUIRE(workspace && workspace_bytes >= fier_margin_errors_workspace(rows, k),
                 "margin_and_errors: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t* top = static_cast<int32_t*>(workspace);
    // the k+1 largest by the fp32 copy: their fp64 values hold s_(k), s_(k+1) unless two
    // exact scores collide in fp32 (then the fp32 order of equal values is immaterial)
    if (int rc = topk_dispatch(exact32, rows, tokens, ld, k + 1, top, st)) return rc;
    margin_errors_kernel<<<rows, 512, 0, st>>>(exact, est, ld, tokens, top, k + 1, report);
    return launched("margin_and_errors");
}

int fier_overlap(const int32_t* sel, int32_t n, const int32_t* oracle, int32_t no, int32_t rows, double* out,
                 void* stream) {
    FIER_REQUIRE(sel && oracle && out && n >= 1 && no >= 1 && rows >= 1, "overlap_fraction: bad arguments");
    overlap_kernel<<<rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(sel, n, oracle, no, out);
    return launched("overlap_fraction");
}

}  // extern "C"
