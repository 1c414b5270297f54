// score.cu -- K2: packed-key importance scorer on CUDA cores.
//
// Replaces approx_scores (reference quant1bit.hpp:121-140):
//     s~_t = sum_j q_j * ((bit_tj ? s_gj : -s_gj) + z_gj)
// evaluated in the decomposed form
//     s~_t = bias_g + 2 * sum_{j : bit_tj = 1} w_gj,
//     w_gj = q_j * s_gj,   bias_g = sum_j q_j z_gj - sum_j q_j s_gj,
// so per (token, channel) the inner loop is one predicated fp32 add.
//
// Fast path (d = 128, 32 | g): one warp per 32-token slab (lane = token).  The
// slab's group parameters (512 B of half2) are read once per warp, turned into
// the per-head w tables in shared memory (broadcast reads in the inner loop)
// and the bias; each lane streams its token's 16-byte bit row with one
// coalesced 128-bit load and keeps one accumulator set per query head of the
// GQA group, so each packed word is read from HBM once for all Hq/Hkv heads.
// Generic path: any d, any g, one thread per (token, head).
#include "common.cuh"

namespace fier_cuda {

constexpr int kScoreWarps = 8;

template <typename T, int HPG>
__global__ void __launch_bounds__(kScoreWarps * 32) score128_kernel(
    const T* __restrict__ q, const uint32_t* __restrict__ bits, const __half2* __restrict__ sz,
    int cap, int G, int hkv, int hq, int tokens, int g, float* __restrict__ scores, int64_t ld) {
    constexpr int D = 128;
    __shared__ float4 wtab[kScoreWarps][HPG][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = blockIdx.y, b = blockIdx.z;
    const int64_t seq = (int64_t)b * hkv + h;

    float qv[HPG][4];
#pragma unroll
    for (int hh = 0; hh < HPG; ++hh) {
        const T* qp = q + ((int64_t)b * hq + h * HPG + hh) * D + 4 * lane;
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[hh][i] = to_f32(qp[i]);
    }
    const uint4* bits4 = reinterpret_cast<const uint4*>(bits + seq * cap * 4);
    const uint4* sz4 = reinterpret_cast<const uint4*>(sz + seq * G * D);
    float* out = scores + ((int64_t)b * hq + h * HPG) * ld;

    const int nslabs = (tokens + 31) >> 5;
    const int stride = gridDim.x * kScoreWarps;
    int slab = blockIdx.x * kScoreWarps + warp;
    if (slab >= nslabs) return;

    // register double buffer: parameters + bit row of the next slab
    uint4 p_cur = sz4[(int64_t)((slab * 32) / g) * 32 + lane];
    uint4 b_cur = make_uint4(0, 0, 0, 0);
    if (slab * 32 + lane < tokens) b_cur = ldg_stream(bits4 + slab * 32 + lane);

    for (; slab < nslabs; slab += stride) {
        const int nxt = slab + stride;
        uint4 p_nxt = p_cur, b_nxt = make_uint4(0, 0, 0, 0);
        if (nxt < nslabs) {
            p_nxt = sz4[(int64_t)((nxt * 32) / g) * 32 + lane];
            if (nxt * 32 + lane < tokens) b_nxt = ldg_stream(bits4 + nxt * 32 + lane);
        }
        // (s, z) of channels 4*lane .. 4*lane+3
        const __half2* ph = reinterpret_cast<const __half2*>(&p_cur);
        float s[4], z[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(ph[i]);
            s[i] = f.x;
            z[i] = f.y;
        }
        float bias[HPG];
#pragma unroll
        for (int hh = 0; hh < HPG; ++hh) {
            float4 w;
            w.x = qv[hh][0] * s[0];
            w.y = qv[hh][1] * s[1];
            w.z = qv[hh][2] * s[2];
            w.w = qv[hh][3] * s[3];
            wtab[warp][hh][lane] = w;
            // sum_j q_j (z_j - s_j) over this lane's 4 channels, one warp reduction
            float bz = qv[hh][0] * (z[0] - s[0]);
            bz = fmaf(qv[hh][1], z[1] - s[1], bz);
            bz = fmaf(qv[hh][2], z[2] - s[2], bz);
            bz = fmaf(qv[hh][3], z[3] - s[3], bz);
            bias[hh] = warp_sum(bz);
        }
        __syncwarp();

        float acc[HPG][4];
#pragma unroll
        for (int hh = 0; hh < HPG; ++hh)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[hh][i] = 0.f;
        const uint32_t words[4] = {b_cur.x, b_cur.y, b_cur.z, b_cur.w};
#pragma unroll
        for (int wd = 0; wd < 4; ++wd) {
            const uint32_t x = words[wd];
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
#pragma unroll
                for (int hh = 0; hh < HPG; ++hh) {
                    const float4 w = wtab[warp][hh][wd * 8 + j4];
                    if (x & (1u << (4 * j4 + 0))) acc[hh][0] += w.x;
                    if (x & (1u << (4 * j4 + 1))) acc[hh][1] += w.y;
                    if (x & (1u << (4 * j4 + 2))) acc[hh][2] += w.z;
                    if (x & (1u << (4 * j4 + 3))) acc[hh][3] += w.w;
                }
            }
        }
        const int t = slab * 32 + lane;
        if (t < tokens) {
#pragma unroll
            for (int hh = 0; hh < HPG; ++hh) {
                const float a = (acc[hh][0] + acc[hh][1]) + (acc[hh][2] + acc[hh][3]);
                out[hh * ld + t] = bias[hh] + 2.f * a;
            }
        }
        __syncwarp();
        p_cur = p_nxt;
        b_cur = b_nxt;
    }
}

// Any d, any g: one thread per (token, q head), the reference's own term order.
template <typename T>
__global__ void score_generic_kernel(const T* __restrict__ q, const uint32_t* __restrict__ bits,
                                     const __half2* __restrict__ sz, int cap, int G, int hkv, int hq,
                                     int tokens, int d, int W, int g, float* __restrict__ scores,
                                     int64_t ld) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int h = blockIdx.y, b = blockIdx.z;
    if (t >= tokens) return;
    const int kv = h / (hq / hkv);
    const int64_t seq = (int64_t)b * hkv + kv;
    const T* qp = q + ((int64_t)b * hq + h) * d;
    const uint32_t* brow = bits + (seq * cap + t) * W;
    const __half2* prow = sz + (seq * G + t / g) * d;
    float acc = 0.f;
    for (int j = 0; j < d; ++j) {
        const float2 p = __half22float2(prow[j]);
        const bool bit = (brow[j >> 5] >> (j & 31)) & 1u;
        acc += to_f32(qp[j]) * ((bit ? p.x : -p.x) + p.y);
    }
    scores[((int64_t)b * hq + h) * ld + t] = acc;
}

template <typename T, int HPG>
static void launch_fast(const fier_shape* s, const void* q, const uint32_t* bits,
                        const void* params, int tokens, float* scores, int64_t ld, cudaStream_t st) {
    const int G = (int)ceil_div(s->capacity, s->group);
    const int nslabs = (int)ceil_div(tokens, 32);
    // ~4 slabs per warp; enough CTAs to cover 148 SMs several times over
    int gx = (int)ceil_div(nslabs, kScoreWarps * 4);
    const int64_t ctas_per_x = (int64_t)s->kv_heads * s->batch;
    while (gx > 1 && gx * ctas_per_x > 148 * 16) gx = (gx + 1) / 2;
    if (gx < 1) gx = 1;
    dim3 grid(gx, s->kv_heads, s->batch);
    score128_kernel<T, HPG><<<grid, kScoreWarps * 32, 0, st>>>(
        static_cast<const T*>(q), bits, static_cast<const __half2*>(params), s->capacity, G,
        s->kv_heads, s->q_heads, tokens, s->group, scores, ld);
}

template <typename T>
static int launch_score(const fier_shape* s, const void* q, const uint32_t* bits, const void* params,
                        int tokens, float* scores, int64_t ld, cudaStream_t st) {
    const int hpg = s->q_heads / s->kv_heads;
    if (s->dim == 128 && s->group % 32 == 0) {
        switch (hpg) {
            case 1: launch_fast<T, 1>(s, q, bits, params, tokens, scores, ld, st); return check_launch("fier_score");
            case 2: launch_fast<T, 2>(s, q, bits, params, tokens, scores, ld, st); return check_launch("fier_score");
            case 4: launch_fast<T, 4>(s, q, bits, params, tokens, scores, ld, st); return check_launch("fier_score");
            case 8: launch_fast<T, 8>(s, q, bits, params, tokens, scores, ld, st); return check_launch("fier_score");
            default: break;
        }
    }
    const int W = (s->dim + 31) / 32;
    const int G = (int)ceil_div(s->capacity, s->group);
    dim3 grid((unsigned)ceil_div(tokens, 128), s->q_heads, s->batch);
    score_generic_kernel<T><<<grid, 128, 0, st>>>(static_cast<const T*>(q), bits,
                                                 static_cast<const __half2*>(params), s->capacity, G,
                                                 s->kv_heads, s->q_heads, tokens, s->dim, W,
                                                 s->group, scores, ld);
    return check_launch("fier_score");
}

int score_dispatch(const fier_shape* s, const void* q, const uint32_t* bits, const void* params,
                   int tokens, float* scores, int64_t ld, cudaStream_t st) {
    switch (s->dtype) {
        case FIER_F32: return launch_score<float>(s, q, bits, params, tokens, scores, ld, st);
        case FIER_F16: return launch_score<__half>(s, q, bits, params, tokens, scores, ld, st);
        case FIER_BF16: return launch_score<__nv_bfloat16>(s, q, bits, params, tokens, scores, ld, st);
    }
    return fail(FIER_EINVAL, "fier_score: unknown dtype");
}

}  // namespace fier_cuda
