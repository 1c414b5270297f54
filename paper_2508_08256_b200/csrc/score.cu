// score.cu -- K2: packed-key importance scorer on CUDA cores (+ the fused
// decode-time append of K1).
//
// Replaces approx_scores (reference quant1bit.hpp:121-140):
//     s~_t = sum_j q_j * ((bit_tj ? s_gj : -s_gj) + z_gj)
// evaluated in the decomposed form
//     s~_t = bias_g + 2 * sum_{j : bit_tj = 1} w_gj,
//     w_gj = q_j * s_gj,   bias_g = sum_j q_j (z_gj - s_gj),
// so per (token, channel) the inner loop is one predicated fp32 add.
//
// Fast path (d = 128, 32 | g): one warp per 32-token slab (lane = token).  The
// slab's group parameters (512 B of half2) are read once per warp, turned into
// the per-head w tables in shared memory (broadcast reads in the inner loop)
// and the bias; each lane streams its token's 16-byte bit row with one
// coalesced 128-bit load and keeps one accumulator set per query head of the
// GQA group, so each packed word is read from HBM once for all Hq/Hkv heads.
// The grid is persistent (exactly the resident CTA count) and warps
// grid-stride over slabs.
//
// Fused append (decode step): CTA 0 of each (sequence, kv head) first writes
// the new k/v row and re-packs the open group [floor(pos/g)*g, pos] (the K1
// append), then scores the open slab(s) itself with coherent loads, while the
// other CTAs score the sealed slabs -- one launch instead of two.
//
// Generic path: any d, any g, one thread per (token, head).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "pack.cuh"

namespace fier_cuda {

constexpr int kScoreWarps = 8;

struct AppendArgs {  // K == nullptr: no fused append
    void* K;
    void* V;
    const void* k_new;
    const void* v_new;
    int pos;
    int* zero_words;
    int zero_n;
    int32_t* nonfinite;  // FIER_NONFINITE_KEY / _QUERY (may be null)
};

// The appending CTA of a (sequence, kv head) flags a non-finite query of its heads
// ("softmax: non-finite logit", core.hpp:122): warp 0's lanes hold every channel.
template <int HPG>
__device__ __forceinline__ void flag_query(const float (&qv)[HPG][4], int32_t* nonfinite) {
    if (!nonfinite || (threadIdx.x >> 5) != 0) return;
    bool bad = false;
#pragma unroll
    for (int hh = 0; hh < HPG; ++hh)
#pragma unroll
        for (int i = 0; i < 4; ++i) bad |= !isfinite(qv[hh][i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 2);
}

__device__ __forceinline__ uint4 ldg_cg(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Score one 32-token slab: p = this lane's 4 (s,z) half2, bw = this lane's bit row.
template <int HPG>
__device__ __forceinline__ void score_slab(const float (&qv)[HPG][4], float4 (*wtab)[32], uint4 p,
                                           uint4 bw, int t, int tokens, float* out, int64_t ld) {
    const int lane = threadIdx.x & 31;
    const __half2* ph = reinterpret_cast<const __half2*>(&p);
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
        wtab[hh][lane] = w;
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
    const uint32_t words[4] = {bw.x, bw.y, bw.z, bw.w};
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
        const uint32_t x = words[wd];
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
#pragma unroll
            for (int hh = 0; hh < HPG; ++hh) {
                const float4 w = wtab[hh][wd * 8 + j4];
                if (x & (1u << (4 * j4 + 0))) acc[hh][0] += w.x;
                if (x & (1u << (4 * j4 + 1))) acc[hh][1] += w.y;
                if (x & (1u << (4 * j4 + 2))) acc[hh][2] += w.z;
                if (x & (1u << (4 * j4 + 3))) acc[hh][3] += w.w;
            }
        }
    }
    if (t < tokens) {
#pragma unroll
        for (int hh = 0; hh < HPG; ++hh) {
            const float a = (acc[hh][0] + acc[hh][1]) + (acc[hh][2] + acc[hh][3]);
            out[hh * ld + t] = bias[hh] + 2.f * a;
        }
    }
    __syncwarp();
}

template <typename T, int HPG>
__global__ void __launch_bounds__(kScoreWarps * 32) score128_kernel(
    const T* __restrict__ q, uint32_t* __restrict__ bits, __half2* __restrict__ sz, int cap, int G,
    int hkv, int hq, int tokens, int g, float* __restrict__ scores, int64_t ld, AppendArgs ap) {
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
    uint32_t* bseq = bits + seq * cap * 4;
    __half2* zseq = sz + seq * G * D;
    const uint4* bits4 = reinterpret_cast<const uint4*>(bseq);
    const uint4* sz4 = reinterpret_cast<const uint4*>(zseq);
    float* out = scores + ((int64_t)b * hq + h * HPG) * ld;

    const int nslabs = (tokens + 31) >> 5;
    // slabs [open0, nslabs) overlap the group re-packed by the fused append
    const int open0 = ap.K ? ((ap.pos / g) * g) >> 5 : nslabs;

    if (ap.K && blockIdx.x == 0) {
        if (ap.zero_words) {  // the fused step's attention-merge counters
            const int per = (ap.zero_n + gridDim.y * gridDim.z - 1) / (gridDim.y * gridDim.z);
            for (int i = threadIdx.x; i < per; i += blockDim.x) {
                const int64_t j = seq * per + i;
                if (j < ap.zero_n) ap.zero_words[j] = 0;
            }
        }
        T* Kseq = static_cast<T*>(ap.K) + seq * cap * D;
        T* Vseq = static_cast<T*>(ap.V) + seq * cap * D;
        // The re-pack takes token pos from k_new; the K/V rows are loaded first and
        // stored after it, so neither the group's loads nor the stores wait in line.
        static_assert(D <= kScoreWarps * 32, "one channel per thread");
        const bool own = threadIdx.x < D;
        T kr{}, vr{};
        if (own) {
            kr = static_cast<const T*>(ap.k_new)[seq * D + threadIdx.x];
            vr = static_cast<const T*>(ap.v_new)[seq * D + threadIdx.x];
        }
        flag_query<HPG>(qv, ap.nonfinite);
        // the compact open-group re-pack of the fused step (pack.cuh): the general pack_group
        // inlined here grew the appending CTA's cold code path (C1 score+append 7.4 -> 9.7 us)
        const float xn = own ? to_f32(kr) : 0.f;
        if (ap.nonfinite && threadIdx.x < 32 * ((D + 31) / 32) &&
            __any_sync(0xffffffffu, own && !isfinite(xn)) && (threadIdx.x & 31) == 0)
            atomicOr(ap.nonfinite, 1);  // "quantize: non-finite key entry" (quant1bit.hpp:68), the new row
        pack_open_group<T>(Kseq, D, g, ap.pos / g, ap.pos + 1, bseq, zseq, xn, ap.pos);
        if (own) {
            Kseq[(int64_t)ap.pos * D + threadIdx.x] = kr;
            Vseq[(int64_t)ap.pos * D + threadIdx.x] = vr;
        }
        __syncthreads();  // the re-packed group is visible to every warp of this CTA
        for (int slab = open0 + warp; slab < nslabs; slab += kScoreWarps) {
            const int t = slab * 32 + lane;
            const uint4 p = ldg_cg(sz4 + (int64_t)((slab * 32) / g) * 32 + lane);
            const uint4 bw = t < tokens ? ldg_cg(bits4 + t) : make_uint4(0, 0, 0, 0);
            score_slab<HPG>(qv, wtab[warp], p, bw, t, tokens, out, ld);
        }
    }

    // With a fused append, CTA 0 (which re-packed and scored the open group) takes no sealed
    // slabs: the launch has one CTA more for them (launch_fast).
    const int skip = (ap.K && gridDim.x > 1) ? 1 : 0;
    if ((int)blockIdx.x < skip) return;
    const int stride = (gridDim.x - skip) * kScoreWarps;
    int slab = (blockIdx.x - skip) * kScoreWarps + warp;
    if (slab >= open0) return;
    // register double buffer: parameters + bit row of the next slab
    uint4 p_cur = sz4[(int64_t)((slab * 32) / g) * 32 + lane];
    uint4 b_cur = make_uint4(0, 0, 0, 0);
    if (slab * 32 + lane < tokens) b_cur = ldg_stream(bits4 + slab * 32 + lane);
    for (; slab < open0; slab += stride) {
        const int nxt = slab + stride;
        uint4 p_nxt = p_cur, b_nxt = make_uint4(0, 0, 0, 0);
        if (nxt < open0) {
            p_nxt = sz4[(int64_t)((nxt * 32) / g) * 32 + lane];
            if (nxt * 32 + lane < tokens) b_nxt = ldg_stream(bits4 + nxt * 32 + lane);
        }
        score_slab<HPG>(qv, wtab[warp], p_cur, b_cur, slab * 32 + lane, tokens, out, ld);
        p_cur = p_nxt;
        b_cur = b_nxt;
    }
}

// Any d, any g: one thread per (token, q head), the reference's own term order.
template <typename T>
__global__ void score_generic_kernel(const T* __restrict__ q, const uint32_t* __restrict__ bits,
                                     const __half2* __restrict__ sz, int cap, int G, int hkv, int hq,
                                     int tokens, int d, int W, int g, float* __restrict__ scores,
                                     int64_t ld, int32_t* nonfinite) {
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
    if (nonfinite && t == 0 && !isfinite(acc)) {  // one thread per q head checks its query
        bool bad = false;
        for (int j = 0; j < d; ++j) bad |= !isfinite(to_f32(qp[j]));
        if (bad) atomicOr(nonfinite, 2);
    }
    scores[((int64_t)b * hq + h) * ld + t] = acc;
}

int append_dispatch(const fier_shape*, void*, void*, const void*, const void*, int32_t, uint32_t*,
                    void*, int32_t*, int*, int, cudaStream_t);

template <typename T, int HPG>
static int launch_fast(const fier_shape* s, const void* q, const uint32_t* bits, const void* params,
                       int tokens, float* scores, int64_t ld, const AppendArgs& ap, cudaStream_t st) {
    const int G = (int)ceil_div(s->capacity, s->group);
    const int nslabs = (int)ceil_div(tokens, 32);
    // persistent: exactly the resident CTA count (no partial last wave)
    static const int per_sm = ctas_per_sm(score128_kernel<T, HPG>, kScoreWarps * 32, 0);
    const int64_t units = (int64_t)s->kv_heads * s->batch;
    int gx = (int)std::max<int64_t>(1, (int64_t)per_sm * num_sms() / units);
    gx = (int)std::min<int64_t>(gx, ceil_div(nslabs, kScoreWarps) + (ap.K ? 1 : 0));
    dim3 grid(gx, s->kv_heads, s->batch);
    score128_kernel<T, HPG><<<grid, kScoreWarps * 32, 0, st>>>(
        static_cast<const T*>(q), const_cast<uint32_t*>(bits),
        static_cast<__half2*>(const_cast<void*>(params)), s->capacity, G, s->kv_heads, s->q_heads, tokens,
        s->group, scores, ld, ap);
    return check_launch("fier_score");
}

bool score_mma_ok(const fier_shape* s);
int score_mma_dispatch(const fier_shape* s, const void* q, const uint32_t* bits, const void* params, int tokens,
                       float* scores, int64_t ld, void* K, void* V, const void* k_new, const void* v_new, int pos,
                       int* zero_words, int zero_n, int32_t* nonfinite, cudaStream_t st);

template <typename T>
static int launch_score(const fier_shape* s, const void* q, const uint32_t* bits, const void* params,
                        int tokens, float* scores, int64_t ld, const AppendArgs& ap, cudaStream_t st) {
    const int hpg = s->q_heads / s->kv_heads;
    // MHA: the CUDA-core kernel is still ahead of the tensor-core one (ncu, profiles/)
    if (score_mma_ok(s) && hpg > 1)
        return score_mma_dispatch(s, q, bits, params, tokens, scores, ld, ap.K, ap.V, ap.k_new, ap.v_new, ap.pos,
                                  ap.zero_words, ap.zero_n, ap.nonfinite, st);
    if (s->dim == 128 && s->group % 32 == 0 && (hpg == 1 || hpg == 2 || hpg == 4 || hpg == 8)) {
        switch (hpg) {
            case 1: return launch_fast<T, 1>(s, q, bits, params, tokens, scores, ld, ap, st);
            case 2: return launch_fast<T, 2>(s, q, bits, params, tokens, scores, ld, ap, st);
            case 4: return launch_fast<T, 4>(s, q, bits, params, tokens, scores, ld, ap, st);
            default: return launch_fast<T, 8>(s, q, bits, params, tokens, scores, ld, ap, st);
        }
    }
    if (ap.K) {  // generic shapes: separate append launch first
        const int rc = append_dispatch(s, ap.K, ap.V, ap.k_new, ap.v_new, ap.pos, const_cast<uint32_t*>(bits),
                                       const_cast<void*>(params), ap.nonfinite, ap.zero_words, ap.zero_n, st);
        if (rc) return rc;
    }
    const int W = (s->dim + 31) / 32;
    const int G = (int)ceil_div(s->capacity, s->group);
    dim3 grid((unsigned)ceil_div(tokens, 128), s->q_heads, s->batch);
    score_generic_kernel<T><<<grid, 128, 0, st>>>(static_cast<const T*>(q), bits,
                                                 static_cast<const __half2*>(params), s->capacity, G,
                                                 s->kv_heads, s->q_heads, tokens, s->dim, W, s->group,
                                                 scores, ld, ap.K ? ap.nonfinite : nullptr);
    return check_launch("fier_score");
}

static int score_typed(const fier_shape* s, const void* q, const uint32_t* bits, const void* params,
                       int tokens, float* scores, int64_t ld, const AppendArgs& ap, cudaStream_t st) {
    switch (s->dtype) {
        case FIER_F32: return launch_score<float>(s, q, bits, params, tokens, scores, ld, ap, st);
        case FIER_F16: return launch_score<__half>(s, q, bits, params, tokens, scores, ld, ap, st);
        case FIER_BF16: return launch_score<__nv_bfloat16>(s, q, bits, params, tokens, scores, ld, ap, st);
    }
    return fail(FIER_EINVAL, "fier_score: unknown dtype");
}

int score_dispatch(const fier_shape* s, const void* q, const uint32_t* bits, const void* params, int tokens,
                   float* scores, int64_t ld, cudaStream_t st) {
    const AppendArgs none = {nullptr, nullptr, nullptr, nullptr, 0, nullptr, 0, nullptr};
    return score_typed(s, q, bits, params, tokens, scores, ld, none, st);
}

// Decode step: append token `pos` (K/V row + open-group re-pack) fused with scoring
// tokens [0, pos] -- zero_words (the attention counters) are cleared on the way.
int append_score_dispatch(const fier_shape* s, const void* q, void* K, void* V, const void* k_new,
                          const void* v_new, int pos, uint32_t* bits, void* params, float* scores,
                          int64_t ld, int* zero_words, int zero_n, int32_t* nonfinite, cudaStream_t st) {
    const AppendArgs ap = {K, V, k_new, v_new, pos, zero_words, zero_n, nonfinite};
    return score_typed(s, q, bits, params, pos + 1, scores, ld, ap, st);
}

}  // namespace fier_cuda
