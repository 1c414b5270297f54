// attention.cu -- K4 sparse decode attention over the selected rows, K0 full-KV
// decode attention (the in-house baseline), and the log-sum-exp merge.
//
// K4 replaces gather_attention (reference core.hpp:152-179) on the Top-k
// selection; K0 is gather_attention over every index (the `full` policy,
// retrieval.hpp:159-166).  Both are split-KV ("flash-decoding"): a CTA owns a
// range of rows of one (sequence, head), each of its 4 warps streams its
// sub-range through a private ring of shared-memory stages filled by the
// bulk-copy engine (cp.async.bulk, one 256-B K row and one V row per copy for
// the gather, one contiguous 8-row block per copy for K0), completion tracked
// by mbarriers.  Per stage of 8 rows: 4 lanes per row compute q.k over d/4
// channels each (fp32), an online softmax in the log2 domain, and lane L
// accumulates p * V over channels [L*d/32, (L+1)*d/32).  The 4 warp states
// are merged in shared memory into one partial (m, l, o[d]) per CTA; the
// merge kernel combines the CTA partials by log-sum-exp.
//
// K0 shares every K/V row across the Hq/Hkv query heads of its GQA group.
#include "common.cuh"

namespace fier_cuda {

constexpr int kAttnWarps = 8;
constexpr int kRowsPerStage = 8;

template <typename T, int D>
struct AttnTraits {
    static constexpr int RB = D * (int)sizeof(T);          // bytes per row
    static constexpr int CH = D / 4;                        // channels per lane (logits)
    static constexpr int EPV = 16 / (int)sizeof(T);         // elements per 16-B vector
    static constexpr int VEC = CH / EPV;                    // 16-B vectors per lane (logits)
    static constexpr int CPL = D / 32;                      // channels per lane (PV)
    static constexpr int STAGE_BYTES = kRowsPerStage * RB;  // per K (or V) stage
};

__device__ __forceinline__ void load_channels(const float* p, float* f, int n) {
    for (int i = 0; i < n; ++i) f[i] = p[i];
}

// PV operand: CPL consecutive channels of a V row in shared memory.
template <typename T, int CPL>
__device__ __forceinline__ void load_v(const T* row, int lane, float* f) {
    if constexpr (sizeof(T) == 4) {
        const float* p = reinterpret_cast<const float*>(row) + lane * CPL;
        if constexpr (CPL == 4) {
            const float4 v = *reinterpret_cast<const float4*>(p);
            f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
        } else {
#pragma unroll
            for (int i = 0; i < CPL; ++i) f[i] = p[i];
        }
    } else {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(row + lane * CPL);
#pragma unroll
        for (int i = 0; i < CPL / 2; ++i) {
            const uint32_t w = p[i];
            if constexpr (std::is_same<T, __nv_bfloat16>::value) {
                f[2 * i] = __uint_as_float(w << 16);
                f[2 * i + 1] = __uint_as_float(w & 0xFFFF0000u);
            } else {
                const float2 x = __half22float2(*reinterpret_cast<const __half2*>(&w));
                f[2 * i] = x.x;
                f[2 * i + 1] = x.y;
            }
        }
    }
}

template <typename T>
__device__ __forceinline__ void unpack_vec(const uint4& v, float* f) {
    if constexpr (sizeof(T) == 4) {
        unpack4(v, f);
    } else {
        unpack8(v, f, static_cast<const T*>(nullptr));
    }
}

// Merge nsplit partials (m, l, o[D]) of `heads` consecutive heads (stride
// nsplit*(D+2)) into out[h][D].  Called by one whole CTA; partials written by
// other CTAs are read with ld.global.cg (L2, not a stale L1).  smem: 2*nsplit floats.
template <int D>
__device__ void merge_partials(const float* part, int nsplit, int heads, float* out, float* smem,
                               float* lse) {
    for (int hh = 0; hh < heads; ++hh) {
        const float* pp = part + (int64_t)hh * nsplit * (D + 2);
        for (int sp = threadIdx.x; sp < nsplit; sp += blockDim.x) {
            smem[sp] = __ldcg(pp + sp * (D + 2) + D);
            smem[nsplit + sp] = __ldcg(pp + sp * (D + 2) + D + 1);
        }
        __syncthreads();
        float M = -INFINITY;
        for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, smem[sp]);
        float L = 0.f;
        for (int sp = 0; sp < nsplit; ++sp)
            if (smem[sp] != -INFINITY) L += smem[nsplit + sp] * exp2f(smem[sp] - M);
        // an empty (ragged) selection gives o = 0 and lse = -inf
        const float inv = L > 0.f ? 1.f / L : 0.f;
        if (lse && threadIdx.x == 0) lse[hh] = L > 0.f ? M + __log2f(L) : -INFINITY;
        for (int c = threadIdx.x; c < D; c += blockDim.x) {
            float o = 0.f;
#pragma unroll 4
            for (int sp = 0; sp < nsplit; ++sp) {
                const float ms = smem[sp];
                const float x = __ldcg(pp + sp * (D + 2) + c);
                if (ms != -INFINITY) o = fmaf(x, exp2f(ms - M), o);
            }
            out[(int64_t)hh * D + c] = o * inv;
        }
        __syncthreads();
    }
}

// (The .L2::cache_hint form of this instruction was miscompiled by ptxas 12.9 for
// sm_100a in one instantiation -- an odd uniform register as the 64-bit policy
// descriptor, trapping as an illegal instruction -- so no hint is used.)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One CTA = kAttnWarps independent warps over rows [r_begin, r_end) of one
// (b, head-set); each warp streams its sub-range through a private NST-stage
// shared-memory ring filled with 16-byte cp.async (every lane copies its share
// of the stage's 8 K rows and 8 V rows; completion by commit/wait groups).
// GATHER: rows are sel[r] of q head `head` (HPG == 1, q kept in registers).
// !GATHER: rows are tokens r of kv head `head`, shared by its HPG query heads.
template <typename T, int D, int HPG, bool GATHER, int NST>
__global__ void __launch_bounds__(kAttnWarps * 32) attn_kernel(
    const T* __restrict__ q, const T* __restrict__ K, const T* __restrict__ V,
    const int32_t* __restrict__ sel, int n, int tokens, int cap, int hkv, int hq, float scale_log2,
    int rows_per_cta, float* __restrict__ part, int nsplit, int* __restrict__ counters,
    float* __restrict__ out, const int32_t* __restrict__ counts, float* __restrict__ lse) {
    using TR = AttnTraits<T, D>;
    constexpr int CH = TR::CH, VEC = TR::VEC, EPV = TR::EPV, CPL = TR::CPL, RB = TR::RB;
    constexpr int QSTRIDE = CH + 4;                 // padded per-part q rows (bank spread)
    constexpr int CPR = RB / 16;                    // 16-byte chunks per row
    constexpr int CPLANE = kRowsPerStage * CPR / 32;  // chunks per lane per K (or V) stage
    static_assert(CPLANE >= 1 && (kRowsPerStage * CPR) % 32 == 0, "row width");

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem;  // [warp][stage][K|V][8 rows][RB]
    float* qs = reinterpret_cast<float*>(ring + (size_t)kAttnWarps * NST * 2 * TR::STAGE_BYTES);
    float* pbuf = qs + (HPG > 1 ? HPG * 4 * QSTRIDE : 0);  // [warp][HPG][8]
    float* wres = pbuf + kAttnWarps * HPG * kRowsPerStage;  // [warp][HPG][D+2]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
    const int kvh = GATHER ? head / (hq / hkv) : head;
    const int64_t seq = (int64_t)b * hkv + kvh;
    const T* Kseq = K + seq * cap * D;
    const T* Vseq = V + seq * cap * D;
    const int total = GATHER ? (counts ? min(n, counts[(int64_t)b * hq + head]) : n) : tokens;
    const int r_begin = split * rows_per_cta;
    const int r_end = max(r_begin, min(r_begin + rows_per_cta, total));
    const int rpw = (int)((((r_end - r_begin) + kAttnWarps - 1) / kAttnWarps + kRowsPerStage - 1) /
                          kRowsPerStage * kRowsPerStage);
    const int wr0 = min(r_begin + warp * rpw, r_end);
    const int wr1 = min(wr0 + rpw, r_end);
    const int nstages = (wr1 - wr0 + kRowsPerStage - 1) / kRowsPerStage;
    const int32_t* selrow = GATHER ? sel + ((int64_t)b * hq + head) * n : nullptr;
    const int qh0 = GATHER ? head : head * HPG;
    const int row = lane >> 2, prt = lane & 3;

    float qreg[HPG == 1 ? CH : 1];
    if constexpr (HPG == 1) {
        const T* qp = q + ((int64_t)b * hq + qh0) * D + prt * CH;
#pragma unroll
        for (int i = 0; i < CH; ++i) qreg[i] = to_f32(qp[i]);
    } else {
        for (int i = threadIdx.x; i < HPG * D; i += blockDim.x) {
            const int hh = i / D, c = i % D;
            qs[hh * 4 * QSTRIDE + (c / CH) * QSTRIDE + (c % CH)] =
                to_f32(q[((int64_t)b * hq + qh0 + hh) * D + c]);
        }
        __syncthreads();
    }

    uint8_t* wring = ring + (size_t)warp * NST * 2 * TR::STAGE_BYTES;
    float* wp = pbuf + warp * HPG * kRowsPerStage;

    auto issue = [&](int st) {  // copy stage st into ring slot st % NST (one commit group)
        if (st < nstages) {
            uint8_t* kdst = wring + (size_t)(st % NST) * 2 * TR::STAGE_BYTES;
            uint8_t* vdst = kdst + TR::STAGE_BYTES;
            const int r0 = wr0 + st * kRowsPerStage;
            const int nr = min(kRowsPerStage, wr1 - r0);
            int tok = 0;
            if constexpr (GATHER) {
                if (lane < nr) tok = __ldg(selrow + r0 + lane);
            }
#pragma unroll
            for (int c = 0; c < CPLANE; ++c) {
                const int chunk = lane + 32 * c;
                const int rr = chunk / CPR, off = chunk % CPR;
                int t;
                if constexpr (GATHER) {
                    t = __shfl_sync(0xffffffffu, tok, rr);
                } else {
                    t = r0 + rr;
                }
                if (rr < nr) {
                    cp_async16(kdst + rr * RB + off * 16, Kseq + (int64_t)t * D + off * (16 / sizeof(T)));
                    cp_async16(vdst + rr * RB + off * 16, Vseq + (int64_t)t * D + off * (16 / sizeof(T)));
                }
            }
        }
        cp_async_commit();
    };

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) issue(s);

    float m[HPG], lloc[HPG], acc[HPG][CPL];
#pragma unroll
    for (int hh = 0; hh < HPG; ++hh) {
        m[hh] = -INFINITY;
        lloc[hh] = 0.f;
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[hh][i] = 0.f;
    }

    for (int st = 0; st < nstages; ++st) {
        issue(st + NST - 1);
        cp_async_wait<NST - 1>();
        __syncwarp();
        const uint8_t* kst = wring + (size_t)(st % NST) * 2 * TR::STAGE_BYTES;
        const uint8_t* vst = kst + TR::STAGE_BYTES;
        const int nr = min(kRowsPerStage, wr1 - (wr0 + st * kRowsPerStage));

        float kf[CH];
        {
            const uint4* kp = reinterpret_cast<const uint4*>(kst + row * RB + prt * CH * sizeof(T));
#pragma unroll
            for (int v = 0; v < VEC; ++v) unpack_vec<T>(kp[v], kf + v * EPV);
        }
#pragma unroll
        for (int hh = 0; hh < HPG; ++hh) {
            float dot0 = 0.f, dot1 = 0.f;
            if constexpr (HPG == 1) {
#pragma unroll
                for (int i = 0; i < CH; i += 2) {
                    dot0 = fmaf(qreg[i], kf[i], dot0);
                    dot1 = fmaf(qreg[i + 1], kf[i + 1], dot1);
                }
            } else {
                const float* qp = qs + hh * 4 * QSTRIDE + prt * QSTRIDE;
#pragma unroll
                for (int i = 0; i < CH; i += 4) {
                    const float4 qq = *reinterpret_cast<const float4*>(qp + i);
                    dot0 = fmaf(qq.x, kf[i], dot0);
                    dot1 = fmaf(qq.y, kf[i + 1], dot1);
                    dot0 = fmaf(qq.z, kf[i + 2], dot0);
                    dot1 = fmaf(qq.w, kf[i + 3], dot1);
                }
            }
            float dot = dot0 + dot1;
            dot += __shfl_xor_sync(0xffffffffu, dot, 1);
            dot += __shfl_xor_sync(0xffffffffu, dot, 2);
            const float logit = row < nr ? dot * scale_log2 : -INFINITY;
            float mst = fmaxf(logit, __shfl_xor_sync(0xffffffffu, logit, 4));
            mst = fmaxf(mst, __shfl_xor_sync(0xffffffffu, mst, 8));
            mst = fmaxf(mst, __shfl_xor_sync(0xffffffffu, mst, 16));
            const float mnew = fmaxf(m[hh], mst);
            const float alpha = exp2f(m[hh] - mnew);
            const float p = exp2f(logit - mnew);
            lloc[hh] = lloc[hh] * alpha + (prt == 0 ? p : 0.f);
            m[hh] = mnew;
#pragma unroll
            for (int i = 0; i < CPL; ++i) acc[hh][i] *= alpha;
            if (prt == 0) wp[hh * kRowsPerStage + row] = p;
        }
        __syncwarp();
#pragma unroll
        for (int hh = 0; hh < HPG; ++hh) {
            const float4 pa = *reinterpret_cast<const float4*>(wp + hh * kRowsPerStage);
            const float4 pb = *reinterpret_cast<const float4*>(wp + hh * kRowsPerStage + 4);
            const float pr[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
            for (int r = 0; r < kRowsPerStage; ++r) {
                if (r < nr) {
                    float vf[CPL];
                    load_v<T, CPL>(reinterpret_cast<const T*>(vst + r * RB), lane, vf);
#pragma unroll
                    for (int i = 0; i < CPL; ++i) acc[hh][i] = fmaf(pr[r], vf[i], acc[hh][i]);
                }
            }
        }
        __syncwarp();
    }
    cp_async_wait<0>();

    // warp states -> smem -> CTA partial
    float* wr = wres + warp * HPG * (D + 2);
#pragma unroll
    for (int hh = 0; hh < HPG; ++hh) {
        const float l = warp_sum(lloc[hh]);
#pragma unroll
        for (int i = 0; i < CPL; ++i) wr[hh * (D + 2) + lane * CPL + i] = acc[hh][i];
        if (lane == 0) {
            wr[hh * (D + 2) + D] = m[hh];
            wr[hh * (D + 2) + D + 1] = l;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HPG * D; i += blockDim.x) {
        const int hh = i / D, c = i % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, wres[(w * HPG + hh) * (D + 2) + D]);
        float o = 0.f, L = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) {
            const float* x = wres + (w * HPG + hh) * (D + 2);
            const float mw = x[D];
            const float sc = mw == -INFINITY ? 0.f : exp2f(mw - M);
            o = fmaf(x[c], sc, o);
            L = fmaf(x[D + 1], sc, L);
        }
        float* dst = part + (((int64_t)b * hq + qh0 + hh) * nsplit + split) * (D + 2);
        dst[c] = o;
        if (c == 0) {
            dst[D] = M;
            dst[D + 1] = L;
        }
    }
    // The last CTA of this (b, head-set) merges the nsplit partials by
    // log-sum-exp (threadFenceReduction pattern) and resets its counter, so
    // the counters stay zero between calls (and CUDA-graph replays).
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int unit = b * (GATHER ? hq : hkv) + head;
        s_last = atomicAdd(&counters[unit], 1) == nsplit - 1;
        if (s_last) counters[unit] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    merge_partials<D>(part + ((int64_t)b * hq + qh0) * nsplit * (D + 2), nsplit, HPG,
                      out + ((int64_t)b * hq + qh0) * D, wres, lse ? lse + (int64_t)b * hq + qh0 : nullptr);
}

// LSE merge of nsplit partials per (b, q head): out = sum_s o_s 2^(m_s-M) / sum_s l_s 2^(m_s-M).
__global__ void merge_kernel(const float* __restrict__ part, int nsplit, int d, int hq,
                             float* __restrict__ out, float* __restrict__ lse) {
    const int h = blockIdx.x, b = blockIdx.y;
    const float* p = part + ((int64_t)b * hq + h) * nsplit * (d + 2);
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, p[s * (d + 2) + d]);
    float L = 0.f;
    for (int s = 0; s < nsplit; ++s) {
        const float ms = p[s * (d + 2) + d];
        if (ms != -INFINITY) L += p[s * (d + 2) + d + 1] * exp2f(ms - M);
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    if (lse && threadIdx.x == 0) lse[(int64_t)b * hq + h] = L > 0.f ? M + __log2f(L) : -INFINITY;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float o = 0.f;
        for (int s = 0; s < nsplit; ++s) {
            const float ms = p[s * (d + 2) + d];
            if (ms != -INFINITY) o = fmaf(p[s * (d + 2) + c], exp2f(ms - M), o);
        }
        out[((int64_t)b * hq + h) * d + c] = o * inv;
    }
}

// Generic fallback (any d <= 1024, any row width): one warp per (b, q head,
// split), lanes over channels, same online softmax.
template <typename T, bool GATHER>
__global__ void attn_generic_kernel(const T* __restrict__ q, const T* __restrict__ K,
                                    const T* __restrict__ V, const int32_t* __restrict__ sel, int n,
                                    int tokens, int cap, int d, int hkv, int hq, float scale_log2,
                                    int rows_per_cta, float* __restrict__ part, int nsplit,
                                    const int32_t* __restrict__ counts) {
    const int lane = threadIdx.x;
    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (hq / hkv);
    const int64_t seq = (int64_t)b * hkv + kvh;
    const T* qp = q + ((int64_t)b * hq + h) * d;
    const int total = GATHER ? (counts ? min(n, counts[(int64_t)b * hq + h]) : n) : tokens;
    const int r0 = split * rows_per_cta, r1 = min(r0 + rows_per_cta, total);
    constexpr int MAXC = 32;  // d <= 1024
    float acc[MAXC];
    for (int i = 0; i < MAXC; ++i) acc[i] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int r = r0; r < r1; ++r) {
        const int tok = GATHER ? sel[((int64_t)b * hq + h) * n + r] : r;
        const T* kr = K + (seq * cap + tok) * d;
        const T* vr = V + (seq * cap + tok) * d;
        float dot = 0.f;
        for (int c = lane; c < d; c += 32) dot = fmaf(to_f32(qp[c]), to_f32(kr[c]), dot);
        const float logit = warp_sum(dot) * scale_log2;
        const float mnew = fmaxf(m, logit);
        const float alpha = exp2f(m - mnew), p = exp2f(logit - mnew);
        l = l * alpha + p;
        m = mnew;
        for (int i = 0, c = lane; c < d; ++i, c += 32) acc[i] = acc[i] * alpha + p * to_f32(vr[c]);
    }
    float* dst = part + (((int64_t)b * hq + h) * nsplit + split) * (d + 2);
    for (int i = 0, c = lane; c < d; ++i, c += 32) dst[c] = acc[i];
    if (lane == 0) {
        dst[d] = m;
        dst[d + 1] = l;
    }
}

// ---- host-side planning --------------------------------------------------------

struct AttnPlan {
    int nsplit;
    int rows_per_cta;
};

// Split rows so the whole grid is one wave of resident CTAs (per_sm per SM).
static AttnPlan plan_split(int64_t units, int total_rows, int min_rows, int per_sm) {
    const int64_t target = (int64_t)per_sm * num_sms();
    int64_t ns = target / units;
    if (ns < 1) ns = 1;
    int rpc = (int)ceil_div(total_rows, ns);
    rpc = (int)ceil_div(rpc, 32) * 32;
    if (rpc < min_rows) rpc = min_rows;
    AttnPlan p;
    p.rows_per_cta = rpc;
    p.nsplit = (int)ceil_div(total_rows, rpc);
    if (p.nsplit < 1) p.nsplit = 1;
    return p;
}

template <typename T, int D>
constexpr int attn_nst() {
    return sizeof(T) == 4 ? 2 : 3;
}

template <typename T, int D, int HPG, bool GATHER>
static size_t attn_smem() {
    using TR = AttnTraits<T, D>;
    constexpr int NST = attn_nst<T, D>();
    return (size_t)kAttnWarps * NST * 2 * TR::STAGE_BYTES + (HPG > 1 ? (size_t)HPG * 4 * (TR::CH + 4) * 4 : 0) +
           (size_t)kAttnWarps * HPG * kRowsPerStage * 4 + (size_t)kAttnWarps * HPG * (D + 2) * 4;
}

template <typename T, int D, int HPG, bool GATHER>
static int launch_attn(const fier_shape* s, const void* q, const void* K, const void* V,
                       const int32_t* sel, int n, int tokens, float scale, float* part,
                       int* counters, float* out, const AttnPlan& p, cudaStream_t st,
                       const int32_t* counts = nullptr, float* lse = nullptr) {
    constexpr int NST = attn_nst<T, D>();
    auto kern = attn_kernel<T, D, HPG, GATHER, NST>;
    const size_t smem = attn_smem<T, D, HPG, GATHER>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("attention: ") + cudaGetErrorString(e));
    dim3 grid(p.nsplit, GATHER ? s->q_heads : s->kv_heads, s->batch);
    kern<<<grid, kAttnWarps * 32, smem, st>>>(
        static_cast<const T*>(q), static_cast<const T*>(K), static_cast<const T*>(V), sel, n, tokens,
        s->capacity, s->kv_heads, s->q_heads, scale * kLog2e, p.rows_per_cta, part, p.nsplit,
        counters, out, counts, lse);
    return check_launch("attention");
}

template <typename T, bool GATHER>
static int launch_generic(const fier_shape* s, const void* q, const void* K, const void* V,
                          const int32_t* sel, int n, int tokens, float scale, float* part,
                          const AttnPlan& p, cudaStream_t st, const int32_t* counts = nullptr) {
    dim3 grid(p.nsplit, s->q_heads, s->batch);
    attn_generic_kernel<T, GATHER><<<grid, 32, 0, st>>>(
        static_cast<const T*>(q), static_cast<const T*>(K), static_cast<const T*>(V), sel, n, tokens,
        s->capacity, s->dim, s->kv_heads, s->q_heads, scale * kLog2e, p.rows_per_cta, part,
        p.nsplit, counts);
    return check_launch("attention");
}

static bool fast_dim(const fier_shape* s) {
    return s->dim == 128 || s->dim == 64;
}

static bool fast_hpg(const fier_shape* s) {
    const int hpg = s->q_heads / s->kv_heads;
    return hpg == 1 || hpg == 2 || hpg == 4 || hpg == 8;
}

constexpr int kMaxSplit = 256;  // the merging CTA keeps 2*nsplit floats in its smem

template <typename T, int D, int HPG, bool GATHER>
static int attn_per_sm() {
    static const int v = [] {
        auto kern = attn_kernel<T, D, HPG, GATHER, attn_nst<T, D>()>;
        const size_t smem = attn_smem<T, D, HPG, GATHER>();
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return ctas_per_sm(kern, kAttnWarps * 32, smem);
    }();
    return v;
}

template <typename T>
static int per_sm_typed(const fier_shape* s, bool gather) {
    const int hpg = s->q_heads / s->kv_heads;
    if (s->dim == 128) {
        if (gather) return attn_per_sm<T, 128, 1, true>();
        return hpg == 1 ? attn_per_sm<T, 128, 1, false>() : hpg == 2 ? attn_per_sm<T, 128, 2, false>()
             : hpg == 4 ? attn_per_sm<T, 128, 4, false>() : attn_per_sm<T, 128, 8, false>();
    }
    if (s->dim == 64) {
        if (gather) return attn_per_sm<T, 64, 1, true>();
        return hpg == 1 ? attn_per_sm<T, 64, 1, false>() : hpg == 2 ? attn_per_sm<T, 64, 2, false>()
             : hpg == 4 ? attn_per_sm<T, 64, 4, false>() : attn_per_sm<T, 64, 8, false>();
    }
    return 8;  // generic one-warp kernel
}

int tc_resident(const fier_shape* s, bool gather);
int tc_dispatch(const fier_shape* s, bool gather, const void* q, const void* K, const void* V,
                const int32_t* sel, int n, int tokens, float scale, float* part, int* counters, float* out,
                int nsplit, int rows_per_cta, const int32_t* counts, float* lse, cudaStream_t st);

static int resident_per_sm(const fier_shape* s, bool gather) {
    if (const int tc = tc_resident(s, gather)) return tc;
    // occupancy needs the opt-in smem limit set on the kernel first
    switch (s->dtype) {
        case FIER_F32: return per_sm_typed<float>(s, gather);
        case FIER_F16: return per_sm_typed<__half>(s, gather);
        default: return per_sm_typed<__nv_bfloat16>(s, gather);
    }
}

AttnPlan sparse_plan(const fier_shape* s, int n) {
    AttnPlan p = plan_split((int64_t)s->batch * s->q_heads, n, 64, resident_per_sm(s, true));
    if (p.nsplit > kMaxSplit) {
        p.rows_per_cta = (int)ceil_div(ceil_div(n, kMaxSplit), 32) * 32;
        p.nsplit = (int)ceil_div(n, p.rows_per_cta);
    }
    if (p.rows_per_cta > 2048) {  // the tensor-core kernel stages <= 2048 indices per CTA
        p.rows_per_cta = 2048;
        p.nsplit = (int)ceil_div(n, p.rows_per_cta);
    }
    return p;
}

AttnPlan full_plan(const fier_shape* s, int tokens) {
    const bool fast = fast_dim(s) && fast_hpg(s);
    const int64_t units = fast ? (int64_t)s->batch * s->kv_heads : (int64_t)s->batch * s->q_heads;
    AttnPlan p = plan_split(units, tokens, 256, resident_per_sm(s, false));
    if (p.nsplit > kMaxSplit) {
        p.rows_per_cta = (int)ceil_div(ceil_div(tokens, kMaxSplit), 32) * 32;
        p.nsplit = (int)ceil_div(tokens, p.rows_per_cta);
    }
    return p;
}

// workspace: [partials f32 B*Hq*nsplit*(d+2)][counters i32 B*Hq] (counters zeroed per call)
static size_t part_bytes(const fier_shape* s, int nsplit) {
    return (((size_t)s->batch * s->q_heads * nsplit * (s->dim + 2) * sizeof(float)) + 255) & ~(size_t)255;
}

size_t sparse_workspace(const fier_shape* s, int n) {
    return part_bytes(s, sparse_plan(s, n).nsplit) + (size_t)s->batch * s->q_heads * sizeof(int);
}

size_t full_workspace(const fier_shape* s, int tokens) {
    return part_bytes(s, full_plan(s, tokens).nsplit) + (size_t)s->batch * s->q_heads * sizeof(int);
}

template <typename T>
static int sparse_typed(const fier_shape* s, const void* q, const void* K, const void* V,
                        const int32_t* sel, int n, int tokens, float scale, float* part, int* ctr,
                        float* out, const AttnPlan& p, cudaStream_t st, const int32_t* counts, float* lse) {
    if (s->dim == 128)
        return launch_attn<T, 128, 1, true>(s, q, K, V, sel, n, tokens, scale, part, ctr, out, p, st, counts, lse);
    if (s->dim == 64)
        return launch_attn<T, 64, 1, true>(s, q, K, V, sel, n, tokens, scale, part, ctr, out, p, st, counts, lse);
    return launch_generic<T, true>(s, q, K, V, sel, n, tokens, scale, part, p, st, counts);
}

template <typename T, int D>
static int full_fast(const fier_shape* s, const void* q, const void* K, const void* V, int tokens,
                     float scale, float* part, int* ctr, float* out, const AttnPlan& p, cudaStream_t st) {
    switch (s->q_heads / s->kv_heads) {
        case 1: return launch_attn<T, D, 1, false>(s, q, K, V, nullptr, 0, tokens, scale, part, ctr, out, p, st);
        case 2: return launch_attn<T, D, 2, false>(s, q, K, V, nullptr, 0, tokens, scale, part, ctr, out, p, st);
        case 4: return launch_attn<T, D, 4, false>(s, q, K, V, nullptr, 0, tokens, scale, part, ctr, out, p, st);
        default: return launch_attn<T, D, 8, false>(s, q, K, V, nullptr, 0, tokens, scale, part, ctr, out, p, st);
    }
}

template <typename T>
static int full_typed(const fier_shape* s, const void* q, const void* K, const void* V, int tokens,
                      float scale, float* part, int* ctr, float* out, const AttnPlan& p, cudaStream_t st) {
    if (fast_hpg(s) && s->dim == 128) return full_fast<T, 128>(s, q, K, V, tokens, scale, part, ctr, out, p, st);
    if (fast_hpg(s) && s->dim == 64) return full_fast<T, 64>(s, q, K, V, tokens, scale, part, ctr, out, p, st);
    return launch_generic<T, false>(s, q, K, V, nullptr, 0, tokens, scale, part, p, st);
}

static int merge(const fier_shape* s, const float* part, int nsplit, float* out, cudaStream_t st,
                 float* lse = nullptr) {
    dim3 grid(s->q_heads, s->batch);
    merge_kernel<<<grid, 128, 0, st>>>(part, nsplit, s->dim, s->q_heads, out, lse);
    return check_launch("attention merge");
}

// counters_zeroed: the caller guarantees the counter words are zero (the fused
// decode step zeroes them in its append kernel); otherwise a memset node is issued.
int sparse_dispatch(const fier_shape* s, const void* q, const void* K, const void* V,
                    const int32_t* sel, int n, int tokens, float scale, float* out, void* ws,
                    bool counters_zeroed, cudaStream_t st, const int32_t* counts, float* lse) {
    const AttnPlan p = sparse_plan(s, n);
    float* part = static_cast<float*>(ws);
    int* ctr = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + part_bytes(s, p.nsplit));
    const bool fused = fast_dim(s);
    if (fused && !counters_zeroed) {
        cudaError_t e = cudaMemsetAsync(ctr, 0, (size_t)s->batch * s->q_heads * sizeof(int), st);
        if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("gather_attention: ") + cudaGetErrorString(e));
    }
    if (tc_resident(s, true) > 0)
        return tc_dispatch(s, true, q, K, V, sel, n, tokens, scale, part, ctr, out, p.nsplit, p.rows_per_cta,
                           counts, lse, st);
    int rc = FIER_OK;
    switch (s->dtype) {
        case FIER_F32: rc = sparse_typed<float>(s, q, K, V, sel, n, tokens, scale, part, ctr, out, p, st, counts, lse); break;
        case FIER_F16: rc = sparse_typed<__half>(s, q, K, V, sel, n, tokens, scale, part, ctr, out, p, st, counts, lse); break;
        case FIER_BF16: rc = sparse_typed<__nv_bfloat16>(s, q, K, V, sel, n, tokens, scale, part, ctr, out, p, st, counts, lse); break;
        default: return fail(FIER_EINVAL, "fier_sparse_attention: unknown dtype");
    }
    if (rc || fused) return rc;
    return merge(s, part, p.nsplit, out, st, lse);
}

int full_dispatch(const fier_shape* s, const void* q, const void* K, const void* V, int tokens,
                  float scale, float* out, void* ws, cudaStream_t st) {
    const AttnPlan p = full_plan(s, tokens);
    float* part = static_cast<float*>(ws);
    int* ctr = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + part_bytes(s, p.nsplit));
    const bool fused = fast_dim(s) && fast_hpg(s);
    if (fused) {
        cudaError_t e = cudaMemsetAsync(ctr, 0, (size_t)s->batch * s->q_heads * sizeof(int), st);
        if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("gather_attention: ") + cudaGetErrorString(e));
    }
    if (tc_resident(s, false) > 0)
        return tc_dispatch(s, false, q, K, V, nullptr, 0, tokens, scale, part, ctr, out, p.nsplit, p.rows_per_cta,
                           nullptr, nullptr, st);
    int rc = FIER_OK;
    switch (s->dtype) {
        case FIER_F32: rc = full_typed<float>(s, q, K, V, tokens, scale, part, ctr, out, p, st); break;
        case FIER_F16: rc = full_typed<__half>(s, q, K, V, tokens, scale, part, ctr, out, p, st); break;
        case FIER_BF16: rc = full_typed<__nv_bfloat16>(s, q, K, V, tokens, scale, part, ctr, out, p, st); break;
        default: return fail(FIER_EINVAL, "fier_full_attention: unknown dtype");
    }
    if (rc || fused) return rc;
    return merge(s, part, p.nsplit, out, st);
}

// True when the sparse attention merges its CTA partials in-kernel (no merge launch).
bool attn_fused_merge(const fier_shape* s) { return fast_dim(s); }

// Offset of the counter words inside a sparse workspace (for the fused step).
size_t sparse_counter_offset(const fier_shape* s, int n) { return part_bytes(s, sparse_plan(s, n).nsplit); }

}  // namespace fier_cuda
