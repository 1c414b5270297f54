// attention_tc.cu -- tensor-core decode attention (bf16 / fp16 K, V; d = 64 or 128).
//
// K4 (gather_attention on the Top-k selection, reference core.hpp:152-179) and
// K0 (gather_attention over every index, retrieval.hpp:159-166) for 16-bit
// caches.  Decode attention moves bytes, not flops; the tensor cores are used
// to cut the instruction count per gathered row (~11 vs ~54 on CUDA cores) so
// the SMs keep enough loads in flight.
//
// Each warp owns a sub-range of rows and streams it through a private NST-stage
// ring of 16-row stages (cp.async 16-byte chunks, XOR-swizzled by row so
// ldmatrix is conflict-free).  Per stage:
//   S[m][n]  = sum_k Q[m][k] K[n][k]     16 x mma.m16n8k16 (A = q rows, B = K
//                                         via ldmatrix), m = query heads of the
//                                         GQA group (rows >= HPG are zero)
//   online softmax per query row in fp32 (log2 domain)
//   O[m][c] += sum_n P[m][n] V[n][c]     P split into bf16 hi + lo parts (two
//                                         mma per tile, ~2^-16 relative error),
//                                         B = V via ldmatrix.trans
// Warp states are merged per CTA, CTA partials by log-sum-exp (the last CTA of
// each head merges), exactly like attention.cu.
#include "attn_tc.cuh"

namespace fier_cuda {

constexpr int kTcWarps = 4;

// wres must also hold the 2 * nsplit (<= 2 * 256) merge weights
template <int D, int HPG>
__host__ __device__ constexpr int tc_wres_floats() {
    return kTcWarps * HPG * (D + 2) > 512 ? kTcWarps * HPG * (D + 2) : 512;
}

template <typename T, int D, int HPG, bool GATHER, int NST>
__global__ void __launch_bounds__(kTcWarps * 32) attn_tc_kernel(
    const T* __restrict__ q, const T* __restrict__ K, const T* __restrict__ V,
    const int32_t* __restrict__ sel, int n, int tokens, int cap, int hkv, int hq, float scale_log2,
    int rows_per_cta, float* __restrict__ part, int nsplit, int* __restrict__ counters,
    float* __restrict__ out, const int32_t* __restrict__ counts, float* __restrict__ lse) {
    static_assert(HPG <= 8, "query rows live in mma rows 0..7");
    constexpr int RB = D * 2;              // bytes per row
    constexpr int KSTEPS = D / 16;         // mma k-steps over channels
    constexpr int STAGE = kTcRows * RB;    // bytes per K (or V) stage

    extern __shared__ __align__(128) uint8_t smem[];
    float* wres = reinterpret_cast<float*>(smem + (size_t)kTcWarps * NST * 2 * STAGE);  // [warp][HPG][D+2]
    // the CTA's selected token indices, staged once (keeps index loads off the gather's critical path)
    int32_t* sidx = reinterpret_cast<int32_t*>(wres + tc_wres_floats<D, HPG>());

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
    const int kvh = GATHER ? head / (hq / hkv) : head;
    const int64_t seq = (int64_t)b * hkv + kvh;
    const T* Kseq = K + seq * cap * D;
    const T* Vseq = V + seq * cap * D;
    // ragged selections (sequence-sharded step): row count per (b, q head)
    const int total = GATHER ? (counts ? min(n, counts[(int64_t)b * hq + head]) : n) : tokens;
    const int r_begin = split * rows_per_cta;
    const int r_end = max(r_begin, min(r_begin + rows_per_cta, total));
    const int rpw = (int)((((r_end - r_begin) + kTcWarps - 1) / kTcWarps + kTcRows - 1) / kTcRows * kTcRows);
    const int wr0 = min(r_begin + warp * rpw, r_end);
    const int wr1 = min(wr0 + rpw, r_end);
    const int32_t* selrow = GATHER ? sel + ((int64_t)b * hq + head) * n : nullptr;
    const int qh0 = GATHER ? head : head * HPG;
    if constexpr (GATHER) {
        // one round of (mostly 16-byte) loads; r_begin is a multiple of 32 and n rows are contiguous
        const int cnt = r_end - r_begin;
        const bool vec = ((reinterpret_cast<uintptr_t>(selrow + r_begin) & 15) == 0);
        if (vec) {
            for (int i = threadIdx.x; i < cnt / 4; i += blockDim.x)
                reinterpret_cast<int4*>(sidx)[i] = __ldg(reinterpret_cast<const int4*>(selrow + r_begin) + i);
            for (int i = (cnt & ~3) + threadIdx.x; i < cnt; i += blockDim.x) sidx[i] = __ldg(selrow + r_begin + i);
        } else {
            for (int i = threadIdx.x; i < cnt; i += blockDim.x) sidx[i] = __ldg(selrow + r_begin + i);
        }
        __syncthreads();
    }

    uint32_t qb[KSTEPS][2];
    tc_load_q<T, D, HPG>(q + ((int64_t)b * hq + qh0) * D, qb);
    TcState<D> st;
    st.init();
    const uint32_t ring = smem_u32(smem) + (uint32_t)warp * NST * 2 * STAGE;
    tc_stream_rows<T, D, GATHER, NST>(qb, Kseq, Vseq, wr0, wr1, ring, scale_log2,
                                      [&](int r) { return sidx[r - r_begin]; }, st);

    // ---- warp states -> smem -> CTA partial -> last-CTA merge ----
    tc_store_state<D, HPG>(st, wres + warp * HPG * (D + 2));
    __syncthreads();
    for (int i = threadIdx.x; i < HPG * D; i += blockDim.x) {
        const int hh = i / D, c = i % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kTcWarps; ++w) M = fmaxf(M, wres[(w * HPG + hh) * (D + 2) + D]);
        float oo = 0.f, L = 0.f;
#pragma unroll
        for (int w = 0; w < kTcWarps; ++w) {
            const float* xx = wres + (w * HPG + hh) * (D + 2);
            const float mw = xx[D];
            const float sc = mw == -INFINITY ? 0.f : exp2f(mw - M);
            oo = fmaf(xx[c], sc, oo);
            L = fmaf(xx[D + 1], sc, L);
        }
        float* dst = part + (((int64_t)b * hq + qh0 + hh) * nsplit + split) * (D + 2);
        dst[c] = oo;
        if (c == 0) {
            dst[D] = M;
            dst[D + 1] = L;
        }
    }
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
    // merge nsplit partials of the HPG heads (smem: 2*nsplit floats in wres)
    for (int hh = 0; hh < HPG; ++hh) {
        const float* pp = part + ((int64_t)b * hq + qh0 + hh) * nsplit * (D + 2);
        for (int sp = threadIdx.x; sp < nsplit; sp += blockDim.x) {
            wres[sp] = __ldcg(pp + sp * (D + 2) + D);
            wres[nsplit + sp] = __ldcg(pp + sp * (D + 2) + D + 1);
        }
        __syncthreads();
        float M = -INFINITY;
        for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, wres[sp]);
        float L = 0.f;
        for (int sp = 0; sp < nsplit; ++sp)
            if (wres[sp] != -INFINITY) L += wres[nsplit + sp] * exp2f(wres[sp] - M);
        // an empty (ragged) selection gives o = 0 and lse = -inf
        const float inv = L > 0.f ? 1.f / L : 0.f;
        if (lse && threadIdx.x == 0) lse[(int64_t)b * hq + qh0 + hh] = L > 0.f ? M + __log2f(L) : -INFINITY;
        for (int c = threadIdx.x; c < D; c += blockDim.x) {
            float oo = 0.f;
#pragma unroll 4
            for (int sp = 0; sp < nsplit; ++sp) {
                const float ms = wres[sp];
                const float xv = __ldcg(pp + sp * (D + 2) + c);
                if (ms != -INFINITY) oo = fmaf(xv, exp2f(ms - M), oo);
            }
            out[((int64_t)b * hq + qh0 + hh) * D + c] = oo * inv;
        }
        __syncthreads();
    }
}

// ---- host side -------------------------------------------------------------------

constexpr int kTcMaxRowsPerCta = 2048;  // staged selection indices per CTA (sparse_plan caps rows_per_cta)

template <int D, int HPG>
constexpr size_t tc_smem(int nst) {
    return (size_t)kTcWarps * nst * 2 * kTcRows * D * 2 + (size_t)tc_wres_floats<D, HPG>() * 4 +
           (size_t)kTcMaxRowsPerCta * 4;
}

constexpr int kTcNst = 3;

template <typename T, int D, int HPG, bool GATHER>
int tc_per_sm() {
    static const int v = [] {
        auto kern = attn_tc_kernel<T, D, HPG, GATHER, kTcNst>;
        const size_t smem = tc_smem<D, HPG>(kTcNst);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return ctas_per_sm(kern, kTcWarps * 32, smem);
    }();
    return v;
}

template <typename T, int D, int HPG, bool GATHER>
int launch_attn_tc(const fier_shape* s, const void* q, const void* K, const void* V, const int32_t* sel,
                   int n, int tokens, float scale, float* part, int* counters, float* out, int nsplit,
                   int rows_per_cta, const int32_t* counts, float* lse, cudaStream_t st) {
    auto kern = attn_tc_kernel<T, D, HPG, GATHER, kTcNst>;
    const size_t smem = tc_smem<D, HPG>(kTcNst);
    (void)tc_per_sm<T, D, HPG, GATHER>();  // sets the smem attribute once
    dim3 grid(nsplit, GATHER ? s->q_heads : s->kv_heads, s->batch);
    kern<<<grid, kTcWarps * 32, smem, st>>>(static_cast<const T*>(q), static_cast<const T*>(K),
                                            static_cast<const T*>(V), sel, n, tokens, s->capacity,
                                            s->kv_heads, s->q_heads, scale * kLog2e, rows_per_cta, part,
                                            nsplit, counters, out, counts, lse);
    return check_launch("attention (tensor core)");
}

// resident CTAs per SM for the tensor-core path of this shape (0: not applicable)
int tc_resident(const fier_shape* s, bool gather) {
    const int hpg = gather ? 1 : s->q_heads / s->kv_heads;
    if (s->dtype != FIER_BF16 && s->dtype != FIER_F16) return 0;
    if (s->dim != 128 && s->dim != 64) return 0;
    if (!(hpg == 1 || hpg == 2 || hpg == 4 || hpg == 8)) return 0;
#define TC_CASE(TT, DD)                                                                          \
    switch (hpg) {                                                                               \
        case 1: return gather ? tc_per_sm<TT, DD, 1, true>() : tc_per_sm<TT, DD, 1, false>();    \
        case 2: return tc_per_sm<TT, DD, 2, false>();                                            \
        case 4: return tc_per_sm<TT, DD, 4, false>();                                            \
        default: return tc_per_sm<TT, DD, 8, false>();                                           \
    }
    if (s->dtype == FIER_BF16) {
        if (s->dim == 128) { TC_CASE(__nv_bfloat16, 128) }
        TC_CASE(__nv_bfloat16, 64)
    }
    if (s->dim == 128) { TC_CASE(__half, 128) }
    TC_CASE(__half, 64)
#undef TC_CASE
}

int tc_dispatch(const fier_shape* s, bool gather, const void* q, const void* K, const void* V,
                const int32_t* sel, int n, int tokens, float scale, float* part, int* counters, float* out,
                int nsplit, int rows_per_cta, const int32_t* counts, float* lse, cudaStream_t st) {
    const int hpg = gather ? 1 : s->q_heads / s->kv_heads;
#define TC_LAUNCH(TT, DD)                                                                               \
    switch (hpg) {                                                                                      \
        case 1:                                                                                         \
            return gather ? launch_attn_tc<TT, DD, 1, true>(s, q, K, V, sel, n, tokens, scale, part,    \
                                                            counters, out, nsplit, rows_per_cta, counts, lse, st)    \
                          : launch_attn_tc<TT, DD, 1, false>(s, q, K, V, sel, n, tokens, scale, part,   \
                                                             counters, out, nsplit, rows_per_cta, counts, lse, st);  \
        case 2:                                                                                         \
            return launch_attn_tc<TT, DD, 2, false>(s, q, K, V, sel, n, tokens, scale, part, counters, \
                                                    out, nsplit, rows_per_cta, counts, lse, st);                     \
        case 4:                                                                                         \
            return launch_attn_tc<TT, DD, 4, false>(s, q, K, V, sel, n, tokens, scale, part, counters, \
                                                    out, nsplit, rows_per_cta, counts, lse, st);                     \
        default:                                                                                        \
            return launch_attn_tc<TT, DD, 8, false>(s, q, K, V, sel, n, tokens, scale, part, counters, \
                                                    out, nsplit, rows_per_cta, counts, lse, st);                     \
    }
    if (s->dtype == FIER_BF16) {
        if (s->dim == 128) { TC_LAUNCH(__nv_bfloat16, 128) }
        TC_LAUNCH(__nv_bfloat16, 64)
    }
    if (s->dim == 128) { TC_LAUNCH(__half, 128) }
    TC_LAUNCH(__half, 64)
#undef TC_LAUNCH
}

}  // namespace fier_cuda
