// attn_tc.cuh -- the per-warp tensor-core decode-attention stream shared by
// attention_tc.cu (K4 / K0 launches) and step_fused.cu (the fused decode step).
//
// A warp streams rows [wr0, wr1) of one (sequence, kv head) through a private
// NST-stage ring of 16-row stages (cp.async 16-byte chunks, XOR-swizzled by row
// so ldmatrix is conflict-free).  Decode has 1..8 query rows per kv head, so they
// sit in the N = 8 dimension of mma.m16n8k16 and the 16 tokens / 16 channels in M:
//   S^T[tok][h] = sum_c K[tok][c] q[h][c]     8 mma per stage: A = K via ldmatrix,
//                                             B = q (column h = query head h)
//   online softmax per head column in fp32 (log2 domain)
//   O^T[c][h]  += sum_tok V^T[c][tok] P^T[tok][h]
//                                             D/16 mma pairs per stage: A = V^T via
//                                             ldmatrix.trans, B = P^T split into
//                                             16-bit hi + lo parts (~2^-16 relative)
// P^T's B fragments are the transpose of S^T's accumulator layout: 8 shuffles.
// Versus q-rows-in-M this halves the mma count and keeps O in D/16 x 4 registers
// with every column usable (the fused step needs the registers).
// This is gather_attention's inner loop (reference core.hpp:165-177) with the
// softmax of core.hpp:115-130 done online.
#pragma once

#include "mma.cuh"

namespace fier_cuda {

constexpr int kTcRows = 16;  // rows per stage

__device__ __forceinline__ void cp_async16_tc(uint32_t smem, const void* gmem) {
#if !defined(FIER_NO_EVICT_FIRST) && !defined(FIER_NO_EVICT_FIRST_KV)
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem), "l"(gmem), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(gmem) : "memory");
#endif
}

// byte offset of 16-byte chunk c of row r inside a stage buffer (rows of RB bytes)
template <int RB>
__device__ __forceinline__ uint32_t swz(int r, int c) {
    return (uint32_t)(r * RB + ((c ^ (r & 7)) << 4));
}

template <int D>
__host__ __device__ constexpr int tc_stage_bytes() {
    return kTcRows * D * 2;  // one K (or V) stage
}

// B fragments of q^T: column n = query head qbase + n (columns >= HPG zero).
template <typename T, int D, int HPG>
__device__ __forceinline__ void tc_load_q(const T* qbase, uint32_t (&qb)[D / 16][2]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
        qb[ks][0] = qb[ks][1] = 0u;
        if (g < HPG) {
            const T* qp = qbase + (int64_t)g * D + ks * 16 + 2 * t;
            qb[ks][0] = *reinterpret_cast<const uint32_t*>(qp);
            qb[ks][1] = *reinterpret_cast<const uint32_t*>(qp + 8);
        }
    }
}

// The same from an fp32 copy of the query heads in shared memory (e.g. after RoPE),
// rounded to T the way a T query would be stored.
template <typename T, int D, int HPG>
__device__ __forceinline__ void tc_load_q_f32(const float* qf, uint32_t (&qb)[D / 16][2]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
        qb[ks][0] = qb[ks][1] = 0u;
        if (g < HPG) {
            const float* qp = qf + g * D + ks * 16 + 2 * t;
            qb[ks][0] = pack2<T>(qp[0], qp[1]);
            qb[ks][1] = pack2<T>(qp[8], qp[9]);
        }
    }
}

// Per-warp attention state: o[mt] = O^T fragment of channels 16mt..16mt+15
// ({c g, h 2t}, {c g, h 2t+1}, {c g+8, h 2t}, {c g+8, h 2t+1}); m[e] / l[e] =
// running max (log2 domain) / partial sum of head 2t+e over this lane's tokens.
template <int D>
struct TcState {
    float o[D / 16][4];
    float m[2], l[2];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int i = 0; i < D / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
        m[0] = m[1] = -INFINITY;
        l[0] = l[1] = 0.f;
    }
};

// Stream granules sg = 0, 1, ... of up to kTcRows rows through the ring at shared
// address `ring` (NST * 2 * tc_stage_bytes<D>() bytes): gran(sg, r0) returns the row
// count of granule sg and its first row r0 (<= 0: the stream has ended; monotone; called
// in order, the loads one stage ahead of the math, so it may wait for rows to appear).
// GATHER: tok_of(r) = token of row r; else row r = token r.
// On return st.l holds the full per-head sums (reduced over the lane's column group).
template <typename T, int D, bool GATHER, int NST, typename Gran, typename TokOf>
__device__ __forceinline__ void tc_stream_granules(const uint32_t (&qb)[D / 16][2], const T* Kseq, const T* Vseq,
                                                   uint32_t ring, float scale_log2, Gran&& gran, TokOf&& tok_of,
                                                   TcState<D>& st) {
    constexpr int RB = D * 2;              // bytes per row
    constexpr int CPR = RB / 16;           // 16-byte chunks per row
    constexpr int KSTEPS = D / 16;         // mma k-steps over channels (S) = m-tiles over channels (PV)
    constexpr int STAGE = tc_stage_bytes<D>();
    constexpr int CPL = kTcRows * CPR / 32;  // chunks per lane per K (or V) stage
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;

    auto issue = [&](int sg) {
        int r0 = 0;
        const int nr = gran(sg, r0);
        if (nr > 0) {
            const uint32_t kdst = ring + (uint32_t)(sg % NST) * 2 * STAGE;
            const uint32_t vdst = kdst + STAGE;
            // rows past the end of a short granule repeat its last row: finite K/V, p = 0 there
            int tok = 0;
            if constexpr (GATHER) tok = tok_of(r0 + min(lane, nr - 1));
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int chunk = lane + 32 * i;
                const int rr = chunk / CPR, c = chunk % CPR;
                int tk;
                if constexpr (GATHER) {
                    tk = __shfl_sync(0xffffffffu, tok, rr);
                } else {
                    tk = r0 + min(rr, nr - 1);  // contiguous rows (K0)
                }
                const uint32_t off = swz<RB>(rr, c);
                cp_async16_tc(kdst + off, Kseq + (int64_t)tk * D + c * 8);
                cp_async16_tc(vdst + off, Vseq + (int64_t)tk * D + c * 8);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

#pragma unroll
    for (int i = 0; i < NST - 1; ++i) issue(i);

    // ldmatrix row addresses: lane L feeds row (L & 7) of matrix L >> 3
    const int krow = (lane & 7) + 8 * ((lane >> 3) & 1), kcol = lane >> 4;  // S: A = K (tok, chunk)
    const int vrow = (lane & 7) + 8 * (lane >> 4), vcol = (lane >> 3) & 1;  // PV: A = V^T via .trans
    // P^T transpose sources: token 2t (+1) of head g lives in lane 4*(2t (+1)) + g/2, register g&1 (+2)
    const int src0 = 8 * t + (g >> 1), src1 = src0 + 4;
    const bool odd = g & 1;

    for (int sg = 0;; ++sg) {
        int r0 = 0;
        const int nr = gran(sg, r0);
        if (nr <= 0) break;
        issue(sg + NST - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
        __syncwarp();
        const uint32_t kst = ring + (uint32_t)(sg % NST) * 2 * STAGE;
        const uint32_t vst = kst + STAGE;

        // ---- S^T = K q^T: 16 tokens x 8 heads ----
        float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < KSTEPS; ++ks) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(kst + swz<RB>(krow, 2 * ks + kcol), a0, a1, a2, a3);
            mma16816<T>(s, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
        }
        // this lane: tokens g (s0, s1) and g + 8 (s2, s3), heads 2t, 2t + 1
        float x[4];
        x[0] = g < nr ? s[0] * scale_log2 : -INFINITY;
        x[1] = g < nr ? s[1] * scale_log2 : -INFINITY;
        x[2] = g + 8 < nr ? s[2] * scale_log2 : -INFINITY;
        x[3] = g + 8 < nr ? s[3] * scale_log2 : -INFINITY;
        float alpha[2], p[4];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            float mx = fmaxf(x[e], x[2 + e]);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            const float mnew = fmaxf(st.m[e], mx);  // finite: every stage has >= 1 real token
            alpha[e] = exp2f(st.m[e] - mnew);
            p[e] = exp2f(x[e] - mnew);
            p[2 + e] = exp2f(x[2 + e] - mnew);
            st.l[e] = st.l[e] * alpha[e] + (p[e] + p[2 + e]);
            st.m[e] = mnew;
        }
        if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
            for (int mt = 0; mt < KSTEPS; ++mt) {
                st.o[mt][0] *= alpha[0];
                st.o[mt][1] *= alpha[1];
                st.o[mt][2] *= alpha[0];
                st.o[mt][3] *= alpha[1];
            }
        }
        // ---- P^T as B fragments: b0 = (P[2t][g], P[2t+1][g]), b1 = (P[2t+8][g], P[2t+9][g]) ----
        const float e00 = __shfl_sync(0xffffffffu, p[0], src0), e01 = __shfl_sync(0xffffffffu, p[1], src0);
        const float e02 = __shfl_sync(0xffffffffu, p[2], src0), e03 = __shfl_sync(0xffffffffu, p[3], src0);
        const float e10 = __shfl_sync(0xffffffffu, p[0], src1), e11 = __shfl_sync(0xffffffffu, p[1], src1);
        const float e12 = __shfl_sync(0xffffffffu, p[2], src1), e13 = __shfl_sync(0xffffffffu, p[3], src1);
        const float pa = odd ? e01 : e00, pb = odd ? e11 : e10;  // tokens 2t, 2t+1
        const float pc = odd ? e03 : e02, pd = odd ? e13 : e12;  // tokens 2t+8, 2t+9
        const uint32_t bh0 = pack2<T>(pa, pb), bh1 = pack2<T>(pc, pd);
        const float2 h0 = unpack2<T>(bh0), h1 = unpack2<T>(bh1);
        const uint32_t bl0 = pack2<T>(pa - h0.x, pb - h0.y), bl1 = pack2<T>(pc - h1.x, pd - h1.y);
        // ---- O^T += V^T P^T: one m-tile of 16 channels per ldmatrix.x4.trans ----
#pragma unroll
        for (int mt = 0; mt < KSTEPS; ++mt) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(vst + swz<RB>(vrow, 2 * mt + vcol), a0, a1, a2, a3);
            mma16816<T>(st.o[mt], a0, a1, a2, a3, bh0, bh1);
            mma16816<T>(st.o[mt], a0, a1, a2, a3, bl0, bl1);
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        st.l[e] += __shfl_xor_sync(0xffffffffu, st.l[e], 4);
        st.l[e] += __shfl_xor_sync(0xffffffffu, st.l[e], 8);
        st.l[e] += __shfl_xor_sync(0xffffffffu, st.l[e], 16);
    }
}

// Rows [wr0, wr1) in granules of kTcRows.
template <typename T, int D, bool GATHER, int NST, typename TokOf>
__device__ __forceinline__ void tc_stream_rows(const uint32_t (&qb)[D / 16][2], const T* Kseq, const T* Vseq,
                                               int wr0, int wr1, uint32_t ring, float scale_log2, TokOf&& tok_of,
                                               TcState<D>& st) {
    tc_stream_granules<T, D, GATHER, NST>(
        qb, Kseq, Vseq, ring, scale_log2,
        [wr0, wr1](int sg, int& r0) {
            r0 = wr0 + sg * kTcRows;
            return min(kTcRows, wr1 - r0);
        },
        tok_of, st);
}

// Warp state -> wr[h][D + 2] (o[0..D), m, l) for heads h < HPG.
template <int D, int HPG>
__device__ __forceinline__ void tc_store_state(const TcState<D>& st, float* wr) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int h = 2 * t + e;
        if (h < HPG) {
            float* w = wr + h * (D + 2);
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {
                w[16 * mt + g] = st.o[mt][e];
                w[16 * mt + g + 8] = st.o[mt][2 + e];
            }
            if (g == 0) {
                w[D] = st.m[e];
                w[D + 1] = st.l[e];
            }
        }
    }
}

}  // namespace fier_cuda
