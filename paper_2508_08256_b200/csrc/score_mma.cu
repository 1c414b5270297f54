// score_mma.cu -- K2 on the tensor cores for GQA layers: packed-key scoring with the
// sign bits applied to the group scales inside mma.sync operands.
//
// Replaces approx_scores (reference quant1bit.hpp:121-140):
//     s~_t = sum_j q_j (z_gj + sigma_tj s_gj),  sigma = +1 for a set bit, -1 otherwise
//          = bias_g + sum_j q_j (sigma_tj s_gj),  bias_g = sum_j q_j z_gj.
// The second sum is a [tokens x 128] x [128 x heads] product per group with
//   A[t][j] = sigma_tj * s_gj   (fp16: s is the index's binary16 scale, exact)
//   B[j][h] = q_hj * 2^-e_h     (fp16 hi + lo pieces of the query, two columns per head)
// so B is built ONCE per (sequence, kv head) and never per group, and A costs two
// instructions per register: LOP3 flips the signs of the scale pair (s_c, s_{c+16}) of the
// token's channel word with the complemented bits c and c+16 of the packed word shifted to
// positions 15 and 31 (channel pairs (c, c + 16) share a register; the k-slot ->
// channel permutation is applied to B).  Products are exact in the fp32 accumulator; all q
// heads of a GQA group share every packed word (columns of B).
//
// Layout per warp and 32-token slab (one group for g = 32):
//   A: m16n8k16 rows = tokens, lane (r, c) owns channel word c of tokens r, r + 8; per k-step
//      s the registers hold channels 32c + 2s (+16) and 32c + 2s + 1 (+16)
//   B: column 2h + p = piece p (hi, lo) of head h, in registers for the whole sequence
//   D: thread (r, c) holds head c's (hi, lo) sums for tokens r, r + 8 (n-tile 0; heads 4..7
//      in n-tile 1 for 8 heads per group)
// Packed bits and (s, z) stream HBM -> smem through a per-warp ring filled by the bulk-copy
// engine (cp.async.bulk + mbarrier), one stage = one slab.
//
// The decode-step variant fuses the K1 append: before its main loop, CTA c writes the new
// k/v row of sequence c and re-packs that sequence's open group (pack_group), then scores
// the open slabs itself.
#include <algorithm>

#include "pack.cuh"

namespace fier_cuda {

constexpr int kMmaWarps = 8;      // consumer warps per CTA (one slab each per stage)
#ifndef FIER_MMA_STAGES
#define FIER_MMA_STAGES 2
#endif
constexpr int kMmaStages = FIER_MMA_STAGES;  // ring depth
constexpr int kSlabBytes = 32 * 16;  // bits of one 32-token slab (d = 128)
constexpr int kParBytes = 128 * 4;   // (s, z) half2 of one group (d = 128)
// The group's (s, z) row lands contiguously (one bulk copy) and the warp re-lays it out as
// 4 channel words of 128 B at a 144-B stride: the 4 lanes of a quad read words 0..3 at
// the same offset, and the 16-B skew puts those reads in different banks (contiguous, they
// were a 4-way conflict; four 128-B bulk copies cost 45 instructions per slab).
constexpr int kParWordStride = 144;
constexpr int kParStage = 4 * kParWordStride;
// A ring stage holds up to kSps consecutive slabs of one sequence: their bit rows
// (contiguous), their groups' (s, z) rows as copied (contiguous), the skewed copies.  Four
// slabs per stage cut the per-slab cost of the bulk-copy issue and the mbarrier wait
// (~60 of ~310 warp-instructions per slab with one slab per stage).
#ifndef FIER_MMA_SPS
#define FIER_MMA_SPS 4
#endif
constexpr int kSps = FIER_MMA_SPS;
constexpr int kStPar = kSps * kSlabBytes;
constexpr int kStSkew = kStPar + kSps * kParBytes;
constexpr int kStage = kStSkew + kSps * kParStage;

struct AppendArgs2 {  // K == nullptr: no fused append
    void* K;
    void* V;
    const void* k_new;
    const void* v_new;
    int pos;
    int* zero_words;
    int zero_n;
    int rebalance;  // sealed slabs fewer per warp of an appending CTA
    int32_t* nonfinite;  // FIER_NONFINITE_KEY / _QUERY (may be null)
};

// sealed slabs fewer per warp of an appending CTA (C3 sweep, K2: 0 -> 75.3 us,
// 6 -> 71.6 us, 8-12 -> 73.2 us with one slab per ring stage; with four-slab stages, C3 / C4
// step us: 0 72.2 / 478.8, 6 68.64 / 477.9, 12 68.18 / 477.1, 20 68.58 / 477.5)
#ifndef FIER_MMA_REBALANCE
#define FIER_MMA_REBALANCE 12
#endif
constexpr int kMmaRebalance = FIER_MMA_REBALANCE;

__device__ __forceinline__ void mma_f16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float pow2f(int k) { return __int_as_float((k + 127) << 23); }  // -126 <= k <= 127

template <int HPG>
struct SgnTraits {
    static constexpr int NT = (2 * HPG + 7) / 8;  // n-tiles of 8 columns (hi, lo per head)
};

// Per-(sequence, kv head) lane constants.
template <int HPG>
struct LaneConst {
    uint32_t bq[SgnTraits<HPG>::NT][8][2];  // B fragments: column 8 nt + (lane >> 2), k-steps 0..7
    float qz[HPG][4];                       // q of this lane's channels 4 lane .. 4 lane + 3
    float up[HPG];                          // 2^e_h
};

// k-slot kappa (0..15) of k-step s -> channel (the A layout above)
__device__ __forceinline__ int sgn_channel(int s, int kappa) {
    return 32 * ((kappa >> 1) & 3) + 2 * s + (kappa >= 8 ? 1 : 0) + 16 * (kappa & 1);
}

template <typename T, int HPG>
__device__ __forceinline__ void lane_q(const T* qg, LaneConst<HPG>& L) {
    const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
    float mx[HPG];
#pragma unroll
    for (int h = 0; h < HPG; ++h) {
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            L.qz[h][i] = to_f32(qg[h * 128 + 4 * lane + i]);
            m = fmaxf(m, fabsf(L.qz[h][i]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        mx[h] = m;
    }
    float dn[HPG];
#pragma unroll
    for (int h = 0; h < HPG; ++h) {  // |q * 2^-e| < 2^14: the fp16 hi + lo pieces keep 22 bits
        int e = 0;
        if (mx[h] > 0.f && isfinite(mx[h])) {
            frexpf(mx[h], &e);
            e = min(max(e - 14, -126), 127);
        }
        L.up[h] = pow2f(e);
        dn[h] = pow2f(-e);
    }
#pragma unroll
    for (int nt = 0; nt < SgnTraits<HPG>::NT; ++nt) {
        const int col = 8 * nt + g, h = col >> 1, piece = col & 1;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            uint32_t r[2] = {0u, 0u};
            if (h < HPG) {
#pragma unroll
                for (int v = 0; v < 2; ++v) {  // b0: kappa 2c, 2c+1; b1: kappa 2c+8, 2c+9
                    float x[2];
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        float hdn = 0.f;
#pragma unroll
                        for (int hh = 0; hh < HPG; ++hh) hdn = hh == h ? dn[hh] : hdn;
                        const float w = to_f32(qg[h * 128 + sgn_channel(s, 2 * c + 8 * v + e2)]) * hdn;
                        const float hi = __half2float(__float2half_rn(w));
                        x[e2] = piece ? w - hi : hi;
                    }
                    const __half2 hv = __floats2half2_rn(x[0], x[1]);
                    r[v] = *reinterpret_cast<const uint32_t*>(&hv);
                }
            }
            L.bq[nt][s][0] = r[0];
            L.bq[nt][s][1] = r[1];
        }
    }
}

// The warp re-lays the group's (s, z) row (128 half2, read as uint2 u = channels 2u, 2u + 1
// through ld(u)) into par_s: channel word c (channels 32c .. 32c + 31) at c * kParWordStride,
// slot ks = (z-pair, s-pair) of channel 32c + 2ks and of 32c + 2ks + 1, each paired with the
// channel 16 above -- exactly the register quad of the bias pass's A operand (k-step ks),
// so score_slab_mma loads it with one LDS.128 and no byte permutes (4 PRMT per lane here
// instead of 32 in every lane there).
template <typename Ld>
__device__ __forceinline__ void skew_params(uint8_t* par_s, Ld ld) {
    const int lane = threadIdx.x & 31, c = lane >> 3, ks = lane & 7;
    const uint2 lo = ld(16 * c + ks), hi = ld(16 * c + ks + 8);  // channels 32c + 2ks (+1) and + 16
    uint4 o;
    o.x = __byte_perm(lo.x, hi.x, 0x7632);
    o.y = __byte_perm(lo.x, hi.x, 0x5410);
    o.z = __byte_perm(lo.y, hi.y, 0x7632);
    o.w = __byte_perm(lo.y, hi.y, 0x5410);
    reinterpret_cast<uint4*>(par_s + c * kParWordStride)[ks] = o;
}

// Score one 32-token slab.  bits_s: 512 B of token rows (smem), par_s: 512 B of the group's
// (s, z) half2 (smem).  ntok valid tokens.
template <int HPG>
__device__ __forceinline__ void score_slab_mma(const LaneConst<HPG>& L, const uint8_t* bits_s, const uint8_t* par_s,
                                               int t0, int ntok, float* out, int64_t ld) {
    constexpr int NT = SgnTraits<HPG>::NT;
    const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
    // ---- the scale pairs (s_{32c+k}, s_{32c+k+16}) and the offset pairs
    // (z_{32c+k}, z_{32c+k+16}) of this lane's channel word ----
    const uint4* pw = reinterpret_cast<const uint4*>(par_s + c * kParWordStride);  // channels 32c .. 32c + 31
    uint32_t sp[16], zp[16];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {  // paired by skew_params
        const uint4 a = pw[ks];
        zp[2 * ks] = a.x, sp[2 * ks] = a.y, zp[2 * ks + 1] = a.z, sp[2 * ks + 1] = a.w;
    }
    // ---- bias = sum_j q_j z_j through the tensor cores: A rows g = the group's z, so one
    // m-tile pass gives it for all 32 tokens.  Rows g + 8 (d[2], d[3]) are never read: they
    // take the scale pairs, which puts (z, s, z', s') in one register quad without the
    // copies a duplicated z would need (16 moves per slab) ----
    float dz[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) dz[nt][0] = dz[nt][1] = dz[nt][2] = dz[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
            mma_f16(dz[nt], zp[2 * ks], sp[2 * ks], zp[2 * ks + 1], sp[2 * ks + 1], L.bq[nt][ks][0], L.bq[nt][ks][1]);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
        // complemented words: a clear bit flips the (positive) scale to -s
        const uint32_t x0 = ~*reinterpret_cast<const uint32_t*>(bits_s + (mt * 16 + r) * 16 + 4 * c);
        const uint32_t x1 = ~*reinterpret_cast<const uint32_t*>(bits_s + (mt * 16 + r + 8) * 16 + 4 * c);
        float d[NT][4], e[NT][4];  // two accumulator chains (even / odd k-steps): MMA latency
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) d[nt][i] = e[nt][i] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            // channels (2ks, 2ks + 16) and (2ks + 1, 2ks + 17) of the word: bits to 15 / 31
            const uint32_t a0 = sp[2 * ks] ^ ((x0 << (15 - 2 * ks)) & 0x80008000u);
            const uint32_t a1 = sp[2 * ks] ^ ((x1 << (15 - 2 * ks)) & 0x80008000u);
            const uint32_t a2 = sp[2 * ks + 1] ^ ((x0 << (14 - 2 * ks)) & 0x80008000u);
            const uint32_t a3 = sp[2 * ks + 1] ^ ((x1 << (14 - 2 * ks)) & 0x80008000u);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                mma_f16((ks & 1) ? e[nt] : d[nt], a0, a1, a2, a3, L.bq[nt][ks][0], L.bq[nt][ks][1]);
            }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) d[nt][i] += e[nt][i];
        // thread (r, c): head h = 4 nt + c, its (hi, lo) in columns 2c, 2c + 1 of n-tile nt
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int h = 4 * nt + c;
            if (h < HPG) {
                float uh = L.up[0];
#pragma unroll
                for (int hh = 1; hh < HPG; ++hh) uh = h == hh ? L.up[hh] : uh;
                const float bz = dz[nt][0] + dz[nt][1];  // sum_j q'_hj z_j (hi + lo)
                const int ta = mt * 16 + r, tb = ta + 8;
                if (ta < ntok) out[h * ld + t0 + ta] = ((d[nt][0] + d[nt][1]) + bz) * uh;
                if (tb < ntok) out[h * ld + t0 + tb] = ((d[nt][2] + d[nt][3]) + bz) * uh;
            }
        }
    }
}

// ---- the kernel -------------------------------------------------------------------
// Every warp owns a contiguous range of the sealed slabs of all sequences and
// streams it through a private kMmaStages-deep smem ring of kSps-slab stages: lane 0
// issues the two bulk copies (the stage's bit rows, its groups' parameters) of stage
// i + kMmaStages - 1 while the warp scores stage i; completion is an mbarrier per ring
// slot.  No CTA-wide barrier in the main loop.  (A/B, K2 us C4 / C3 / C5: 1 slab x 4
// stages 126.8 / 21.7 / 125.9, 2 x 4 120.9 / 22.4 / 120.3, 2 x 3 120.3 / 21.5 / 119.5,
// 2 x 2 119.8 / 20.9 / -, 4 x 2 113.5 / 21.2 / -; 4 x 2 = 102 KB per CTA, two CTAs per SM.)
template <int HPG>
constexpr size_t mma_smem() {
    return (size_t)kMmaWarps * kMmaStages * kStage + (size_t)kMmaWarps * kMmaStages * 8;
}

template <typename T, int HPG>
__global__ void __launch_bounds__(kMmaWarps * 32, HPG <= 4 ? 2 : 1) score_mma_kernel(const T* __restrict__ q, uint32_t* bits,
                                                                   __half2* sz, int cap, int G, int hkv, int hq,
                                                                   int nseq, int tokens, int lg, float* __restrict__ scores,
                                                                   int64_t ld, AppendArgs2 ap) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = 32 << lg;  // group size, a power of two >= 32 (lg = log2(g / 32))
    uint8_t* ring = smem + (size_t)warp * kMmaStages * kStage;  // [slot] {bits, params}
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kMmaWarps * kMmaStages * kStage) +
                     warp * kMmaStages;
    LaneConst<HPG> L;  // per (sequence, kv head): lane_q

    const int nslabs = (tokens + 31) >> 5;
    // slabs [open0, nslabs) overlap the group re-packed by the fused append
    const int open0 = ap.K ? (((ap.pos >> 5) >> lg) << lg) : nslabs;

    // ---- fused append + open slabs (before the pipeline starts) ----
    if (ap.K) {
        if (ap.zero_words) {  // the fused step's attention-merge counters
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ap.zero_n; i += gridDim.x * blockDim.x)
                ap.zero_words[i] = 0;
        }
        for (int seq = blockIdx.x; seq < nseq; seq += gridDim.x) {
            const int b = seq / hkv, h = seq - b * hkv;
            T* Kseq = static_cast<T*>(ap.K) + (int64_t)seq * cap * 128;
            T* Vseq = static_cast<T*>(ap.V) + (int64_t)seq * cap * 128;
            uint32_t* bseq = bits + (int64_t)seq * cap * 4;
            __half2* zseq = sz + (int64_t)seq * G * 128;
            // token pos comes from k_new; the K/V rows are loaded first and stored after
            // the re-pack, so neither the group's loads nor the stores wait in line
            const bool own = threadIdx.x < 128;
            T kr{}, vr{};
            if (own) {
                kr = static_cast<const T*>(ap.k_new)[(int64_t)seq * 128 + threadIdx.x];
                vr = static_cast<const T*>(ap.v_new)[(int64_t)seq * 128 + threadIdx.x];
            }
            if (ap.nonfinite && threadIdx.x < 32) {  // the query heads of this kv head
                bool bad = false;
                for (int i = threadIdx.x; i < HPG * 128; i += 32)
                    bad |= !isfinite(to_f32(q[((int64_t)b * hq + h * HPG) * 128 + i]));
                if (__any_sync(0xffffffffu, bad) && threadIdx.x == 0) atomicOr(ap.nonfinite, 2);
            }
            // the compact open-group re-pack (pack.cuh), the new row's non-finite check first
            const float xn = own ? to_f32(kr) : 0.f;
            if (ap.nonfinite && threadIdx.x < 128 && __any_sync(0xffffffffu, !isfinite(xn)) &&
                (threadIdx.x & 31) == 0)
                atomicOr(ap.nonfinite, 1);  // "quantize: non-finite key entry" (quant1bit.hpp:68)
            pack_open_group<T>(Kseq, 128, g, ap.pos >> (5 + lg), ap.pos + 1, bseq, zseq, xn, ap.pos);
            if (own) {
                Kseq[(int64_t)ap.pos * 128 + threadIdx.x] = kr;
                Vseq[(int64_t)ap.pos * 128 + threadIdx.x] = vr;
            }
            __syncthreads();
            lane_q<T, HPG>(q + ((int64_t)b * hq + h * HPG) * 128, L);
            for (int slab = open0 + warp; slab < nslabs; slab += kMmaWarps) {
                uint8_t* bs = ring;
                uint8_t* ps = bs + kStSkew;
                const int t0 = slab * 32, ntok = min(32, tokens - t0);
                // coherent (L1-bypassing) reads of what this CTA just wrote
                reinterpret_cast<uint4*>(bs)[lane] =
                    lane < ntok ? __ldcg(reinterpret_cast<const uint4*>(bseq) + t0 + lane) : make_uint4(0, 0, 0, 0);
                const uint4* zrow = reinterpret_cast<const uint4*>(zseq + (int64_t)(slab >> lg) * 128);
                skew_params(ps, [&](int u) { return __ldcg(reinterpret_cast<const uint2*>(zrow) + u); });
                __syncwarp();
                score_slab_mma<HPG>(L, bs, ps, t0, ntok, scores + ((int64_t)b * hq + h * HPG) * ld, ld);
                __syncwarp();
            }
            __syncthreads();
        }
    }

    // ---- this warp's contiguous range of sealed slabs over all sequences ----
    const int64_t total = (int64_t)open0 * nseq;
    const int64_t nwarps = (int64_t)gridDim.x * kMmaWarps;
    const int64_t gw = (int64_t)blockIdx.x * kMmaWarps + warp;
    // The warps of the CTAs that ran the fused append start late: they take `ra` slabs fewer
    // (when every appending CTA appended once, nseq <= gridDim.x).
    const int64_t na = (ap.K && nseq <= (int)gridDim.x) ? (int64_t)nseq * kMmaWarps : 0;
    int64_t per = (total + nwarps - 1) / nwarps, ra = 0;
    if (na > 0) {
        ra = min((int64_t)ap.rebalance, per);
        per = (total + na * ra + nwarps - 1) / nwarps;
        ra = min(ra, per);
    }
    const int64_t w0 = min(total, gw < na ? gw * (per - ra) : na * (per - ra) + (gw - na) * per);
    const int64_t w1 = min(total, w0 + (gw < na ? per - ra : per));
    if (w0 >= w1) return;
    if (lane == 0) {
        for (int s = 0; s < kMmaStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    fence_proxy_async();  // generic-proxy writes to the ring (open slabs) before bulk copies reuse it
    __syncwarp();
    const uint64_t pol = policy_evict_first();
    // Stages: up to kSps consecutive slabs of one sequence.  The issuer (lane 0, kMmaStages - 1
    // stages ahead) and the consumer walk the same (seq, slab, count) sequence.
    const int64_t n = w1 - w0;  // slabs of this warp
    auto stage_len = [&](int slab_, int64_t left) {
        const int c = min(kSps, open0 - slab_);
        return left < (int64_t)c ? (int)left : c;
    };
    int iseq = (int)(w0 / open0), islab = (int)(w0 - (int64_t)iseq * open0);
    int64_t ileft = n;
    auto issue = [&](int slot) {  // lane 0
        const int cnt = stage_len(islab, ileft);
        const int t0 = islab * 32, ntok = min(32 * cnt, tokens - t0);
        const int gfirst = islab >> lg, ng = ((islab + cnt - 1) >> lg) - gfirst + 1;
        uint8_t* dst = ring + (size_t)slot * kStage;
        mbar_arrive_expect_tx(&full[slot], (uint32_t)ntok * 16 + (uint32_t)ng * kParBytes);
        bulk_g2s_evict_first(dst, bits + ((int64_t)iseq * cap + t0) * 4, (uint32_t)ntok * 16, &full[slot], pol);
        bulk_g2s_evict_first(dst + kStPar, sz + ((int64_t)iseq * G + gfirst) * 128, (uint32_t)ng * kParBytes,
                             &full[slot], pol);
        ileft -= cnt;
        if ((islab += cnt) == open0) {
            islab = 0;
            ++iseq;
        }
    };
    if (lane == 0)
        for (int s = 0; s < kMmaStages - 1 && ileft > 0; ++s) issue(s);
    int seq = (int)(w0 / open0), slab = (int)(w0 - (int64_t)seq * open0);
    int b = seq / hkv, h = seq - b * hkv;
    lane_q<T, HPG>(q + ((int64_t)b * hq + h * HPG) * 128, L);
    float* out = scores + ((int64_t)b * hq + h * HPG) * ld;
    int64_t left = n;
    for (int i = 0; left > 0; ++i) {
        const int slot = i % kMmaStages;
        if (lane == 0 && ileft > 0) issue((i + kMmaStages - 1) % kMmaStages);
        mbar_wait(&full[slot], (uint32_t)((i / kMmaStages) & 1));
        uint8_t* stg = ring + (size_t)slot * kStage;
        const int cnt = stage_len(slab, left);
#pragma unroll
        for (int u = 0; u < kSps; ++u) {
            if (u < cnt) {  // skewed, paired copy of the group's (s, z) row (skew_params)
                const uint2* row =
                    reinterpret_cast<const uint2*>(stg + kStPar + (((slab + u) >> lg) - (slab >> lg)) * kParBytes);
                skew_params(stg + kStSkew + u * kParStage, [&](int v) { return row[v]; });
            }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kSps; ++u) {
            if (u < cnt) {
                const int t0 = (slab + u) * 32;
                score_slab_mma<HPG>(L, stg + u * kSlabBytes, stg + kStSkew + u * kParStage, t0, min(32, tokens - t0),
                                    out, ld);
            }
        }
        __syncwarp();  // every lane is done with `slot` before lane 0 refills it
        left -= cnt;
        if ((slab += cnt) == open0 && left > 0) {
            slab = 0;
            ++seq;
            b = seq / hkv;
            h = seq - b * hkv;
            lane_q<T, HPG>(q + ((int64_t)b * hq + h * HPG) * 128, L);
            out = scores + ((int64_t)b * hq + h * HPG) * ld;
        }
    }
}

// ---- host side --------------------------------------------------------------------------
int append_dispatch(const fier_shape*, void*, void*, const void*, const void*, int32_t, uint32_t*, void*, int32_t*,
                    int*, int, cudaStream_t);

template <typename T, int HPG>
static int launch_mma(const fier_shape* s, const void* q, const uint32_t* bits, const void* params, int tokens,
                      float* scores, int64_t ld, const AppendArgs2& ap, cudaStream_t st) {
    auto kern = score_mma_kernel<T, HPG>;
    constexpr size_t smem = mma_smem<HPG>();
    static const int per_sm = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return ctas_per_sm(kern, kMmaWarps * 32, smem);
    }();
    const int G = (int)ceil_div(s->capacity, s->group);
    const int nseq = s->batch * s->kv_heads;
    const int nslabs = (int)ceil_div(tokens, 32);
    const int open0 = ap.K ? ((ap.pos / s->group) * s->group) / 32 : nslabs;
    const int64_t total = (int64_t)open0 * nseq;
    int64_t grid = std::min<int64_t>((int64_t)per_sm * num_sms(), std::max<int64_t>(ceil_div(total, kMmaWarps), 1));
    if (ap.K) grid = std::max<int64_t>(grid, std::min<int64_t>(nseq, (int64_t)per_sm * num_sms()));
    int lg = 0;
    while ((32 << lg) < s->group) ++lg;
    kern<<<(unsigned)grid, kMmaWarps * 32, smem, st>>>(
        static_cast<const T*>(q), const_cast<uint32_t*>(bits), static_cast<__half2*>(const_cast<void*>(params)),
        s->capacity, G, s->kv_heads, s->q_heads, nseq, tokens, lg, scores, ld, ap);
    return check_launch("fier_score (tensor core)");
}

// d = 128, g a power of two >= 32, q_heads / kv_heads in {1, 2, 4, 8}
bool score_mma_ok(const fier_shape* s) {
    const int hpg = s->q_heads / s->kv_heads;
    const bool pow2 = s->group >= 32 && (s->group & (s->group - 1)) == 0;
    return s->dim == 128 && pow2 && (hpg == 1 || hpg == 2 || hpg == 4 || hpg == 8);
}

template <typename T>
static int mma_typed(const fier_shape* s, const void* q, const uint32_t* bits, const void* params, int tokens,
                     float* scores, int64_t ld, const AppendArgs2& ap, cudaStream_t st) {
    switch (s->q_heads / s->kv_heads) {
        case 1: return launch_mma<T, 1>(s, q, bits, params, tokens, scores, ld, ap, st);
        case 2: return launch_mma<T, 2>(s, q, bits, params, tokens, scores, ld, ap, st);
        case 4: return launch_mma<T, 4>(s, q, bits, params, tokens, scores, ld, ap, st);
        default: return launch_mma<T, 8>(s, q, bits, params, tokens, scores, ld, ap, st);
    }
}

int score_mma_dispatch(const fier_shape* s, const void* q, const uint32_t* bits, const void* params, int tokens,
                       float* scores, int64_t ld, void* K, void* V, const void* k_new, const void* v_new, int pos,
                       int* zero_words, int zero_n, int32_t* nonfinite, cudaStream_t st) {
    const AppendArgs2 ap = {K, V, k_new, v_new, pos, zero_words, zero_n, kMmaRebalance, nonfinite};
    switch (s->dtype) {
        case FIER_F32: return mma_typed<float>(s, q, bits, params, tokens, scores, ld, ap, st);
        case FIER_F16: return mma_typed<__half>(s, q, bits, params, tokens, scores, ld, ap, st);
        default: return mma_typed<__nv_bfloat16>(s, q, bits, params, tokens, scores, ld, ap, st);
    }
}

}  // namespace fier_cuda
