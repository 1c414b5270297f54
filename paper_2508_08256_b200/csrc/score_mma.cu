// score_mma.cu -- K2 on the tensor cores: packed-key scoring with the bits fed
// straight into mma.sync as bf16 "exponent-bit" operands.
//
// Replaces approx_scores (reference quant1bit.hpp:121-140):
//     s~_t = sum_j q_j ((bit_tj ? s_gj : -s_gj) + z_gj) = bias_g + 2 sum_j bit_tj w_gj,
//     w_gj = q_j s_gj,  bias_g = sum_j q_j (z_gj - s_gj).
// The sum over bits is a [tokens x 128] x [128 x heads] product per group.
//
// Operand A (tokens x channels) comes from the packed words with ONE LOP3 per
// two elements: a bf16 half-word with a single bit set at position 7+i
// (0 <= i < 8) is the normal number 2^(2^i - 127), so `x & mask` turns two bits
// of a word into two bf16 values {0, 2^e}; a rotate by 8 brings the other 16
// bits of the word into those positions (17 instructions per 32 bits).  The
// per-k-slot factor 2^-e is folded into operand B = w * 2^(-e - sigma), split
// into three bf16 pieces hi + mid + lo (exact for an fp32 w: two pieces leave a
// 2^-17 relative error per term, too coarse when large terms cancel), so every
// product is exactly bit * w * 2^-sigma and the fp32 accumulation sees only
// w-sized terms.  The
// channel permutation this implies (k-slot -> channel, see kslot_channel) is
// applied to B; the sum does not care about channel order.
//
// Layout per warp and 32-token slab (one group for g = 32):
//   A: m16n8k16 rows = tokens, lane (r, c) owns word c of tokens r, r+8 -> 16 regs
//      per 16-token m-tile per k-step pair ... 8 k-steps cover the 128 channels
//   B: columns 2h, 2h+1 = (hi, mid) and column 2*HPG + h = lo of query head h of
//      the GQA group; built once per group by the whole warp (lane = 4 k-slots)
//      into a swizzled smem tile and read back with ldmatrix
//   D: thread (r, c) sums (hi, mid) of head 4*tile + c for tokens r, r + 8 and
//      fetches lo with two shuffles
// Packed bits and (s, z) stream HBM -> smem through a per-CTA ring filled by the
// bulk-copy engine (cp.async.bulk + mbarrier), one stage = one slab per warp.
//
// The decode-step variant fuses the K1 append: before its main loop, CTA c
// writes the new k/v row of sequence c and re-packs that sequence's open group
// (pack_group), then scores the open slabs itself.
#include <algorithm>

#include "pack.cuh"

namespace fier_cuda {

constexpr int kMmaWarps = 8;      // consumer warps per CTA (one slab each per stage)
constexpr int kMmaStages = 4;     // ring depth
constexpr int kSigma = 60;        // B = w * 2^(-e - sigma) stays inside the fp32/bf16 range
constexpr int kSlabBytes = 32 * 16;  // bits of one 32-token slab (d = 128)
constexpr int kParBytes = 128 * 4;   // (s, z) half2 of one group (d = 128)

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
// 6 -> 71.6 us, 8-12 -> 73.2 us)
constexpr int kMmaRebalance = 6;

// k-slot (0..127, = 16 * k-step + k) -> channel and exponent of its A value
__host__ __device__ constexpr int kslot_i(int ks) { return 2 * (ks >> 4) + ((ks & 15) >= 8 ? 1 : 0); }
__host__ __device__ constexpr int kslot_channel(int ks) {
    const int k = ks & 15, h = k & 1, c = (k & 7) >> 1, i = kslot_i(ks);
    const int off = i < 8 ? (h == 0 ? 7 + i : 23 + i) : (h == 0 ? 15 + (i - 8) : (31 + (i - 8)) & 31);
    return 32 * c + off;
}
__host__ __device__ constexpr int kslot_exp(int ks) { return (1 << (kslot_i(ks) & 7)) - 127; }

__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// A register R_i (0..15) of word x: bits (7+i, 23+i) for i < 8, else of rotr(x, 8)
template <int I>
__device__ __forceinline__ uint32_t abits(uint32_t x, uint32_t y) {
    constexpr uint32_t m = (0x80u << (I & 7)) | (0x800000u << (I & 7));
    return (I < 8 ? x : y) & m;
}

// B tile of one warp: [NCOL][128 k-slots] bf16, rows of 256 B, 16-B chunks XOR-swizzled by row
__device__ __forceinline__ uint32_t btile_off(int col, int kslot) {
    return (uint32_t)(col * 256 + ((((kslot >> 3) ^ (col & 7)) & 15) << 4) + (kslot & 7) * 2);
}

template <int HPG>
struct MmaTraits {
    static constexpr int NT = (3 * HPG + 7) / 8;  // n-tiles of 8 columns (hi, mid, lo per head)
    static constexpr int NHM = (2 * HPG + 7) / 8;  // n-tiles holding (hi, mid)
    static constexpr int NCOL = 8 * NT;
    static constexpr int BTILE = NCOL * 256;    // bytes of a warp's B tile
};

// Per-lane constants: q' = q * 2^(-e - sigma) for this lane's 4 k-slots x HPG heads,
// the slot channels and the 2^(e + sigma) factors (for the bias).
template <int HPG>
struct LaneConst {
    float qp[HPG][4];
    int ch[4];
    float up[4];
};

// Score one 32-token slab.  bits_s: 512 B of token rows (smem), par_s: 512 B of the
// group's (s, z) half2 (smem), btile: this warp's B tile (smem).  ntok valid tokens.
template <int HPG>
__device__ __forceinline__ void score_slab_mma(const LaneConst<HPG>& L, const uint8_t* bits_s, const uint8_t* par_s,
                                               uint8_t* btile, int t0, int ntok, float* out, int64_t ld) {
    using TR = MmaTraits<HPG>;
    const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
    // ---- B = w * 2^(-e - sigma) as bf16 hi + lo, and the per-head bias ----
    float bias[HPG];
#pragma unroll
    for (int h = 0; h < HPG; ++h) bias[h] = 0.f;
    {
        float sv[4], dz[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const __half2 p = *reinterpret_cast<const __half2*>(par_s + L.ch[u] * 4);
            const float2 f = __half22float2(p);
            sv[u] = f.x;
            dz[u] = (f.y - f.x) * L.up[u];  // (z - s) * 2^(e + sigma): q' * dz = q (z - s)
        }
#pragma unroll
        for (int h = 0; h < HPG; ++h) {
            float w[4];
            uint32_t hi[2], mid[2], lo[2];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                w[u] = L.qp[h][u] * sv[u];
                bias[h] = fmaf(L.qp[h][u], dz[u], bias[h]);
            }
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                __nv_bfloat162 hb = __floats2bfloat162_rn(w[2 * v], w[2 * v + 1]);
                hi[v] = *reinterpret_cast<uint32_t*>(&hb);
                const float h0 = __uint_as_float(hi[v] << 16), h1 = __uint_as_float(hi[v] & 0xFFFF0000u);
                const float r0 = w[2 * v] - h0, r1 = w[2 * v + 1] - h1;  // exact
                __nv_bfloat162 mb = __floats2bfloat162_rn(r0, r1);
                mid[v] = *reinterpret_cast<uint32_t*>(&mb);
                const float m0 = __uint_as_float(mid[v] << 16), m1 = __uint_as_float(mid[v] & 0xFFFF0000u);
                __nv_bfloat162 lb = __floats2bfloat162_rn(r0 - m0, r1 - m1);
                lo[v] = *reinterpret_cast<uint32_t*>(&lb);
            }
            // (hi, mid) of head h in columns (2h, 2h+1), lo in column 2*HPG + h
            *reinterpret_cast<uint2*>(btile + btile_off(2 * h, 4 * lane)) = make_uint2(hi[0], hi[1]);
            *reinterpret_cast<uint2*>(btile + btile_off(2 * h + 1, 4 * lane)) = make_uint2(mid[0], mid[1]);
            *reinterpret_cast<uint2*>(btile + btile_off(2 * HPG + h, 4 * lane)) = make_uint2(lo[0], lo[1]);
        }
    }
    // full-warp reductions of the biases (every lane ends with every head's total)
#pragma unroll
    for (int h = 0; h < HPG; ++h) bias[h] = warp_sum(bias[h]);
    __syncwarp();
    // ---- B fragments: ldmatrix.x4 per pair of k-steps per n-tile ----
    uint32_t bf[TR::NT][8][2];
    const uint32_t bt = smem_u32(btile);
#pragma unroll
    for (int nt = 0; nt < TR::NT; ++nt)
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
            // matrix m = lane / 8: k-step 2kp + m/2, k-half m%2; row = column nt*8 + lane%8
            const int m = lane >> 3, col = nt * 8 + (lane & 7);
            const int kslot = (2 * kp + (m >> 1)) * 16 + (m & 1) * 8;
            ldsm_x4(bt + btile_off(col, kslot), bf[nt][2 * kp][0], bf[nt][2 * kp][1], bf[nt][2 * kp + 1][0],
                    bf[nt][2 * kp + 1][1]);
        }
    __syncwarp();  // the tile may be rewritten by the next slab
    // ---- two m-tiles of 16 tokens ----
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
        const uint32_t x0 = *reinterpret_cast<const uint32_t*>(bits_s + (mt * 16 + r) * 16 + 4 * c);
        const uint32_t x1 = *reinterpret_cast<const uint32_t*>(bits_s + (mt * 16 + r + 8) * 16 + 4 * c);
        const uint32_t y0 = __funnelshift_r(x0, x0, 8), y1 = __funnelshift_r(x1, x1, 8);
        float d[TR::NT][4];
#pragma unroll
        for (int nt = 0; nt < TR::NT; ++nt) d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
#define FIER_KSTEP(KS)                                                                                        \
    {                                                                                                         \
        const uint32_t a0 = abits<2 * KS>(x0, y0), a1 = abits<2 * KS>(x1, y1);                               \
        const uint32_t a2 = abits<2 * KS + 1>(x0, y0), a3 = abits<2 * KS + 1>(x1, y1);                       \
        _Pragma("unroll") for (int nt = 0; nt < TR::NT; ++nt)                                                 \
            mma_bf16(d[nt], a0, a1, a2, a3, bf[nt][KS][0], bf[nt][KS][1]);                                    \
    }
        FIER_KSTEP(0) FIER_KSTEP(1) FIER_KSTEP(2) FIER_KSTEP(3) FIER_KSTEP(4) FIER_KSTEP(5) FIER_KSTEP(6)
        FIER_KSTEP(7)
#undef FIER_KSTEP
        // thread (r, c): head h = nt*4 + c, columns (hi, mid) in tile nt, lo in
        // column 2*HPG + h = lane (r, lc/2) element lc%2 of tile lc/8
        constexpr float kScale = 2.f * 1152921504606846976.f;  // 2 * 2^sigma
#pragma unroll
        for (int nt = 0; nt < TR::NHM; ++nt) {
            const int h = nt * 4 + c;
            const int lc = 2 * HPG + (h < HPG ? h : 0);
            const int lt = lc >> 3, src = (lane & ~3) | ((lc & 7) >> 1), el = lc & 1;
            float la0 = 0.f, la1 = 0.f, lb0 = 0.f, lb1 = 0.f;
#pragma unroll
            for (int t = (2 * HPG) / 8; t <= (3 * HPG - 1) / 8; ++t) {  // the lo tile(s)
                const float x0 = __shfl_sync(0xffffffffu, d[t][0], src);
                const float x1 = __shfl_sync(0xffffffffu, d[t][1], src);
                const float y0 = __shfl_sync(0xffffffffu, d[t][2], src);
                const float y1 = __shfl_sync(0xffffffffu, d[t][3], src);
                if (t == lt) {
                    la0 = x0; la1 = x1; lb0 = y0; lb1 = y1;
                }
            }
            if (h < HPG) {
                float bh = bias[0];
#pragma unroll
                for (int hh = 1; hh < HPG; ++hh) bh = (h == hh) ? bias[hh] : bh;
                const float loa = el ? la1 : la0, lob = el ? lb1 : lb0;
                const int ta = mt * 16 + r, tb = ta + 8;
                if (ta < ntok) out[h * ld + t0 + ta] = fmaf((d[nt][0] + d[nt][1]) + loa, kScale, bh);
                if (tb < ntok) out[h * ld + t0 + tb] = fmaf((d[nt][2] + d[nt][3]) + lob, kScale, bh);
            }
        }
    }
}

// ---- the kernel -------------------------------------------------------------------
// Every warp owns a contiguous range of the sealed slabs of all sequences and
// streams it through a private kMmaStages-deep smem ring: lane 0 issues the
// bulk copies (512 B of bits + 512 B of the slab's group parameters) of slab
// i + kMmaStages - 1 while the warp scores slab i; completion is an mbarrier
// per ring slot.  No CTA-wide barrier in the main loop.
template <int HPG>
constexpr size_t mma_smem() {
    return (size_t)kMmaWarps * kMmaStages * (kSlabBytes + kParBytes) + (size_t)kMmaWarps * MmaTraits<HPG>::BTILE +
           (size_t)kMmaWarps * kMmaStages * 8;
}

__device__ __forceinline__ float pow2f(int k) { return __int_as_float((k + 127) << 23); }  // -126 <= k <= 127

template <typename T, int HPG>
__device__ __forceinline__ void lane_q(const T* qg, const int (&ch)[4], const float (&dn)[4], LaneConst<HPG>& L) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int h = 0; h < HPG; ++h) L.qp[h][u] = to_f32(qg[h * 128 + ch[u]]) * dn[u];
}

template <typename T, int HPG>
__global__ void __launch_bounds__(kMmaWarps * 32) score_mma_kernel(const T* __restrict__ q, uint32_t* bits,
                                                                   __half2* sz, int cap, int G, int hkv, int hq,
                                                                   int nseq, int tokens, int lg, float* __restrict__ scores,
                                                                   int64_t ld, AppendArgs2 ap) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = 32 << lg;  // group size, a power of two >= 32 (lg = log2(g / 32))
    uint8_t* ring = smem + (size_t)warp * kMmaStages * (kSlabBytes + kParBytes);  // [slot] {bits, params}
    uint8_t* btiles = smem + (size_t)kMmaWarps * kMmaStages * (kSlabBytes + kParBytes);
    uint8_t* btile = btiles + (size_t)warp * MmaTraits<HPG>::BTILE;
    uint64_t* full = reinterpret_cast<uint64_t*>(btiles + (size_t)kMmaWarps * MmaTraits<HPG>::BTILE) +
                     warp * kMmaStages;
    // zero this warp's B tile once: columns >= 3*HPG stay zero
    for (int i = lane; i < MmaTraits<HPG>::BTILE / 16; i += 32)
        reinterpret_cast<uint4*>(btile)[i] = make_uint4(0, 0, 0, 0);

    // per-lane slot constants (independent of the sequence)
    LaneConst<HPG> L;
    float dn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int ks = 4 * lane + u;
        L.ch[u] = kslot_channel(ks);
        const int e = kslot_exp(ks);
        L.up[u] = pow2f(e + kSigma);
        dn[u] = pow2f(-e - kSigma);
    }

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
            pack_group<T>(Kseq, 128, 4, g, ap.pos >> (5 + lg), ap.pos + 1, bseq, zseq, ap.nonfinite,
                          static_cast<const T*>(ap.k_new) + (int64_t)seq * 128, ap.pos);
            if (own) {
                Kseq[(int64_t)ap.pos * 128 + threadIdx.x] = kr;
                Vseq[(int64_t)ap.pos * 128 + threadIdx.x] = vr;
            }
            __syncthreads();
            lane_q<T, HPG>(q + ((int64_t)b * hq + h * HPG) * 128, L.ch, dn, L);
            for (int slab = open0 + warp; slab < nslabs; slab += kMmaWarps) {
                uint8_t* bs = ring;
                uint8_t* ps = bs + kSlabBytes;
                const int t0 = slab * 32, ntok = min(32, tokens - t0);
                // coherent (L1-bypassing) reads of what this CTA just wrote
                reinterpret_cast<uint4*>(bs)[lane] =
                    lane < ntok ? __ldcg(reinterpret_cast<const uint4*>(bseq) + t0 + lane) : make_uint4(0, 0, 0, 0);
                reinterpret_cast<uint4*>(ps)[lane] =
                    __ldcg(reinterpret_cast<const uint4*>(zseq + (int64_t)(slab >> lg) * 128) + lane);
                __syncwarp();
                score_slab_mma<HPG>(L, bs, ps, btile, t0, ntok, scores + ((int64_t)b * hq + h * HPG) * ld, ld);
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
    // (seq, slab) of the next slab to issue, advanced incrementally (no divisions)
    int iseq = (int)(w0 / open0), islab = (int)(w0 - (int64_t)iseq * open0);
    auto issue = [&](int slot) {  // lane 0
        const int t0 = islab * 32, ntok = min(32, tokens - t0);
        uint8_t* dst = ring + (size_t)slot * (kSlabBytes + kParBytes);
        mbar_arrive_expect_tx(&full[slot], (uint32_t)ntok * 16 + kParBytes);
        bulk_g2s_evict_first(dst, bits + ((int64_t)iseq * cap + t0) * 4, (uint32_t)ntok * 16, &full[slot], pol);
        bulk_g2s_evict_first(dst + kSlabBytes, sz + ((int64_t)iseq * G + (islab >> lg)) * 128, kParBytes,
                             &full[slot], pol);
        if (++islab == open0) {
            islab = 0;
            ++iseq;
        }
    };
    const int n = (int)(w1 - w0);
    if (lane == 0)
        for (int s = 0; s < kMmaStages - 1 && s < n; ++s) issue(s);
    int seq = (int)(w0 / open0), slab = (int)(w0 - (int64_t)seq * open0);
    int b = seq / hkv, h = seq - b * hkv;
    lane_q<T, HPG>(q + ((int64_t)b * hq + h * HPG) * 128, L.ch, dn, L);
    float* out = scores + ((int64_t)b * hq + h * HPG) * ld;
    for (int i = 0; i < n; ++i) {
        const int slot = i % kMmaStages;
        if (lane == 0 && i + kMmaStages - 1 < n) issue((i + kMmaStages - 1) % kMmaStages);
        mbar_wait(&full[slot], (uint32_t)((i / kMmaStages) & 1));
        const uint8_t* stg = ring + (size_t)slot * (kSlabBytes + kParBytes);
        const int t0 = slab * 32;
        score_slab_mma<HPG>(L, stg, stg + kSlabBytes, btile, t0, min(32, tokens - t0), out, ld);
        __syncwarp();  // every lane is done with `slot` before lane 0 refills it
        if (++slab == open0 && i + 1 < n) {
            slab = 0;
            ++seq;
            b = seq / hkv;
            h = seq - b * hkv;
            lane_q<T, HPG>(q + ((int64_t)b * hq + h * HPG) * 128, L.ch, dn, L);
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
