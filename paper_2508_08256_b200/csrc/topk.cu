// topk.cu -- K3: per-head Top-k token selector.
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores,
// ties to the LOWER index, returned in ascending index order.
//
// One thread-block cluster (C <= 8 CTAs of 512 or 256 threads) per score row;
// CTA r owns the contiguous slice [r*S, (r+1)*S) and keeps its keys in
// registers (KPT per thread, slot j of lane L of warp w = position
// w*32*KPT + 32j + L).  Shared-memory atomics cost ~2 cycles per lane on this
// part, so histograms are counted WITHOUT atomics: per 32-key slot a warp
// multisplit (__match_any_sync gives every lane the mask of lanes sharing its
// bin; the lowest such lane adds the popcount into the warp's private smem row).
//
//   1. (lo, hi) = min/max of the finite scores of the row (cluster exchange).
//   2. 32 linear bins over [lo, hi] -> bin b1 holding the k-th largest.
//   3. 32 linear sub-bins over b1's range -> b2.  Both binnings are monotone
//      non-decreasing functions of the value, so everything in a higher bin is
//      strictly larger than everything in a lower one.
//   4. Candidates = keys in (b1, b2) (typically tens): gathered over DSMEM and
//      ranked exactly by (value desc, index asc) -> threshold T and the number
//      r of T-valued keys to keep.
//   5. Compaction in index order with ballots: kept iff above (b1,b2), or a
//      candidate with key > T, or key == T among the first r ties; output slot
//      = #kept before it.  Output is ascending without a sort.
// If the candidate set overflows (massive ties / degenerate ranges) the
// cluster switches to an exact 3-pass radix select on the order-preserving
// keys (smem histograms), then the same compaction.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace fier_cuda {

constexpr int kTkMaxWarps = 16;
constexpr int kTkMaxCluster = 8;
constexpr int kTkCandCta = 256;   // candidates one CTA may contribute (fast path)
constexpr int kTkFlat = 1024;     // candidates a cluster may rank (fast path)
constexpr int kTkRadixBins = 2048;

struct TopkShared {
    // pushed by every CTA of the cluster into every CTA (slot = sender's rank),
    // then read locally after one cluster barrier
    float mm[kTkMaxCluster][2];               // min, max of finite values
    uint32_t h1[kTkMaxCluster][32];           // pass-1 histograms
    uint32_t h2[kTkMaxCluster][32];           // pass-2 histograms
    uint32_t ncand[kTkMaxCluster];            // candidates per CTA
    uint32_t nabove[kTkMaxCluster];           // strictly-above count per CTA
    uint32_t ckey[kTkMaxCluster][kTkCandCta];  // candidate keys
    int32_t cidx[kTkMaxCluster][kTkCandCta];   // candidate global indices
    // fallback radix path (pulled over DSMEM; rare)
    uint32_t rhist[2][kTkRadixBins];
    uint32_t rsel[2];
    uint32_t tot[kTkRadixBins];
    // CTA-private
    uint32_t wh[kTkMaxWarps][32];             // per-warp histogram rows
    uint32_t wcnt[kTkMaxWarps];
    float fscratch[2 * kTkMaxWarps];
    uint32_t lcand;                           // local candidate counter
    uint32_t res[8];
    uint32_t wnab[kTkMaxWarps];               // strictly-above keys per warp (this CTA)
    uint32_t wg[kTkMaxWarps], we[kTkMaxWarps];  // candidates > T / == T per warp
    uint32_t cg[kTkMaxCluster], ce[kTkMaxCluster];  // candidates > T / == T per CTA
    uint32_t fkey[kTkFlat];                   // flattened candidates (CTA-rank order)
    int32_t fidx[kTkFlat];
    uint8_t fcta[kTkFlat];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp multisplit of a bin id: adds each bin's lane count into row[bin] (bins
// >= 32 are ignored).  No atomics: __match_any_sync gives every lane the mask
// of lanes sharing its bin; the lowest lane of each group does a plain RMW.
__device__ __forceinline__ void warp_count_bins(uint32_t bin, uint32_t* row) {
    const uint32_t peers = __match_any_sync(0xffffffffu, bin);
    if (bin < 32 && (peers & lanemask_lt()) == 0) row[bin] += __popc(peers);
}

// suffix search over 32 bins held one per lane (lane b has count of bin b):
// returns in all lanes the bin b* with above(b*) < krem <= above(b*)+cnt(b*),
// above(b) = sum of bins > b.
__device__ __forceinline__ void find_bin32(uint32_t cnt, uint32_t krem, uint32_t* bin,
                                           uint32_t* above) {
    const int lane = threadIdx.x & 31;
    // inclusive suffix sum: s(b) = sum_{b' >= b}
    uint32_t s = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, s, o);
        if (lane + o < 32) s += y;
    }
    const uint32_t ab = s - cnt;
    const uint32_t hit = __ballot_sync(0xffffffffu, ab < krem && krem <= s);
    const int b = 31 - __clz(hit);  // unique in exact arithmetic; highest if any
    *bin = (uint32_t)b;
    *above = __shfl_sync(0xffffffffu, ab, b);
}

__device__ __forceinline__ int lin_bin(float x, float lo, float inv) {
    // +-inf clamp to bins 31 / 0 (inv > 0 on the fast path)
    float t = (x - lo) * inv;
    t = fminf(fmaxf(t, 0.f), 31.f);
    return (int)t;  // truncation == floor on [0, 31]
}

// Block-wide exclusive scan over warps of one value per warp (lane 0 holds it);
// returns the warp's exclusive prefix in all lanes and the block total.
template <int kTkWarps>
__device__ __forceinline__ uint32_t warp_prefix(uint32_t v, uint32_t* wcnt, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wcnt[warp] = v;
    __syncthreads();
    uint32_t ex = 0, t = 0;
#pragma unroll
    for (int w = 0; w < kTkWarps; ++w) {
        const uint32_t x = wcnt[w];
        ex += w < warp ? x : 0u;
        t += x;
    }
    __syncthreads();
    *total = t;
    return ex;
}

template <int KPT, int kTkThreads>
__global__ void __launch_bounds__(kTkThreads) topk_kernel(const float* __restrict__ scores, int tokens,
                                                          int64_t ld, int k, int slice,
                                                          int32_t* __restrict__ sel) {
    constexpr int kTkWarps = kTkThreads / 32;
    cg::cluster_group cluster = cg::this_cluster();
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* srow = scores + (int64_t)row * ld;
    const int s0 = rank * slice;
    const int cnt = max(0, min(s0 + slice, tokens) - s0);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    TopkShared& S = *reinterpret_cast<TopkShared*>(smem_raw);

    // Every CTA of the cluster must have started before anyone writes into its
    // shared memory: arrive now, wait just before the first remote store.
    asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
    // ---- load: slot j of this lane = position warp*32*KPT + 32j + lane ----
    const int wbase = warp * 32 * KPT;
    float x[KPT];
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const int p = wbase + 32 * j + lane;
        x[j] = p < cnt ? srow[s0 + p] : __int_as_float(0x7fffffff);  // NaN = empty slot
        if (isfinite(x[j])) {
            mn = fminf(mn, x[j]);
            mx = fmaxf(mx, x[j]);
        }
    }
    for (int i = tid; i < kTkWarps * 32; i += kTkThreads) (&S.wh[0][0])[i] = 0;
    mn = -warp_max(-mn);
    mx = warp_max(mx);
    if (lane == 0) {
        S.fscratch[warp] = mn;
        S.fscratch[kTkWarps + warp] = mx;
    }
    if (tid == 0) S.lcand = 0;
    __syncthreads();
    asm volatile("barrier.cluster.wait;" ::: "memory");
    if (tid < nct) {  // push this CTA's (min, max) into slot [rank] of CTA tid
        float a = INFINITY, b = -INFINITY;
        for (int w = 0; w < kTkWarps; ++w) {
            a = fminf(a, S.fscratch[w]);
            b = fmaxf(b, S.fscratch[kTkWarps + w]);
        }
        float* dst = cluster.map_shared_rank(&S.mm[rank][0], tid);
        dst[0] = a;
        dst[1] = b;
    }
    cluster.sync();  // #1
    float lo = INFINITY, hi = -INFINITY;
    for (int r = 0; r < nct; ++r) {
        lo = fminf(lo, S.mm[r][0]);
        hi = fmaxf(hi, S.mm[r][1]);
    }
    if (!(lo <= hi)) {  // no finite values
        lo = 0.f;
        hi = 0.f;
    }
    const float inv1 = hi > lo ? 32.f / (hi - lo) : 0.f;

    // ---- pass 1: 32 bins over [lo, hi]; code[j] caches the bin (63 = empty) ----
    int code[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        code[j] = isnan(x[j]) ? 63 : lin_bin(x[j], lo, inv1);
        warp_count_bins((uint32_t)code[j], S.wh[warp]);
    }
    __syncthreads();
    if (tid < 32 * nct) {  // push histogram bin (tid % 32) to CTA tid / 32
        const int b = tid & 31;
        uint32_t c = 0;
        for (int w = 0; w < kTkWarps; ++w) c += S.wh[w][b];
        *cluster.map_shared_rank(&S.h1[rank][b], tid >> 5) = c;
    }
    __syncthreads();
    for (int i = tid; i < kTkWarps * 32; i += kTkThreads) (&S.wh[0][0])[i] = 0;
    cluster.sync();  // #2
    uint32_t b1, above1, b2, above2;
    {
        uint32_t c = 0;
        for (int r = 0; r < nct; ++r) c += S.h1[r][lane];
        find_bin32(c, (uint32_t)k, &b1, &above1);
    }
    // ---- pass 2: 32 sub-bins over bin b1 ----
    const float w1 = (hi - lo) / 32.f;
    const float lo2 = lo + (float)b1 * w1;
    const float inv2 = w1 > 0.f ? 32.f / w1 : 0.f;
    // code[j] becomes: -1 below b1 (or empty), 64 above b1, else the sub-bin
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const int c1 = code[j];
        int c = c1 == 63 ? -1 : (c1 < (int)b1 ? -1 : (c1 > (int)b1 ? 64 : lin_bin(x[j], lo2, inv2)));
        code[j] = c;
        warp_count_bins(c >= 0 && c < 32 ? (uint32_t)c : 63u, S.wh[warp]);
    }
    __syncthreads();
    if (tid < 32 * nct) {
        const int b = tid & 31;
        uint32_t c = 0;
        for (int w = 0; w < kTkWarps; ++w) c += S.wh[w][b];
        *cluster.map_shared_rank(&S.h2[rank][b], tid >> 5) = c;
    }
    cluster.sync();  // #3
    {
        uint32_t c = 0;
        for (int r = 0; r < nct; ++r) c += S.h2[r][lane];
        find_bin32(c, (uint32_t)k - above1, &b2, &above2);
    }
    uint32_t krem = (uint32_t)k - above1 - above2;  // >= 1

    // ---- candidates (b1, b2) pushed to every CTA; strictly-above counts ----
    uint32_t nab = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const int c = code[j] > (int)b2 ? 2 : (code[j] == (int)b2 ? 1 : 0);  // above / candidate / below
        nab += __popc(__ballot_sync(0xffffffffu, c == 2));
        const uint32_t m = __ballot_sync(0xffffffffu, c == 1);
        if (m) {
            uint32_t base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&S.lcand, (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            const uint32_t slot = base + __popc(m & lanemask_lt());
            if (c == 1 && slot < kTkCandCta) {
                const uint32_t key = float_key(x[j]);
                const int32_t idx = s0 + wbase + 32 * j + lane;
                for (int r = 0; r < nct; ++r) {
                    *cluster.map_shared_rank(&S.ckey[rank][slot], r) = key;
                    *cluster.map_shared_rank(&S.cidx[rank][slot], r) = idx;
                }
            }
        }
    }
    if (lane == 0) S.wnab[warp] = nab;
    uint32_t tot_ab;
    warp_prefix<kTkWarps>(nab, S.wcnt, &tot_ab);  // (contains __syncthreads: lcand final)
    if (tid < nct) {
        *cluster.map_shared_rank(&S.ncand[rank], tid) = S.lcand;
        *cluster.map_shared_rank(&S.nabove[rank], tid) = tot_ab;
    }
    cluster.sync();  // #4 -- after this, the fast path reads only local smem
    uint32_t off[kTkMaxCluster + 1];
    off[0] = 0;
    uint32_t ncand_max = 0;
#pragma unroll
    for (int r = 0; r < kTkMaxCluster; ++r) {
        const uint32_t c = r < nct ? S.ncand[r] : 0u;
        off[r + 1] = off[r] + c;
        ncand_max = max(ncand_max, c);
    }
    const uint32_t ncand_all = off[kTkMaxCluster];

    uint32_t T;                 // threshold key
    uint32_t sel_before = 0;    // kept elements in lower-ranked CTAs
    uint32_t eq_before = 0;     // T-valued keys in lower-ranked CTAs
    uint32_t gt_w = 0, eq_w = 0;  // (> T) / (== T) keys of this CTA in lower warps
    // uniform over the cluster: overflow, or a degenerate range (hi == lo: the
    // linear bins cannot order +inf against the finite values)
    const bool radix = ncand_max > kTkCandCta || ncand_all > kTkFlat || !(inv1 > 0.f);
    if (!radix) {
        // flatten the candidates (CTA-rank order), classify after T is known
        for (uint32_t i = tid; i < ncand_all; i += kTkThreads) {
            int r = 0;
#pragma unroll
            for (int rr = 1; rr < kTkMaxCluster; ++rr) r += i >= off[rr];
            S.fkey[i] = S.ckey[r][i - off[r]];
            S.fidx[i] = S.cidx[r][i - off[r]];
            S.fcta[i] = (uint8_t)r;
        }
        if (tid < kTkMaxCluster) {
            S.cg[tid] = 0;
            S.ce[tid] = 0;
        }
        if (tid < kTkWarps) {
            S.wg[tid] = 0;
            S.we[tid] = 0;
        }
        __syncthreads();
        // rank by (key desc, index asc), one warp per candidate, lanes split j;
        // the candidate of rank krem-1 is the threshold T
        for (uint32_t i = warp; i < ncand_all; i += kTkWarps) {
            const uint32_t ki = S.fkey[i];
            const int32_t ii = S.fidx[i];
            uint32_t rk = 0;
            for (uint32_t j = lane; j < ncand_all; j += 32) {
                const uint32_t kj = S.fkey[j];
                rk += (kj > ki) || (kj == ki && S.fidx[j] < ii);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
            if (lane == 0 && rk == krem - 1) S.res[0] = ki;
        }
        __syncthreads();
        T = S.res[0];
        // per-CTA and (this CTA) per-warp counts of candidates > T and == T
        for (uint32_t i = tid; i < ncand_all; i += kTkThreads) {
            const uint32_t key = S.fkey[i];
            const int r = S.fcta[i];
            const bool g = key > T, e = key == T;
            if (g) atomicAdd(&S.cg[r], 1u);
            if (e) atomicAdd(&S.ce[r], 1u);
            if (r == rank) {
                const int w = (S.fidx[i] - s0) / (32 * KPT);
                if (g) atomicAdd(&S.wg[w], 1u);
                if (e) atomicAdd(&S.we[w], 1u);
            }
        }
        __syncthreads();
        uint32_t gtT = 0;
        for (int r = 0; r < nct; ++r) gtT += S.cg[r];
        const uint32_t rties = krem - gtT;  // T-valued keys to keep (global index order)
        uint32_t ties_seen = 0;
        for (int r = 0; r < rank; ++r) {
            const uint32_t ce = S.ce[r];
            sel_before += S.nabove[r] + S.cg[r] + min(ce, rties > ties_seen ? rties - ties_seen : 0u);
            ties_seen += ce;
        }
        eq_before = ties_seen;
        krem = rties;
        for (int w = 0; w < warp; ++w) {
            gt_w += S.wnab[w] + S.wg[w];
            eq_w += S.we[w];
        }
    } else {
        // ---- exact radix fallback on the order-preserving keys ----
        uint32_t prefix = 0, pmask = 0, kr = (uint32_t)k;
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
            const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
            const int bins = pass == 2 ? 1024 : 2048;
            uint32_t* h = S.rhist[pass & 1];
            for (int i = tid; i < bins; i += kTkThreads) h[i] = 0;
            __syncthreads();
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                if (!isnan(x[j])) {
                    const uint32_t key = float_key(x[j]);
                    if ((key & pmask) == prefix) atomicAdd(&h[(key >> shift) & (bins - 1)], 1u);
                }
            }
            cluster.sync();
            for (int i = tid; i < bins; i += kTkThreads) {
                uint32_t a = 0;
                for (int r = 0; r < nct; ++r) a += cluster.map_shared_rank(h, r)[i];
                S.tot[i] = a;
            }
            __syncthreads();
            if (warp == 0) {  // descending scan, 32 lanes x bins/32 bins each
                const int per = bins / 32;
                uint32_t loc = 0;
                for (int j = 0; j < per; ++j) loc += S.tot[bins - 1 - (lane * per + j)];
                uint32_t inc = loc;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                uint32_t ab = inc - loc;
                for (int j = 0; j < per; ++j) {
                    const int bin = bins - 1 - (lane * per + j);
                    const uint32_t c = S.tot[bin];
                    if (ab < kr && kr <= ab + c) {
                        S.res[1] = (uint32_t)bin;
                        S.res[2] = ab;
                    }
                    ab += c;
                }
            }
            __syncthreads();
            kr -= S.res[2];
            prefix |= S.res[1] << shift;
            pmask |= (uint32_t)(bins - 1) << shift;
            __syncthreads();
        }
        T = prefix;
        // CTA counts of (> T, == T) -> prefixes over lower CTAs and lower warps
        uint32_t g = 0, e = 0;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const uint32_t key = isnan(x[j]) ? 0u : float_key(x[j]);
            g += __popc(__ballot_sync(0xffffffffu, !isnan(x[j]) && key > T));
            e += __popc(__ballot_sync(0xffffffffu, !isnan(x[j]) && key == T));
        }
        uint32_t tg, te;
        gt_w = warp_prefix<kTkWarps>(g, S.wcnt, &tg);
        eq_w = warp_prefix<kTkWarps>(e, S.wcnt, &te);
        if (tid == 0) {
            S.rsel[0] = tg;
            S.rsel[1] = te;
        }
        cluster.sync();
        uint32_t gb = 0, eb = 0;
        for (int r = 0; r < rank; ++r) {
            const uint32_t* m = cluster.map_shared_rank(S.rsel, r);
            gb += m[0];
            eb += m[1];
        }
        sel_before = gb + min(eb, kr);
        eq_before = eb;
        krem = kr;
        cluster.sync();  // remote reads of rsel done before any CTA exits
    }

    // ---- single compaction pass in index order ----
    // kept iff key > T or (key == T and tie rank < krem); slot = #(> T before) +
    // min(#(== T before), krem), counted from the row start.
    uint32_t gt_run = (sel_before - min(eq_before, krem)) + gt_w;
    uint32_t eq_run = eq_before + eq_w;
    int32_t* out = sel + (int64_t)row * k;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const bool v = !isnan(x[j]);
        const uint32_t key = v ? float_key(x[j]) : 0u;
        const bool g = v && key > T, e = v && key == T;
        const uint32_t mg = __ballot_sync(0xffffffffu, g);
        const uint32_t me = __ballot_sync(0xffffffffu, e);
        const uint32_t my_gt = gt_run + __popc(mg & lt);
        const uint32_t my_eq = eq_run + __popc(me & lt);
        if (g || (e && my_eq < krem)) out[my_gt + min(my_eq, krem)] = s0 + wbase + 32 * j + lane;
        gt_run += __popc(mg);
        eq_run += __popc(me);
    }
}

// Long rows (> 8 * 256 * 64 keys): the original smem-radix kernel streaming keys
// from global memory each pass (correct for any length; not the fast path).
__global__ void __launch_bounds__(1024, 1)
    topk_stream_kernel(const float* __restrict__ scores, int tokens, int64_t ld, int k, int slice,
                       int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* srow = scores + (int64_t)row * ld;
    const int s0 = rank * slice;
    const int cnt = max(0, min(s0 + slice, tokens) - s0);
    __shared__ uint32_t hist[2][kTkRadixBins];
    __shared__ uint32_t tot[kTkRadixBins];
    __shared__ uint32_t misc[160];
    uint32_t prefix = 0, pmask = 0, krem = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
        const int bins = pass == 2 ? 1024 : 2048;
        uint32_t* h = hist[pass & 1];
        for (int i = tid; i < bins; i += 1024) h[i] = 0;
        __syncthreads();
        for (int i = tid; i < cnt; i += 1024) {
            const uint32_t key = float_key(srow[s0 + i]);
            if ((key & pmask) == prefix) atomicAdd(&h[(key >> shift) & (bins - 1)], 1u);
        }
        cluster.sync();
        for (int i = tid; i < bins; i += 1024) {
            uint32_t a = 0;
            for (int r = 0; r < nct; ++r) a += cluster.map_shared_rank(h, r)[i];
            tot[i] = a;
        }
        __syncthreads();
        if (warp == 0) {
            const int per = bins / 32;
            uint32_t loc = 0;
            for (int j = 0; j < per; ++j) loc += tot[bins - 1 - (lane * per + j)];
            uint32_t inc = loc;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            uint32_t ab = inc - loc;
            for (int j = 0; j < per; ++j) {
                const int bin = bins - 1 - (lane * per + j);
                const uint32_t c = tot[bin];
                if (ab < krem && krem <= ab + c) {
                    misc[64] = (uint32_t)bin;
                    misc[65] = ab;
                }
                ab += c;
            }
        }
        __syncthreads();
        krem -= misc[65];
        prefix |= misc[64] << shift;
        pmask |= (uint32_t)(bins - 1) << shift;
        __syncthreads();
    }
    const uint32_t T = prefix;
    const int per_w = (int)(((cnt + 32 * 32 - 1) / (32 * 32)) * 32);
    const int w0 = warp * per_w, w1 = min(w0 + per_w, cnt);
    uint32_t gt = 0, eq = 0;
    for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const uint32_t key = i < w1 ? float_key(srow[s0 + i]) : 0u;
        gt += __popc(__ballot_sync(0xffffffffu, key > T));
        eq += __popc(__ballot_sync(0xffffffffu, key == T));
    }
    uint32_t* wgt = misc + 72;
    uint32_t* weq = misc + 104;
    if (lane == 0) {
        wgt[warp] = gt;
        weq[warp] = eq;
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t a = wgt[lane], e = weq[lane];
        uint32_t ia = a, ie = e;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
            const uint32_t ye = __shfl_up_sync(0xffffffffu, ie, o);
            if (lane >= o) {
                ia += ya;
                ie += ye;
            }
        }
        wgt[lane] = ia - a;
        weq[lane] = ie - e;
        if (lane == 31) {
            misc[66] = ia;
            misc[67] = ie;
        }
    }
    cluster.sync();
    uint32_t cta_gt = 0, cta_eq = 0;
    for (int r = 0; r < rank; ++r) {
        const uint32_t* m = cluster.map_shared_rank(misc, r);
        cta_gt += m[66];
        cta_eq += m[67];
    }
    uint32_t gt_before = cta_gt + wgt[warp];
    uint32_t eq_before = cta_eq + weq[warp];
    int32_t* out = sel + (int64_t)row * k;
    const uint32_t lower = (1u << lane) - 1u;
    for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const uint32_t key = i < w1 ? float_key(srow[s0 + i]) : 0u;
        const bool g = key > T, e = key == T;
        const uint32_t mg = __ballot_sync(0xffffffffu, g);
        const uint32_t me = __ballot_sync(0xffffffffu, e);
        const uint32_t my_gt = gt_before + __popc(mg & lower);
        const uint32_t my_eq = eq_before + __popc(me & lower);
        if (g || (e && my_eq < krem)) out[my_gt + min(my_eq, krem)] = s0 + i;
        gt_before += __popc(mg);
        eq_before += __popc(me);
    }
    cluster.sync();
}

size_t topk_workspace(int rows, int tokens, int k) {
    (void)rows;
    (void)tokens;
    (void)k;
    return 0;
}

template <typename Kern, typename... Args>
static int launch_cluster(Kern kern, int cluster, int rows, int threads, size_t smem, cudaStream_t st,
                          Args... args) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

int topk2_dispatch(const float*, int, int, int64_t, int, int32_t*, cudaStream_t);

int topk_rx_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st);
int topk_long_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st);

int topk_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel,
                  cudaStream_t st) {
    {  // adaptive cluster select (topk2.cu); FIER_TOPK=rx: the fixed-radix one (topk_rx.cu)
        int rc = topk_rx_dispatch(scores, rows, tokens, ld, k, sel, st);
        if (rc >= 0) return rc;
        rc = topk2_dispatch(scores, rows, tokens, ld, k, sel, st);
        if (rc >= 0) return rc;
    }
    // Register path: CTA slices up to 512 x 16 (or 256 x 64) keys, cluster of
    // C <= 8 CTAs per row, C grown until the grid covers the chip.
    constexpr int kMaxSlice = 256 * 64;
    int c = 1;
    while (c < kTkMaxCluster && ((int64_t)rows * c < 2 * num_sms() || ceil_div(tokens, c) > kMaxSlice)) c *= 2;
    while (c > 1 && ceil_div(tokens, c) < 512 * 2) c /= 2;
    const int64_t slice = ceil_div(tokens, c);
    const size_t smem = sizeof(TopkShared);
    if (slice <= kMaxSlice) {
        if (slice <= 512 * 2) return launch_cluster(topk_kernel<2, 512>, c, rows, 512, smem, st, scores, tokens, ld, k, 1024, sel);
        if (slice <= 512 * 4) return launch_cluster(topk_kernel<4, 512>, c, rows, 512, smem, st, scores, tokens, ld, k, 2048, sel);
        if (slice <= 512 * 8) return launch_cluster(topk_kernel<8, 512>, c, rows, 512, smem, st, scores, tokens, ld, k, 4096, sel);
        if (slice <= 512 * 16) return launch_cluster(topk_kernel<16, 512>, c, rows, 512, smem, st, scores, tokens, ld, k, 8192, sel);
        if (slice <= 256 * 32) return launch_cluster(topk_kernel<32, 256>, c, rows, 256, smem, st, scores, tokens, ld, k, 8192, sel);
        return launch_cluster(topk_kernel<64, 256>, c, rows, 256, smem, st, scores, tokens, ld, k, kMaxSlice, sel);
    }
    {  // rows too long for the on-chip paths (C5): three streaming passes, radix threshold
        const int rc = topk_long_dispatch(scores, rows, tokens, ld, k, sel, st);
        if (rc >= 0) return rc;
    }
    const int sl = (int)(ceil_div(slice, 32) * 32);
    return launch_cluster(topk_stream_kernel, c, rows, 1024, 0, st, scores, tokens, ld, k, sl, sel);
}

}  // namespace fier_cuda
