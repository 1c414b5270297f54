// select_radix.cuh -- Top-k threshold of the fused decode step with a FIXED radix
// digit histogram built while scoring.
//
// Reference: topk_oracle (core.hpp:134-148): the k largest, ties to the lower
// index, ascending output.  Same cluster/key layout as select.cuh (warp w owns
// slots [w*32*kpt, (w+1)*32*kpt) of its CTA's slice; key 0 = empty), but the
// first histogram needs no (min, max) exchange: digit 1 = the top 12 bits of the
// order-preserving key (sign, exponent, 3 mantissa bits), counted by the scorer
// as it produces each key (rx_count).  Then:
//   [cluster barrier]  merge the 64 coarse sums (64 digit-1 bins each) over DSMEM ->
//                      coarse bin of the k-th largest -> merge its 64 fine bins ->
//                      bin b1, krem (one warp, shuffles; 2 KB of remote reads);
//   one pass over the keys: candidates (digit 1 == b1) -> this CTA's list, and
//                      per-warp counts of keys above b1; publish (candidates,
//                      above);
//   [cluster barrier]  every CTA gathers all candidates (identical list) and
//                      refines it by 8-bit digits (bits 19..12, 11..4, 3..0)
//                      down to <= 32 -> exact rank (value desc, index asc) ->
//                      (T, idx_T); a tie group larger than 32 is resolved by the
//                      same digit refinement on the indices;
//   keep rule:         key > T, or key == T and index <= idx_T -- a local test, so
//                      every CTA derives every CTA's kept count from the published
//                      "above" counts and the shared candidate list: the output
//                      offsets need no further cluster barrier.
// Two cluster barriers instead of four, two passes over the keys instead of four.
// Candidate overflow (a digit-1 bin holding more than kRxCand keys: very narrow
// score ranges) falls back to the exact MSD radix select of select.cuh.
#pragma once

#include "select.cuh"

namespace fier_cuda {

constexpr int kRxBins = 4096;      // digit 1: key >> 20 (64 coarse x 64 fine bins)
constexpr int kRxCtaCand = 512;    // candidates one CTA may contribute
constexpr int kRxCand = 2048;      // merged candidates per row

// Read by peers until the kernel's final cluster barrier: must not alias anything the
// CTA reuses after the second barrier.
struct RxPublished {
    uint32_t pub[4];               // (candidates, keys above b1) of this CTA
    uint32_t ckey[kRxCtaCand];     // this CTA's candidates
    int32_t cidx[kRxCtaCand];
};

// hist and coarse come last: they are dead after the second cluster barrier, so the
// fused step overlays its attention rings on them (step_fused.cu).
struct RxShared {
    alignas(16) uint32_t tot[kT2Bins];       // refinement histograms (8-bit digits); fallback merges
    uint32_t mkey[3][kRxCand];  // [0] all candidates of the row (kept), [1], [2] refinement
    int32_t midx[3][kRxCand];
    uint32_t cn[kT2MaxCluster], ca[kT2MaxCluster];     // every CTA's published pair
    uint32_t ck[kT2MaxCluster];                        // kept candidates per CTA
    uint32_t wab[32], wkc[32];                         // per warp: keys above b1, kept candidates
    uint32_t wsum[32], wsuf[32];
    uint32_t wg[kT2Warps], we[kT2Warps];               // (fallback compaction)
    uint32_t cgt[kT2MaxCluster], ceq[kT2MaxCluster];
    uint32_t res[8];
    uint32_t over, nabove, nkept;  // split variant: overflow flag, gather-list lengths
    uint32_t gclaim;               // the fused step's gather queue (granules claimed)
    alignas(256) uint32_t hist[kRxBins + 4];  // digit-1 histogram (scoring; read remotely); [kRxBins] = trash
    alignas(16) uint32_t coarse[64];          // sums of 64 consecutive digit-1 bins (read remotely)
};

// The scorer's contribution: count key kj (0 = empty -> trash bin).
__device__ __forceinline__ void rx_count(RxShared& S, uint32_t kj) {
    atomicAdd(&S.hist[kj ? kj >> 20 : kRxBins], 1u);
}

// Zero this CTA's digit-1 histogram (before any rx_count; then __syncthreads).
template <int NT>
__device__ __forceinline__ void rx_clear(RxShared& S) {
    for (int i = threadIdx.x; i < kRxBins + 4; i += NT) S.hist[i] = 0u;
}

// Refine list `src` (n entries) to the entries of the bin holding the krem-th
// largest of digit(value) (BINS bins); returns the survivors' count (in `dst`).
template <int NT, int BINS, typename Bar = CtaBar, typename Digit, typename SH>
__device__ __forceinline__ uint32_t rx_refine(SH& S, const uint32_t* sk, const int32_t* si, uint32_t n,
                                              uint32_t* dk, int32_t* di, uint32_t& krem, Digit&& digit) {
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < BINS; i += NT) S.tot[i] = 0u;
    Bar::sync();
    for (uint32_t i = tid; i < n; i += NT) atomicAdd(&S.tot[digit(sk[i], si[i])], 1u);
    Bar::sync();
    t2_find_bin<NT, BINS, SH, Bar>(S.tot, krem, S);
    const uint32_t b = S.res[0];
    krem -= S.res[1];
    if (tid == 0) S.res[2] = 0;
    Bar::sync();
    for (uint32_t i0 = 0; i0 < n; i0 += NT) {
        const uint32_t i = i0 + tid;
        const bool c = i < n && digit(sk[i], si[i]) == b;
        const uint32_t m = __ballot_sync(0xffffffffu, c);
        if (m) {
            uint32_t base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&S.res[2], (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            if (c) {
                const uint32_t slot = base + __popc(m & t2_lanemask_lt());
                dk[slot] = sk[i];
                di[slot] = si[i];
            }
        }
    }
    Bar::sync();
    return S.res[2];
}

// Exact rank of <= 32 (key, index) pairs by (key desc, index asc): the krem-th -> (T, idx_T).
template <typename Bar = CtaBar, typename SH>
__device__ __forceinline__ void rx_rank32(SH& S, const uint32_t* mk, const int32_t* mi, uint32_t n,
                                          uint32_t krem) {
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) == 0) {
        const bool v = (uint32_t)lane < n;
        const uint32_t ki = v ? mk[lane] : 0u;
        const int32_t ii = v ? mi[lane] : 0x7fffffff;
        uint32_t rk = 0;
        for (uint32_t o = 0; o < n; ++o) {  // smem broadcast reads
            const uint32_t kj = mk[o];
            const int32_t ij = mi[o];
            rk += (kj > ki) || (kj == ki && ij < ii);
        }
        const uint32_t hit = __ballot_sync(0xffffffffu, v && rk == krem - 1);
        const int src = __ffs(hit) - 1;  // unique
        if (lane == 0) {
            S.res[4] = __shfl_sync(0xffffffffu, ki, src);
            S.res[5] = (uint32_t)__shfl_sync(0xffffffffu, ii, src);
        } else {
            __shfl_sync(0xffffffffu, ki, src);
            __shfl_sync(0xffffffffu, ii, src);
        }
    }
    Bar::sync();
}

// One warp, 64 bins held 2 per lane (bin 2l -> c0, 2l+1 -> c1): the bin b with
// above(b) < kr <= above(b) + cnt(b), above(b) = count in bins > b.  Returns b (-1 if none)
// and above(b) in *ab (every lane).
__device__ __forceinline__ int rx_warp_find64(uint32_t c0, uint32_t c1, uint32_t kr, uint32_t* ab) {
    const int lane = threadIdx.x & 31;
    const uint32_t sl = c0 + c1;
    uint32_t suf = sl;  // inclusive suffix over lanes (higher lanes hold higher bins)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += y;
    }
    const uint32_t a1 = suf - sl, a0 = a1 + c1;
    const bool h1 = a1 < kr && kr <= a1 + c1, h0 = a0 < kr && kr <= a0 + c0;
    const uint32_t m = __ballot_sync(0xffffffffu, h0 || h1);
    if (!m) return -1;
    const int src = __ffs(m) - 1;
    const int b = 2 * src + (__shfl_sync(0xffffffffu, (int)h1, src) ? 1 : 0);
    *ab = __shfl_sync(0xffffffffu, h1 ? a1 : a0, src);
    return b;
}

// Sum over the cluster's CTAs of two consecutive u32 words at local shared address `a`.
__device__ __forceinline__ uint2 rx_cluster_sum2(uint32_t a, int nct) {
    uint2 t = make_uint2(0u, 0u);
    for (int r0 = 0; r0 < nct; r0 += 4) {
        uint2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            v[u] = make_uint2(0u, 0u);
            if (r0 + u < nct) {
                uint32_t ra;
                asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r0 + u));
                asm volatile("ld.shared::cluster.v2.u32 {%0,%1}, [%2];" : "=r"(v[u].x), "=r"(v[u].y) : "r"(ra));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            t.x += v[u].x;
            t.y += v[u].y;
        }
    }
    return t;
}

struct RxResult {
    bool fallback;      // cluster-uniform: the caller runs t2_radix_select + t2_compact
    uint32_t T;         // key of the k-th largest
    int32_t idxT;       // T-valued keys with index <= idxT are kept
    uint32_t cta_base;  // this CTA's first output slot
    uint32_t cta_count; // this CTA's kept keys
};

// The caller has cleared (rx_clear + __syncthreads) and filled (rx_count) the digit-1
// histogram and passes slice = tokens per CTA (s0 = rank * slice).  No cluster
// barrier may be pending: the first one here also proves every CTA is running.
template <int NT, typename Keys>
__device__ __forceinline__ RxResult rx_threshold(cg::cluster_group& cluster, const Keys& keys, int s0, int wbase,
                                                 int slice, int k, RxShared& S, RxPublished& P) {
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kpt = keys.count();
    RxResult R = {false, 0u, 0, 0u, 0u};
    __syncthreads();  // this CTA's histogram is complete
    for (int c = warp; c < 64; c += NT / 32) {  // coarse bins: 64 fine bins each, two per lane
        const uint2 v = reinterpret_cast<const uint2*>(S.hist + 64 * c)[lane];
        uint32_t x = v.x + v.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S.coarse[c] = x;
    }
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    T2_MARK(8);
    // ---- digit 1 over the cluster: coarse bin, then its 64 fine bins (2 KB of DSMEM reads) ----
    if (tid < 32) {
        S.wkc[tid] = 0u;
        if (tid < kT2MaxCluster) S.ck[tid] = 0u;
    }
    if (tid == 0) P.pub[0] = 0u;
    if (warp == 0) {
        uint32_t ab = 0, kr = (uint32_t)k;
        const uint2 cc = rx_cluster_sum2(smem_u32(S.coarse) + 8u * lane, nct);
        const int cb = rx_warp_find64(cc.x, cc.y, kr, &ab);
        int b = -1;
        if (cb >= 0) {
            kr -= ab;
            const uint2 ff = rx_cluster_sum2(smem_u32(S.hist + 64 * cb) + 8u * lane, nct);
            const int fb = rx_warp_find64(ff.x, ff.y, kr, &ab);
            if (fb >= 0) {
                b = 64 * cb + fb;
                kr -= ab;
            }
        }
        if (lane == 0) {
            S.res[0] = (uint32_t)b;
            S.res[1] = kr;
        }
    }
    __syncthreads();
    T2_MARK(14);
    const uint32_t b1 = S.res[0];  // ~0u: fewer keys than k (NaN scores) -> fallback
    uint32_t krem = S.res[1];
    T2_MARK(9);
    // ---- candidates (digit 1 == b1) and per-warp counts above b1 ----
    uint32_t mine = 0, above = 0;
    t2_for_keys(keys, [&](int j, uint32_t kj) {
        const uint32_t d = kj ? kj >> 20 : 0u;  // empty slots: never above, never candidates
        mine |= (uint32_t)(kj != 0u && d == b1) << j;
        above += __popc(__ballot_sync(0xffffffffu, kj != 0u && d > b1));
    });
    {
        const uint32_t c = __popc(mine);
        uint32_t pre = c;  // inclusive prefix over lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
        uint32_t base = 0;
        if (lane == 0) {
            S.wab[warp] = above;
            if (total) base = atomicAdd(&P.pub[0], total);
        }
        uint32_t slot = __shfl_sync(0xffffffffu, base, 0) + pre - c;
        for (uint32_t m = mine; m; m &= m - 1, ++slot) {
            const int j = __ffs(m) - 1;
            if (slot < kRxCtaCand) {
                P.ckey[slot] = keys(j);
                P.cidx[slot] = s0 + wbase + 32 * j + lane;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t a = 0;
        for (int w = 0; w < NT / 32; ++w) a += S.wab[w];
        P.pub[1] = a;
    }
    T2_MARK(10);
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    T2_MARK(11);
    if (tid < nct) {
        const uint32_t* pp = cluster.map_shared_rank(P.pub, tid);
        S.cn[tid] = pp[0];
        S.ca[tid] = pp[1];
    }
    __syncthreads();
    uint32_t n = 0;
    bool over = b1 == ~0u;
    for (int r = 0; r < nct; ++r) {
        over |= S.cn[r] > kRxCtaCand;
        n += S.cn[r];
    }
    over |= n > kRxCand;
    if (over) {  // cluster-uniform
        R.fallback = true;
        return R;
    }
    // ---- all candidates of the row, identical in every CTA ----
    for (uint32_t i = tid; i < n; i += NT) {
        int r = 0;
        uint32_t base = 0;
        while (i >= base + S.cn[r]) base += S.cn[r++];
        S.mkey[0][i] = cluster.map_shared_rank(P.ckey, r)[i - base];
        S.midx[0][i] = cluster.map_shared_rank(P.cidx, r)[i - base];
    }
    __syncthreads();
    T2_MARK(12);
    // ---- refine by digits 2 and 3 of the key, then rank; big exact-tie groups by the index ----
    const uint32_t* ck = S.mkey[0];
    const int32_t* ci = S.midx[0];
    int buf = 1;
#pragma unroll 1
    for (int lvl = 0; lvl < 3 && n > 32u; ++lvl) {  // key bits 19..12, 11..4, 3..0
        const int sh = lvl == 0 ? 12 : (lvl == 1 ? 4 : 0);
        const uint32_t msk = lvl == 2 ? 0xFu : 0xFFu;
        n = rx_refine<NT, 256>(S, ck, ci, n, S.mkey[buf], S.midx[buf], krem,
                               [sh, msk](uint32_t kk, int32_t) { return (kk >> sh) & msk; });
        ck = S.mkey[buf];
        ci = S.midx[buf];
        buf ^= 3;  // 1 <-> 2
    }
    if (n > 32u) {
        // n > 32 keys all equal to T: keep the krem lowest indices -> the krem-th largest of ~idx
        const uint32_t T = ck[0];
#pragma unroll 1
        for (int lvl = 0; lvl < 4 && n > 1u; ++lvl) {
            const int sh = 24 - 8 * lvl;
            n = rx_refine<NT, 256>(S, ck, ci, n, S.mkey[buf], S.midx[buf], krem,
                                   [sh](uint32_t, int32_t ii) { return (~(uint32_t)ii >> sh) & 0xFFu; });
            ck = S.mkey[buf];
            ci = S.midx[buf];
            buf ^= 3;
        }
        if (tid == 0) {
            S.res[4] = T;
            S.res[5] = (uint32_t)ci[0];
        }
        __syncthreads();
    } else {
        rx_rank32(S, ck, ci, n, krem);
    }
    R.T = S.res[4];
    R.idxT = (int32_t)S.res[5];
    T2_MARK(13);
    // ---- kept counts: per CTA (from the shared list), per warp (from this CTA's list) ----
    const uint32_t T = R.T;
    const int32_t idxT = R.idxT;
    const uint32_t n0 = [&] {
        uint32_t t = 0;
        for (int r = 0; r < nct; ++r) t += S.cn[r];
        return t;
    }();
    for (uint32_t i = tid; i < n0; i += NT) {
        const uint32_t kk = S.mkey[0][i];
        const int32_t ii = S.midx[0][i];
        if (kk > T || (kk == T && ii <= idxT)) atomicAdd(&S.ck[ii / slice], 1u);
    }
    for (uint32_t i = tid; i < S.cn[rank]; i += NT) {
        const uint32_t kk = P.ckey[i];
        const int32_t ii = P.cidx[i];
        if (kk > T || (kk == T && ii <= idxT)) atomicAdd(&S.wkc[(ii - s0) / (32 * kpt)], 1u);
    }
    __syncthreads();
    uint32_t cb = 0;
    for (int r = 0; r < rank; ++r) cb += S.ca[r] + S.ck[r];
    R.cta_base = cb;
    R.cta_count = S.ca[rank] + S.ck[rank];
    return R;
}

// Emit pass: emit(slot, j) for every kept key j of this thread (slot = position in the
// row's ascending selection).
template <int NT, typename Keys, typename Emit>
__device__ __forceinline__ void rx_emit(const Keys& keys, const RxResult& R, int s0, int wbase, RxShared& S,
                                        Emit&& emit) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t run = R.cta_base;
    for (int w = 0; w < warp; ++w) run += S.wab[w] + S.wkc[w];
    const uint32_t lt = t2_lanemask_lt();
    const uint32_t T = R.T;
    const int32_t idxT = R.idxT;
    uint32_t kept = 0;  // stage 1: this lane's kept slots (keys.count() <= 32), branch-free
    t2_for_keys(keys, [&](int j, uint32_t kj) {
        const int32_t idx = s0 + wbase + 32 * j + lane;
        kept |= (uint32_t)(kj > T || (kj == T && idx <= idxT)) << j;
    });
    const int n = keys.count();  // stage 2: positions by ballots, no key reads
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
        const bool kb = (kept >> j) & 1u;
        const uint32_t m = __ballot_sync(0xffffffffu, kb);
        if (kb) emit(run + __popc(m & lt), j);
        run += __popc(m);
    }
}

// ---- split variant (the fused decode step) -----------------------------------------
// After the second cluster barrier the CTA splits in two: the gather warps start the
// attention over the keys above b1 -- certainly kept, since fewer than k keys of the
// row lie above bin b1 -- while the select warps resolve the candidates (digit 1 ==
// b1), append this CTA's kept candidates to the gather list and write the selection
// from per-(warp, slot) lane masks.  Candidate overflow is decided before the split,
// from the merged and the per-CTA counts of bin b1 (cluster-uniform), and then the
// exact MSD path of select.cuh runs instead, with every warp.

struct RxFind {
    uint32_t b1, krem;
    bool over;
};

// Sum and per-element max over the cluster's CTAs of two consecutive u32 words.
__device__ __forceinline__ uint2 rx_cluster_sum2_max(uint32_t a, int nct, uint2* mx) {
    uint2 t = make_uint2(0u, 0u), m = make_uint2(0u, 0u);
    for (int r0 = 0; r0 < nct; r0 += 4) {
        uint2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            v[u] = make_uint2(0u, 0u);
            if (r0 + u < nct) {
                uint32_t ra;
                asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r0 + u));
                asm volatile("ld.shared::cluster.v2.u32 {%0,%1}, [%2];" : "=r"(v[u].x), "=r"(v[u].y) : "r"(ra));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            t.x += v[u].x;
            t.y += v[u].y;
            m.x = max(m.x, v[u].x);
            m.y = max(m.y, v[u].y);
        }
    }
    *mx = m;
    return t;
}

// All NT threads: cluster barrier 1, then bin b1 of digit 1 holding the k-th largest,
// krem = its rank inside b1, and the overflow decision.
// Cluster barrier 1 is the mbarrier `cbar` of every CTA (nct arrivals, phase 0): warp 0
// arrives on all of them and waits on its own; the other warps follow at CTA scope.
// Warp 0 also arrives on every CTA's cbar[3] once its DSMEM reads of the peers'
// histograms are done.
template <int NT>
__device__ __forceinline__ RxFind rx_find(int nct, int k, RxShared& S, RxPublished& P, uint64_t* cbar) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __syncthreads();  // this CTA's histogram is complete
    T2_MARK(17);
    for (int c = warp; c < 64; c += NT / 32) {  // coarse bins: 64 fine bins each, two per lane
        const uint2 v = reinterpret_cast<const uint2*>(S.hist + 64 * c)[lane];
        uint32_t x = v.x + v.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S.coarse[c] = x;
    }
    __syncthreads();
    if (warp == 0) {
        if (lane < nct) mbar_arrive_remote(smem_u32(cbar), lane);
        mbar_wait(cbar, 0);
    }
    T2_MARK(8);
    if (tid < kT2MaxCluster) S.ck[tid] = 0u;
    if (tid == 32) {
        P.pub[0] = 0u;
        S.nkept = 0u;
    }
    if (warp == 0) {
        uint32_t ab = 0, kr = (uint32_t)k;
        int b = -1;
        bool over = true;
        const uint2 cc = rx_cluster_sum2(smem_u32(S.coarse) + 8u * lane, nct);
        const int cb = rx_warp_find64(cc.x, cc.y, kr, &ab);
        if (cb >= 0) {
            kr -= ab;
            uint2 mx;
            const uint2 ff = rx_cluster_sum2_max(smem_u32(S.hist + 64 * cb) + 8u * lane, nct, &mx);
            const int fb = rx_warp_find64(ff.x, ff.y, kr, &ab);
            if (fb >= 0) {  // warp-uniform
                b = 64 * cb + fb;
                kr -= ab;
                const uint32_t n = __shfl_sync(0xffffffffu, (fb & 1) ? ff.y : ff.x, fb >> 1);
                const uint32_t m = __shfl_sync(0xffffffffu, (fb & 1) ? mx.y : mx.x, fb >> 1);
                over = n > (uint32_t)kRxCand || m > (uint32_t)kRxCtaCand;  // = rx_threshold's test
            }
        }
        // this CTA is done reading its peers' histograms: barrier cbar[3] (nct arrivals)
        // lets a peer overwrite them (the fused step's rings) before cluster barrier 2
        if (lane < nct) mbar_arrive_remote(smem_u32(cbar + 3), lane);
        if (lane == 0) {
            S.res[0] = (uint32_t)b;
            S.res[1] = kr;
            S.over = over ? 1u : 0u;
        }
    }
    __syncthreads();
    T2_MARK(14);
    return RxFind{S.res[0], S.res[1], S.over != 0u};
}

// All NT threads, one pass over the keys: candidates -> P (published); keys above b1 ->
// lane masks amask[warp * kpt + j] and this CTA's gather list alist[0 .. nabove) in index
// order; kmask zeroed; P.pub[1] = S.nabove.  The caller's cluster barrier 2 follows.
template <int NT, typename Keys>
__device__ __forceinline__ void rx_partition(const Keys& keys, int s0, int wbase, uint32_t b1, RxShared& S,
                                             RxPublished& P, uint32_t* amask, uint32_t* kmask, uint16_t* alist) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kpt = keys.count();
    uint32_t mine = 0, fa = 0, myw = 0;  // lane j keeps the above-mask of slot j
    t2_for_keys(keys, [&](int j, uint32_t kj) {
        const uint32_t d = kj ? kj >> 20 : 0u;  // empty slots: never above, never candidates
        mine |= (uint32_t)(kj != 0u && d == b1) << j;
        const bool a = kj != 0u && d > b1;
        fa |= (uint32_t)a << j;
        const uint32_t m = __ballot_sync(0xffffffffu, a);
        myw = lane == j ? m : myw;
    });
    const uint32_t na = __popc(fa);
    uint32_t pa = na;  // inclusive prefix over lanes of the keys above b1
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, pa, o);
        if (lane >= o) pa += y;
    }
    const uint32_t above = __shfl_sync(0xffffffffu, pa, 31);
    T2_MARK(18);
    if (lane < kpt) {
        amask[warp * kpt + lane] = myw;
        kmask[warp * kpt + lane] = 0u;
    }
    {
        const uint32_t c = __popc(mine);
        uint32_t pre = c;  // inclusive prefix over lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
        uint32_t base = 0;
        if (lane == 0) {
            S.wab[warp] = above;
            if (total) base = atomicAdd(&P.pub[0], total);
        }
        uint32_t slot = __shfl_sync(0xffffffffu, base, 0) + pre - c;
        for (uint32_t m = mine; m; m &= m - 1, ++slot) {
            const int j = __ffs(m) - 1;
            if (slot < kRxCtaCand) {
                P.ckey[slot] = keys(j);
                P.cidx[slot] = s0 + wbase + 32 * j + lane;
            }
        }
    }
    T2_MARK(19);
    __syncthreads();
    T2_MARK(20);
    // the gather list: each lane writes its own keys above b1 (a set-bit loop) at its
    // warp's offset + its exclusive prefix -- lane-major inside a warp (the attention does
    // not need index order; the selection itself is written from the per-slot masks)
    uint32_t run = 0;
    for (int w = 0; w < warp; ++w) run += S.wab[w];
    uint32_t o = run + pa - na;
    for (uint32_t m = fa; m; m &= m - 1) alist[o++] = (uint16_t)(wbase + 32 * (__ffs(m) - 1) + lane);
    if (tid == NT - 1) {  // the last warp's end is the CTA's total
        P.pub[1] = run + above;
        S.nabove = run + above;
    }
}

// The select warps (NT threads, barrier Bar), after cluster barrier 2: all candidates of
// the row -> (T, idx_T) -> kept counts per CTA; this CTA's kept candidates -> kmask bits
// and klist[0 .. S.nkept) (any order).
template <int NT, typename Bar>
__device__ __forceinline__ RxResult rx_resolve(cg::cluster_group& cluster, int s0, int slice, uint32_t krem,
                                               RxShared& S, RxPublished& P, uint32_t* kmask, uint16_t* klist) {
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31;
    RxResult R = {false, 0u, 0, 0u, 0u};
    if (tid < nct) {
        const uint32_t* pp = cluster.map_shared_rank(P.pub, tid);
        S.cn[tid] = pp[0];
        S.ca[tid] = pp[1];
    }
    Bar::sync();
    uint32_t n = 0, off = 0;
    for (int r = 0; r < nct; ++r) {
        if (r == rank) off = n;
        n += S.cn[r];
    }
    const uint32_t n0 = n, nmine = S.cn[rank];
    for (uint32_t i = tid; i < n; i += NT) {  // all candidates of the row, rank-ordered
        int r = 0;
        uint32_t base = 0;
        while (i >= base + S.cn[r]) base += S.cn[r++];
        S.mkey[0][i] = cluster.map_shared_rank(P.ckey, r)[i - base];
        S.midx[0][i] = cluster.map_shared_rank(P.cidx, r)[i - base];
    }
    Bar::sync();
    T2_MARK(12);
    const uint32_t* ck = S.mkey[0];
    const int32_t* ci = S.midx[0];
    int buf = 1;
#pragma unroll 1
    for (int lvl = 0; lvl < 3 && n > 32u; ++lvl) {  // key bits 19..12, 11..4, 3..0
        const int sh = lvl == 0 ? 12 : (lvl == 1 ? 4 : 0);
        const uint32_t msk = lvl == 2 ? 0xFu : 0xFFu;
        n = rx_refine<NT, 256, Bar>(S, ck, ci, n, S.mkey[buf], S.midx[buf], krem,
                                    [sh, msk](uint32_t kk, int32_t) { return (kk >> sh) & msk; });
        ck = S.mkey[buf];
        ci = S.midx[buf];
        buf ^= 3;
    }
    if (n > 32u) {  // > 32 keys all equal to T: the krem lowest indices (digits of ~idx)
        const uint32_t T = ck[0];
#pragma unroll 1
        for (int lvl = 0; lvl < 4 && n > 1u; ++lvl) {
            const int sh = 24 - 8 * lvl;
            n = rx_refine<NT, 256, Bar>(S, ck, ci, n, S.mkey[buf], S.midx[buf], krem,
                                        [sh](uint32_t, int32_t ii) { return (~(uint32_t)ii >> sh) & 0xFFu; });
            ck = S.mkey[buf];
            ci = S.midx[buf];
            buf ^= 3;
        }
        if (tid == 0) {
            S.res[4] = T;
            S.res[5] = (uint32_t)ci[0];
        }
        Bar::sync();
    } else {
        rx_rank32<Bar>(S, ck, ci, n, krem);
    }
    const uint32_t T = S.res[4];
    const int32_t idxT = (int32_t)S.res[5];
    R.T = T;
    R.idxT = idxT;
    T2_MARK(13);
    for (uint32_t i = tid; i < n0; i += NT) {
        const uint32_t kk = S.mkey[0][i];
        const int32_t ii = S.midx[0][i];
        if (kk > T || (kk == T && ii <= idxT)) atomicAdd(&S.ck[ii / slice], 1u);
    }
    const uint32_t lt = t2_lanemask_lt();
    for (uint32_t i0 = 0; i0 < nmine; i0 += NT) {
        const uint32_t i = i0 + tid;
        bool kp = false;
        int local = 0;
        if (i < nmine) {
            const uint32_t kk = S.mkey[0][off + i];
            const int32_t ii = S.midx[0][off + i];
            kp = kk > T || (kk == T && ii <= idxT);
            local = ii - s0;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, kp);
        if (m) {
            const int src = __ffs(m) - 1;
            uint32_t base = 0;
            if (lane == src) base = atomicAdd(&S.nkept, (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, src);
            if (kp) {
                klist[base + __popc(m & lt)] = (uint16_t)local;
                atomicOr(&kmask[local >> 5], 1u << (local & 31));
            }
        }
    }
    Bar::sync();
    uint32_t cb = 0;
    for (int r = 0; r < rank; ++r) cb += S.ca[r] + S.ck[r];
    R.cta_base = cb;
    R.cta_count = S.ca[rank] + S.ck[rank];
    return R;
}

// The select warps: emit(slot, kw, j) for every kept key (key-warp kw < KW, slot j, this
// lane) from amask | kmask, slots ascending with the index.
template <int NT, int KW, int KMAX, typename Bar, typename Emit>
__device__ __forceinline__ void rx_emit_masks(const RxResult& R, int kpt, const uint32_t* amask,
                                              const uint32_t* kmask, RxShared& S, Emit&& emit) {
    static_assert(KW <= 32, "");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) {
        uint32_t c = 0;
        if (lane < KW) {
            c = S.wab[lane];
#pragma unroll
            for (int j = 0; j < KMAX; ++j)
                if (j < kpt) c += __popc(kmask[lane * kpt + j]);
        }
        uint32_t pre = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
        }
        if (lane < KW) S.wsum[lane] = pre - c;
    }
    Bar::sync();
    const uint32_t lt = t2_lanemask_lt();
    for (int kw = warp; kw < KW; kw += NT / 32) {
        uint32_t run = R.cta_base + S.wsum[kw];
        // every slot's mask loaded first: one shared-memory latency per key-warp instead of kpt
        // (the fused step: 30.63 -> 30.30 us, the emit runs next to the gather warps)
        uint32_t mm[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) mm[j] = j < kpt ? (amask[kw * kpt + j] | kmask[kw * kpt + j]) : 0u;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            if ((mm[j] >> lane) & 1u) emit(run + __popc(mm[j] & lt), kw, j);
            run += __popc(mm[j]);
        }
    }
}

}  // namespace fier_cuda
