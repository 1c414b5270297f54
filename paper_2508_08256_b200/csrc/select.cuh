// select.cuh -- the cluster Top-k core of K3, shared by topk2.cu (scores read
// from memory) and step_fused.cu (scores produced in registers by the scorer).
//
// Reference: topk_oracle (core.hpp:134-148): the k largest scores, ties to the
// LOWER index, returned in ascending index order.
//
// One thread-block cluster of C <= 16 CTAs (NT = 256 or 512 threads each) per row; CTA r
// holds its slice as KPT keys per thread (warp w owns the contiguous run
// [w*32*KPT, (w+1)*32*KPT) of the slice, slot j of lane L = 32j + L), either in
// registers (RegKeys: compile-time KPT, loops fully unrolled) or in shared
// memory (SmemKeys: runtime KPT, compact loops -- for kernels whose phases each
// run once, where unrolled straight-line code would stream from a cold
// instruction cache).  Keys are order-preserving u32 (float_key); key 0 marks an empty
// slot (past the row end, or NaN) and is never counted or selected.
//   1. (lo, hi) = min / max of the finite scores (cluster exchange).
//   2. One 512-bin linear histogram over [lo, hi] (shared-memory atomics; the
//      bins are a monotone function of the value, so everything in a higher bin
//      is strictly larger), merged over the cluster through DSMEM -> bin b*
//      holding the k-th largest, krem = k - #(bins above b*).
//   3. Candidates = the keys in b* (typically ~L/300), gathered from every CTA.
//      While there are more than 32 of them, a sub-histogram over their own
//      [min, max] narrows them (all equal -> pure index tie).
//   4. Exact rank of the remaining <= 32 candidates by (value desc, index asc)
//      in one warp: the krem-th is (T, idx_T); ties with T kept = those with
//      index <= idx_T.
//   5. Compaction in index order with ballots: kept iff key > T or (key == T and
//      tie rank < kept ties); slot = #(> T before) + min(#(== T before), ties).
// Degenerate rows (no finite spread, +-inf range, candidate overflow) take an
// exact 9/9/9/5-bit MSD radix select on the keys instead.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

// Optional phase marks (a kernel's trace build defines T2_MARK before including this header).
#ifndef T2_MARK
#define T2_MARK(i) \
    do {           \
    } while (0)
#endif

namespace fier_cuda {

namespace cg = cooperative_groups;

constexpr int kT2Threads = 512;            // CTA size of the standalone K3 kernel
constexpr int kT2Warps = kT2Threads / 32;  // max warps per CTA (T2Shared sizing)
constexpr int kT2MaxCluster = 16;  // 16 needs the non-portable cluster size opt-in
constexpr int kT2Bins = 512;       // one bin per thread: the DSMEM merge reads C words per thread
constexpr int kT2CtaCand = 1024;   // candidates one CTA may contribute
constexpr int kT2Cand = 2048;      // merged candidates per row

struct T2Shared {
    float mm[kT2MaxCluster][2];          // pushed (min, max) of every CTA
    alignas(16) uint32_t hist[kT2Bins + 4];  // this CTA's histogram (read remotely); [kT2Bins] = trash
    alignas(16) uint32_t tot[kT2Bins];   // merged histogram / scratch
    uint32_t ncand;                      // this CTA's candidate count (read remotely)
    uint32_t ckey[kT2CtaCand];           // this CTA's candidates (read remotely)
    int32_t cidx[kT2CtaCand];
    uint32_t mkey[2][kT2Cand];  // merged candidates (ping-pong for refinement)
    int32_t midx[2][kT2Cand];
    uint32_t wsum[32];
    uint32_t wsuf[32];
    uint32_t wg[kT2Warps], we[kT2Warps];              // per-warp (> T, == T) counts
    uint32_t cgt[kT2MaxCluster], ceq[kT2MaxCluster];  // pushed per-CTA (> T, == T) counts
    uint32_t cn[kT2MaxCluster];                       // candidate counts of every CTA
    uint32_t res[8];
    float fr[2 * kT2Warps];
};

struct T2Threshold {
    uint32_t T;          // key of the k-th largest
    uint32_t keep_ties;  // T-valued keys kept (the lowest-index ones)
    uint32_t ties;       // T-valued keys present
};

__device__ __forceinline__ uint32_t t2_lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// inverse of float_key for finite/inf keys (the canonical +0 maps back to +0)
__device__ __forceinline__ float key_float(uint32_t k) {
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(u);
}

__device__ __forceinline__ int t2_bin(float x, float lo, float inv) {
    float t = (x - lo) * inv;
    t = fminf(fmaxf(t, 0.f), (float)(kT2Bins - 1));
    return (int)t;
}

// Key sources: keys(j) = key of slot j of this thread (0 = empty).
template <int KPT>
struct RegKeys {
    static constexpr int kStatic = KPT;
    const uint32_t (&k)[KPT];
    __device__ __forceinline__ uint32_t operator()(int j) const { return k[j]; }
    __device__ __forceinline__ int count() const { return KPT; }
};
struct SmemKeys {
    static constexpr int kStatic = 0;
    const uint32_t* run;  // this warp's run: slot j of lane L at run[32*j + L]
    int n;                // slots per thread
    __device__ __forceinline__ uint32_t operator()(int j) const { return run[32 * j + (threadIdx.x & 31)]; }
    __device__ __forceinline__ int count() const { return n; }
};

// f(j, key of slot j) for every slot of this thread.  Shared-memory keys are read in
// batches of 8 before any use, so their load latency overlaps (the bodies contain
// shared-memory atomics, which the compiler will not move loads across).
template <typename Keys, typename F>
__device__ __forceinline__ void t2_for_keys(const Keys& keys, F&& f) {
    if constexpr (Keys::kStatic > 0) {
#pragma unroll
        for (int j = 0; j < Keys::kStatic; ++j) f(j, keys(j));
    } else {
        const int n = keys.count();
        int j0 = 0;
        for (; j0 + 8 <= n; j0 += 8) {
            uint32_t kk[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) kk[u] = keys(j0 + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) f(j0 + u, kk[u]);
        }
        for (; j0 < n; ++j0) f(j0, keys(j0));
    }
}

// Barriers of a thread group: the whole CTA, or the first N threads (named barrier ID).
struct CtaBar {
    __device__ static __forceinline__ void sync() { __syncthreads(); }
};
template <int ID, int N>
struct NamedBar {
    __device__ static __forceinline__ void sync() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory"); }
};

// Over bins held in cnt[0..kT2Bins) (smem), find b with above(b) < krem <= above(b) + cnt[b],
// above(b) = sum of bins > b.  Writes (b, above) to res[0..1] (res[0] = ~0u if none).
template <int NT, int BINS = kT2Bins, typename SH = T2Shared, typename Bar = CtaBar>
__device__ __forceinline__ void t2_find_bin(const uint32_t* cnt, uint32_t krem, SH& S) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int BPT = BINS >= NT ? BINS / NT : 1;  // bins per thread
    if (tid == 0) S.res[0] = ~0u;
    uint32_t cb[BPT];
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
        cb[i] = (BINS >= NT || BPT * tid + i < BINS) ? cnt[BPT * tid + i] : 0u;
        c += cb[i];
    }
    uint32_t s = c;  // inclusive suffix within the warp (higher lanes own higher bins)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, s, o);
        if (lane + o < 32) s += y;
    }
    if (lane == 0) S.wsum[warp] = s;
    Bar::sync();
    if (warp == 0) {  // exclusive suffix scan of the warp totals
        const uint32_t v = lane < NT / 32 ? S.wsum[lane] : 0u;
        uint32_t t = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(0xffffffffu, t, o);
            if (lane + o < 32) t += y;
        }
        if (lane < NT / 32) S.wsuf[lane] = t - v;
    }
    Bar::sync();
    uint32_t a = S.wsuf[warp] + s - c;  // count above this thread's highest bin
#pragma unroll
    for (int i = BPT - 1; i >= 0; --i) {
        if (a < krem && krem <= a + cb[i]) {
            S.res[0] = BPT * tid + i;
            S.res[1] = a;
        }
        a += cb[i];
    }
    Bar::sync();
}

// tot[i] = sum over the cluster's CTAs of hist[i]: 16-byte DSMEM loads
// (scattered 4-byte remote loads are throughput-bound).
template <int BINS = kT2Bins>
__device__ __forceinline__ void t2_merge_hist(cg::cluster_group& cluster, int nct, uint32_t* hist, uint32_t* tot) {
    for (int t = threadIdx.x; t < BINS / 4; t += blockDim.x) {
        uint4 a = make_uint4(0, 0, 0, 0);
        for (int r = 0; r < nct; ++r) {
            const uint4 v = reinterpret_cast<const uint4*>(cluster.map_shared_rank(hist, r))[t];
            a.x += v.x;
            a.y += v.y;
            a.z += v.z;
            a.w += v.w;
        }
        reinterpret_cast<uint4*>(tot)[t] = a;
    }
}

// Exact MSD radix select on the order-preserving keys (9/9/9/5-bit digits, one
// cluster barrier + DSMEM histogram merge per digit): the degenerate-row path.
template <int NT, typename Keys, typename SH>
__device__ __forceinline__ T2Threshold t2_radix_select(cg::cluster_group& cluster, const Keys& keys, int k, SH& S) {
    const int nct = (int)cluster.num_blocks();
    const int tid = threadIdx.x;
    T2Threshold res = {0u, 0u, 0u};
    uint32_t prefix = 0, pmask = 0, kr = (uint32_t)k;
    uint32_t* h = S.hist;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 23 - 9 * pass > 0 ? 23 - 9 * pass : 0;
        const int bins = pass == 3 ? 32 : 512;
        cluster.sync();  // remote readers of the previous histogram are done
        for (int i = tid; i < kT2Bins; i += NT) h[i] = 0;
        __syncthreads();
        t2_for_keys(keys, [&](int, uint32_t kj) {
            if (kj && (kj & pmask) == prefix) atomicAdd(&h[(kj >> shift) & (bins - 1)], 1u);
        });
        cluster.sync();
        t2_merge_hist(cluster, nct, h, S.tot);  // (bins beyond `bins` are zero everywhere)
        __syncthreads();
        t2_find_bin<NT>(S.tot, kr, S);
        kr -= S.res[1];
        if (pass == 3) res.ties = S.tot[S.res[0]];
        prefix |= S.res[0] << shift;
        pmask |= (uint32_t)(bins - 1) << shift;
    }
    res.T = prefix;
    res.keep_ties = kr;
    return res;
}

// Steps 1-4 (+ the radix fallback): the threshold of the k largest over the
// cluster's keys.  mn / mx = this thread's min / max over its finite scores.
// The caller must have executed `barrier.cluster.arrive` (no wait) before: the
// wait here is the first point where peers' shared memory is written.
// s0 + wbase + 32*j + lane is the row index of keys(j).
template <int NT, typename Keys>
__device__ __forceinline__ T2Threshold t2_threshold(cg::cluster_group& cluster, const Keys& keys,
                                                    float mn, float mx, int s0, int wbase, int k, T2Shared& S) {
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kT2Bins; i += NT) S.hist[i] = 0;
    mn = -warp_max(-mn);
    mx = warp_max(mx);
    if (lane == 0) {
        S.fr[warp] = mn;
        S.fr[NT / 32 + warp] = mx;
    }
    if (tid == 0) S.ncand = 0;
    __syncthreads();
    asm volatile("barrier.cluster.wait;" ::: "memory");
    if (tid < nct) {
        float a = INFINITY, b = -INFINITY;
        for (int w = 0; w < NT / 32; ++w) {
            a = fminf(a, S.fr[w]);
            b = fmaxf(b, S.fr[NT / 32 + w]);
        }
        float* dst = cluster.map_shared_rank(&S.mm[rank][0], tid);
        dst[0] = a;
        dst[1] = b;
    }
    cluster.sync();  // #1
    T2_MARK(8);
    float lo = INFINITY, hi = -INFINITY;
    for (int r = 0; r < nct; ++r) {
        lo = fminf(lo, S.mm[r][0]);
        hi = fmaxf(hi, S.mm[r][1]);
    }
    const float span = hi - lo;
    bool radix = !(span > 0.f) || !isfinite(span);  // cluster-uniform
    const float inv = radix ? 0.f : (float)kT2Bins / span;

    T2Threshold res = {0u, 0u, 0u};
    constexpr bool kCacheBin = Keys::kStatic > 0 && Keys::kStatic <= 16;
    uint16_t binc[kCacheBin ? Keys::kStatic : 1];
    auto bin_of = [&](int j) -> int {
        if constexpr (kCacheBin) return (int)binc[j];
        return t2_bin(key_float(keys(j)), lo, inv);
    };
    if (!radix) {
        // ---- 2. histogram ----
        t2_for_keys(keys, [&](int j, uint32_t kj) {  // branch-free: empty slots count into the trash bin
            const int b = t2_bin(key_float(kj), lo, inv);
            if constexpr (kCacheBin) binc[j] = (uint16_t)b;
            atomicAdd(&S.hist[kj ? b : kT2Bins], 1u);
        });
        T2_MARK(9);
        cluster.sync();  // #2
        T2_MARK(10);
        t2_merge_hist(cluster, nct, S.hist, S.tot);
        __syncthreads();
        t2_find_bin<NT>(S.tot, (uint32_t)k, S);
        T2_MARK(11);
        const uint32_t bstar = S.res[0];
        uint32_t krem = (uint32_t)k - S.res[1];
        // ---- 3. candidates of bin b* ----
        if (bstar != ~0u) {
            if constexpr (Keys::kStatic == 0) {
                // two stages: branch-free candidate masks (keys.count() <= 32), then the rare hits
                uint32_t mine = 0;
                t2_for_keys(keys, [&](int j, uint32_t kj) {
                    mine |= (uint32_t)(kj != 0u && t2_bin(key_float(kj), lo, inv) == (int)bstar) << j;
                });
                const uint32_t c = __popc(mine);
                uint32_t pre = c;  // inclusive prefix over lanes
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
                    if (lane >= o) pre += y;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
                if (total) {
                    uint32_t base = 0;
                    if (lane == 0) base = atomicAdd(&S.ncand, total);
                    uint32_t slot = __shfl_sync(0xffffffffu, base, 0) + pre - c;
                    for (uint32_t m = mine; m; m &= m - 1, ++slot) {
                        const int j = __ffs(m) - 1;
                        if (slot < kT2CtaCand) {
                            S.ckey[slot] = keys(j);
                            S.cidx[slot] = s0 + wbase + 32 * j + lane;
                        }
                    }
                }
            } else {
                t2_for_keys(keys, [&](int j, uint32_t kj) {
                    const bool c = kj != 0u && bin_of(j) == (int)bstar;
                    const uint32_t m = __ballot_sync(0xffffffffu, c);
                    if (m) {
                        uint32_t base = 0;
                        if (lane == __ffs(m) - 1) base = atomicAdd(&S.ncand, (uint32_t)__popc(m));
                        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
                        const uint32_t slot = base + __popc(m & t2_lanemask_lt());
                        if (c && slot < kT2CtaCand) {
                            S.ckey[slot] = kj;
                            S.cidx[slot] = s0 + wbase + 32 * j + lane;
                        }
                    }
                });
            }
        }
        T2_MARK(12);
        cluster.sync();  // #3: candidate lists complete; merged histogram reads done
        T2_MARK(13);
        if (tid < nct) S.cn[tid] = *cluster.map_shared_rank(&S.ncand, tid);
        __syncthreads();
        uint32_t n = 0;
        bool over = bstar == ~0u;
        for (int r = 0; r < nct; ++r) {
            const uint32_t c = S.cn[r];
            over |= c > kT2CtaCand;
            n += c;
        }
        over |= n > kT2Cand;
        radix = over;  // cluster-uniform
        if (!radix) {
            // flattened gather: every remote load of the merge is in flight at once
            for (uint32_t i = tid; i < n; i += NT) {
                int r = 0;
                uint32_t base = 0;
                while (i >= base + S.cn[r]) base += S.cn[r++];
                S.mkey[0][i] = cluster.map_shared_rank(S.ckey, r)[i - base];
                S.midx[0][i] = cluster.map_shared_rank(S.cidx, r)[i - base];
            }
            __syncthreads();
            T2_MARK(14);
            // ---- refinement: sub-histograms over the candidates' own range, down to one warp ----
            int buf = 0;
            bool all_equal = false;
            for (int round = 0; n > 32u && !all_equal; ++round) {
                if (round == 4) {
                    radix = true;
                    break;
                }
                float cmn = INFINITY, cmx = -INFINITY;
                for (uint32_t i = tid; i < n; i += NT) {
                    const float v = key_float(S.mkey[buf][i]);
                    cmn = fminf(cmn, v);
                    cmx = fmaxf(cmx, v);
                }
                cmn = -warp_max(-cmn);
                cmx = warp_max(cmx);
                if (lane == 0) {
                    S.fr[warp] = cmn;
                    S.fr[NT / 32 + warp] = cmx;
                }
                for (int i = tid; i < kT2Bins; i += NT) S.tot[i] = 0;
                __syncthreads();
                cmn = INFINITY;
                cmx = -INFINITY;
                for (int w = 0; w < NT / 32; ++w) {
                    cmn = fminf(cmn, S.fr[w]);
                    cmx = fmaxf(cmx, S.fr[NT / 32 + w]);
                }
                const float csp = cmx - cmn;
                if (!(csp > 0.f)) {  // every candidate has the same value: a pure index tie
                    all_equal = true;
                    break;
                }
                if (!isfinite(csp)) {
                    radix = true;
                    break;
                }
                const float cinv = (float)kT2Bins / csp;
                for (uint32_t i = tid; i < n; i += NT)
                    atomicAdd(&S.tot[t2_bin(key_float(S.mkey[buf][i]), cmn, cinv)], 1u);
                __syncthreads();
                t2_find_bin<NT>(S.tot, krem, S);
                const int b2 = (int)S.res[0];
                krem -= S.res[1];
                if (tid == 0) S.res[2] = 0;
                __syncthreads();
                for (uint32_t i0 = 0; i0 < n; i0 += NT) {
                    const uint32_t i = i0 + tid;
                    const bool c = i < n && t2_bin(key_float(S.mkey[buf][i]), cmn, cinv) == b2;
                    const uint32_t m = __ballot_sync(0xffffffffu, c);
                    if (m) {
                        uint32_t base = 0;
                        if (lane == __ffs(m) - 1) base = atomicAdd(&S.res[2], (uint32_t)__popc(m));
                        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
                        if (c) {
                            const uint32_t slot = base + __popc(m & t2_lanemask_lt());
                            S.mkey[buf ^ 1][slot] = S.mkey[buf][i];
                            S.midx[buf ^ 1][slot] = S.midx[buf][i];
                        }
                    }
                }
                __syncthreads();
                n = S.res[2];
                buf ^= 1;
            }
            if (!radix) {
                if (all_equal) {
                    res.T = S.mkey[buf][0];
                    res.keep_ties = krem;
                    res.ties = n;
                } else {
                    // ---- 4. exact rank of <= 32 candidates by (value desc, index asc): one warp ----
                    if (warp == 0) {
                        const bool v = (uint32_t)lane < n;
                        const uint32_t ki = v ? S.mkey[buf][lane] : 0u;
                        const int32_t ii = v ? S.midx[buf][lane] : 0x7fffffff;
                        uint32_t rk = 0;
                        for (uint32_t o = 0; o < n; ++o) {  // smem broadcast reads
                            const uint32_t kj = S.mkey[buf][o];
                            const int32_t ij = S.midx[buf][o];
                            rk += (kj > ki) || (kj == ki && ij < ii);
                        }
                        const uint32_t hit = __ballot_sync(0xffffffffu, v && rk == krem - 1);
                        const int src = __ffs(hit) - 1;  // unique
                        const uint32_t tk = __shfl_sync(0xffffffffu, ki, src);
                        const int32_t ti = __shfl_sync(0xffffffffu, ii, src);
                        const uint32_t tie = __ballot_sync(0xffffffffu, v && ki == tk);
                        const uint32_t kept = __ballot_sync(0xffffffffu, v && ki == tk && ii <= ti);
                        if (lane == 0) {
                            S.res[4] = tk;
                            S.res[3] = __popc(kept);
                            S.res[6] = __popc(tie);
                        }
                    }
                    __syncthreads();
                    res.T = S.res[4];
                    res.keep_ties = S.res[3];
                    res.ties = S.res[6];
                }
            }
        }
    }
    if (radix) res = t2_radix_select<NT>(cluster, keys, k, S);
    return res;
}

// Step 5: compaction in index order.  emit(slot, j) is called for every kept key
// j of this thread, slot = its position in the row's ascending selection.
// Returns this CTA's first slot in *cta_base and its kept count in *cta_count.
// Ends with a cluster barrier: after it no CTA touches a peer's shared memory.
template <int NT, typename Keys, typename Emit, typename SH>
__device__ __forceinline__ void t2_compact(cg::cluster_group& cluster, const Keys& keys,
                                           const T2Threshold& th, SH& S, uint32_t* cta_base,
                                           uint32_t* cta_count, Emit&& emit) {
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t T = th.T, keep_ties = th.keep_ties;
    // Common case: every T-valued key is kept -> kept iff key >= T, one ballot per slot.
    // Otherwise ties are ranked by index: kept iff key > T or (key == T and tie rank < keep_ties).
    const bool all_ties = keep_ties >= th.ties;  // cluster-uniform
    uint32_t g = 0, e = 0;
    if (all_ties) {
        t2_for_keys(keys, [&](int, uint32_t kj) { g += __popc(__ballot_sync(0xffffffffu, kj >= T)); });
    } else {
        t2_for_keys(keys, [&](int, uint32_t kj) {
            g += __popc(__ballot_sync(0xffffffffu, kj > T));
            e += __popc(__ballot_sync(0xffffffffu, kj == T));
        });
    }
    if (lane == 0) {
        S.wg[warp] = g;
        S.we[warp] = e;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive prefix of the warp counts, and the CTA totals pushed to every CTA
        const uint32_t a = lane < NT / 32 ? S.wg[lane] : 0u, b = lane < NT / 32 ? S.we[lane] : 0u;
        uint32_t ia = a, ib = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
            const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += ya;
                ib += yb;
            }
        }
        if (lane < NT / 32) {
            S.wsum[lane] = ia - a;
            S.wsuf[lane] = ib - b;
        }
        const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31), tb = __shfl_sync(0xffffffffu, ib, 31);
        if (lane < nct) {
            *cluster.map_shared_rank(&S.cgt[rank], lane) = ta;
            *cluster.map_shared_rank(&S.ceq[rank], lane) = tb;
        }
    }
    cluster.sync();  // also: no CTA leaves while others may still read its smem
    uint32_t gb = 0, eb = 0;
    for (int r = 0; r < rank; ++r) {
        gb += S.cgt[r];
        eb += S.ceq[r];
    }
    *cta_base = gb + min(eb, keep_ties);
    *cta_count = S.cgt[rank] + min(eb + S.ceq[rank], keep_ties) - min(eb, keep_ties);
    uint32_t gt_run = gb + S.wsum[warp], eq_run = eb + S.wsuf[warp];
    const uint32_t lt = t2_lanemask_lt();
    if (all_ties) {
        t2_for_keys(keys, [&](int j, uint32_t kj) {
            const bool gg = kj >= T;
            const uint32_t mg = __ballot_sync(0xffffffffu, gg);
            if (gg) emit(gt_run + __popc(mg & lt), j);
            gt_run += __popc(mg);
        });
    } else {
        t2_for_keys(keys, [&](int j, uint32_t kj) {
            const bool gg = kj > T, ee = kj == T;
            const uint32_t mg = __ballot_sync(0xffffffffu, gg);
            const uint32_t me = __ballot_sync(0xffffffffu, ee);
            const uint32_t my_gt = gt_run + __popc(mg & lt);
            const uint32_t my_eq = eq_run + __popc(me & lt);
            if (gg || (ee && my_eq < keep_ties)) emit(my_gt + min(my_eq, keep_ties), j);
            gt_run += __popc(mg);
            eq_run += __popc(me);
        });
    }
}

}  // namespace fier_cuda
