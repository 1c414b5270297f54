// topk2.cu -- K3 (register path): per-row Top-k with one wide histogram pass.
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores, ties
// to the LOWER index, returned in ascending index order.
//
// One thread-block cluster of C <= 16 CTAs (512 threads each) per row; CTA r keeps
// its slice in registers (KPT keys per thread; warp w owns the contiguous run
// [w*32*KPT, (w+1)*32*KPT) of the slice, slot j of lane L = 32j + L).
//   1. (lo, hi) = min / max of the finite scores (cluster exchange).
//   2. One 512-bin linear histogram over [lo, hi] (shared-memory atomics; the
//      bins are a monotone function of the value, so everything in a higher bin
//      is strictly larger), merged over the cluster through DSMEM -> bin b*
//      holding the k-th largest, krem = k - #(bins above b*).
//   3. Candidates = the keys in b* (typically ~L/300), gathered from every CTA.
//      While there are more than 32 of them, a sub-histogram over their own
//      [min, max] narrows them (all equal -> pure index tie).
//   4. Exact rank of the remaining <= 32 candidates by (value desc, index asc)
//      in one warp (shuffles): the krem-th is (T, idx_T); ties with T kept =
//      those with index <= idx_T.
//   5. Compaction in index order with ballots: kept iff key > T or (key == T and
//      tie rank < kept ties); slot = #(> T before) + min(#(== T before), ties).
// Degenerate rows (no finite spread, +-inf range, candidate overflow) take an
// exact 3-pass MSD radix select on the order-preserving u32 keys instead.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include <cstdio>
__device__ unsigned long long g_trace[4096][16];
#define FIER_TRACE(i) do { if (threadIdx.x == 0) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_trace[blockIdx.y * 16 + blockIdx.x][i] = t; } } while (0)


namespace cg = cooperative_groups;

namespace fier_cuda {

constexpr int kT2Threads = 512;
constexpr int kT2Warps = kT2Threads / 32;
constexpr int kT2MaxCluster = 16;  // 16 needs the non-portable cluster size opt-in
constexpr int kT2Bins = 512;  // one bin per thread: the DSMEM merge reads C words per thread
constexpr int kT2CtaCand = 1024;  // candidates one CTA may contribute
constexpr int kT2Cand = 2048;     // merged candidates per row

struct T2Shared {
    float mm[kT2MaxCluster][2];         // pushed (min, max) of every CTA
    alignas(16) uint32_t hist[kT2Bins];  // this CTA's histogram (read remotely)
    alignas(16) uint32_t tot[kT2Bins];   // merged histogram / scratch
    uint32_t ncand;                     // this CTA's candidate count (read remotely)
    uint32_t ckey[kT2CtaCand];          // this CTA's candidates (read remotely)
    int32_t cidx[kT2CtaCand];
    uint32_t mkey[2][kT2Cand];          // merged candidates (ping-pong for refinement)
    int32_t midx[2][kT2Cand];
    uint32_t wsum[32];
    uint32_t wsuf[32];
    uint32_t wg[kT2Warps], we[kT2Warps];  // per-warp (> T, == T) counts
    uint32_t cgt[kT2MaxCluster], ceq[kT2MaxCluster];  // pushed per-CTA (> T, == T) counts
    uint32_t cn[kT2MaxCluster];                        // candidate counts of every CTA
    uint32_t res[8];
    float fr[2 * kT2Warps];
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

// Over bins held in cnt[0..kT2Bins) (smem), find b with above(b) < krem <= above(b) + cnt[b],
// above(b) = sum of bins > b.  Writes (b, above) to res[0..1] (res[0] = ~0u if none).
__device__ __forceinline__ void t2_find_bin(const uint32_t* cnt, uint32_t krem, T2Shared& S) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int BPT = kT2Bins / kT2Threads;  // bins per thread (4)
    if (tid == 0) S.res[0] = ~0u;
    uint32_t cb[BPT];
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
        cb[i] = cnt[BPT * tid + i];
        c += cb[i];
    }
    uint32_t s = c;  // inclusive suffix within the warp (higher lanes own higher bins)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, s, o);
        if (lane + o < 32) s += y;
    }
    if (lane == 0) S.wsum[warp] = s;
    __syncthreads();
    if (warp == 0) {  // exclusive suffix scan of the warp totals
        const uint32_t v = lane < kT2Warps ? S.wsum[lane] : 0u;
        uint32_t t = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(0xffffffffu, t, o);
            if (lane + o < 32) t += y;
        }
        if (lane < kT2Warps) S.wsuf[lane] = t - v;
    }
    __syncthreads();
    uint32_t a = S.wsuf[warp] + s - c;  // count above this thread's highest bin
#pragma unroll
    for (int i = BPT - 1; i >= 0; --i) {
        if (a < krem && krem <= a + cb[i]) {
            S.res[0] = BPT * tid + i;
            S.res[1] = a;
        }
        a += cb[i];
    }
    __syncthreads();
}

// tot[i] = sum over the cluster's CTAs of hist[i]: 16-byte DSMEM loads by the first
// kT2Bins/4 threads (scattered 4-byte remote loads are throughput-bound).
__device__ __forceinline__ void t2_merge_hist(cg::cluster_group& cluster, int nct, uint32_t* hist, uint32_t* tot) {
    const int t = threadIdx.x;
    if (t < kT2Bins / 4) {
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

template <int KPT>
__global__ void __launch_bounds__(kT2Threads, 2) topk2_kernel(const float* __restrict__ scores, int tokens,
                                                              int64_t ld, int k, int slice,
                                                              int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* srow = scores + (int64_t)row * ld;
    const int s0 = rank * slice;
    const int cnt = max(0, min(s0 + slice, tokens) - s0);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    T2Shared& S = *reinterpret_cast<T2Shared*>(smem_raw);

    FIER_TRACE(0);
    // every CTA of the cluster must be running before anyone stores into its smem
    asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
    const int wbase = warp * 32 * KPT;
    // key 0 marks an empty slot (past the row end, or NaN): below every real key
    // (float_key(-inf) = 0x007fffff), so it is never counted or selected.
    uint32_t key[KPT];
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const int p = wbase + 32 * j + lane;
        const float v = p < cnt ? srow[s0 + p] : __int_as_float(0x7fffffff);
        key[j] = isnan(v) ? 0u : float_key(v);
        if (isfinite(v)) {
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
    }
    for (int i = tid; i < kT2Bins; i += kT2Threads) S.hist[i] = 0;
    mn = -warp_max(-mn);
    mx = warp_max(mx);
    if (lane == 0) {
        S.fr[warp] = mn;
        S.fr[kT2Warps + warp] = mx;
    }
    if (tid == 0) S.ncand = 0;
    __syncthreads();
    asm volatile("barrier.cluster.wait;" ::: "memory");
    FIER_TRACE(1);
    if (tid < nct) {
        float a = INFINITY, b = -INFINITY;
        for (int w = 0; w < kT2Warps; ++w) {
            a = fminf(a, S.fr[w]);
            b = fmaxf(b, S.fr[kT2Warps + w]);
        }
        float* dst = cluster.map_shared_rank(&S.mm[rank][0], tid);
        dst[0] = a;
        dst[1] = b;
    }
    cluster.sync();  // #1
    FIER_TRACE(2);
    float lo = INFINITY, hi = -INFINITY;
    for (int r = 0; r < nct; ++r) {
        lo = fminf(lo, S.mm[r][0]);
        hi = fmaxf(hi, S.mm[r][1]);
    }
    const float span = hi - lo;
    bool radix = !(span > 0.f) || !isfinite(span);  // cluster-uniform
    const float inv = radix ? 0.f : (float)kT2Bins / span;

    uint32_t T = 0, keep_ties = 0, ties = 0;  // threshold key, T-valued keys kept / present
    constexpr bool kCacheBin = KPT <= 16;
    uint16_t binc[kCacheBin ? KPT : 1];
    auto bin_of = [&](int j) -> int {
        if constexpr (kCacheBin) return (int)binc[j];
        return t2_bin(key_float(key[j]), lo, inv);
    };
    if (!radix) {
        // ---- 2. histogram ----
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            if (key[j]) {
                const int b = t2_bin(key_float(key[j]), lo, inv);
                if constexpr (kCacheBin) binc[j] = (uint16_t)b;
                atomicAdd(&S.hist[b], 1u);
            }
        }
        cluster.sync();  // #2
    FIER_TRACE(3);
        t2_merge_hist(cluster, nct, S.hist, S.tot);
        __syncthreads();
        t2_find_bin(S.tot, (uint32_t)k, S);
    FIER_TRACE(4);
        const uint32_t bstar = S.res[0];
        uint32_t krem = (uint32_t)k - S.res[1];
        // ---- 3. candidates of bin b* ----
        if (bstar != ~0u) {
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                const bool c = key[j] != 0u && bin_of(j) == (int)bstar;
                const uint32_t m = __ballot_sync(0xffffffffu, c);
                if (m) {
                    uint32_t base = 0;
                    if (lane == __ffs(m) - 1) base = atomicAdd(&S.ncand, (uint32_t)__popc(m));
                    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
                    const uint32_t slot = base + __popc(m & t2_lanemask_lt());
                    if (c && slot < kT2CtaCand) {
                        S.ckey[slot] = key[j];
                        S.cidx[slot] = s0 + wbase + 32 * j + lane;
                    }
                }
            }
        }
        cluster.sync();  // #3: candidate lists complete; merged histogram reads done
    FIER_TRACE(5);
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
            for (uint32_t i = tid; i < n; i += kT2Threads) {
                int r = 0;
                uint32_t base = 0;
                while (i >= base + S.cn[r]) base += S.cn[r++];
                S.mkey[0][i] = cluster.map_shared_rank(S.ckey, r)[i - base];
                S.midx[0][i] = cluster.map_shared_rank(S.cidx, r)[i - base];
            }
            __syncthreads();
            // ---- refinement: sub-histograms over the candidates' own range, down to one warp ----
    FIER_TRACE(6);
            int buf = 0;
            bool all_equal = false;
            for (int round = 0; n > 32u && !all_equal; ++round) {
                if (round == 4) {
                    radix = true;
                    break;
                }
                float cmn = INFINITY, cmx = -INFINITY;
                for (uint32_t i = tid; i < n; i += kT2Threads) {
                    const float v = key_float(S.mkey[buf][i]);
                    cmn = fminf(cmn, v);
                    cmx = fmaxf(cmx, v);
                }
                cmn = -warp_max(-cmn);
                cmx = warp_max(cmx);
                if (lane == 0) {
                    S.fr[warp] = cmn;
                    S.fr[kT2Warps + warp] = cmx;
                }
                for (int i = tid; i < kT2Bins; i += kT2Threads) S.tot[i] = 0;
                __syncthreads();
                cmn = INFINITY;
                cmx = -INFINITY;
                for (int w = 0; w < kT2Warps; ++w) {
                    cmn = fminf(cmn, S.fr[w]);
                    cmx = fmaxf(cmx, S.fr[kT2Warps + w]);
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
                for (uint32_t i = tid; i < n; i += kT2Threads)
                    atomicAdd(&S.tot[t2_bin(key_float(S.mkey[buf][i]), cmn, cinv)], 1u);
                __syncthreads();
                t2_find_bin(S.tot, krem, S);
                const int b2 = (int)S.res[0];
                krem -= S.res[1];
                if (tid == 0) S.res[2] = 0;
                __syncthreads();
                for (uint32_t i0 = 0; i0 < n; i0 += kT2Threads) {
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
                    T = S.mkey[buf][0];
                    keep_ties = krem;
                    ties = n;
                } else {
                    // ---- 4. exact rank of <= 32 candidates by (value desc, index asc): one warp ----
    FIER_TRACE(7);
                    if (warp == 0) {
                        const bool v = (uint32_t)lane < n;
                        const uint32_t ki = v ? S.mkey[buf][lane] : 0u;
                        const int32_t ii = v ? S.midx[buf][lane] : 0x7fffffff;
                        uint32_t rk = 0;
    FIER_TRACE(12);
                        for (uint32_t o = 0; o < n; ++o) {  // smem broadcast reads
                            const uint32_t kj = S.mkey[buf][o];
                            const int32_t ij = S.midx[buf][o];
                            rk += (kj > ki) || (kj == ki && ij < ii);
                        }
    FIER_TRACE(13);
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
    FIER_TRACE(11);
                    __syncthreads();
                    T = S.res[4];
                    keep_ties = S.res[3];
                    ties = S.res[6];
                }
            }
        }
    }
    if (radix) {
        // ---- exact MSD radix select on the order-preserving keys (9/9/9/5 bits) ----
        uint32_t prefix = 0, pmask = 0, kr = (uint32_t)k;
        uint32_t* h = S.hist;
#pragma unroll 1
        for (int pass = 0; pass < 4; ++pass) {
            const int shift = 23 - 9 * pass > 0 ? 23 - 9 * pass : 0;
            const int bins = pass == 3 ? 32 : 512;
            cluster.sync();  // remote readers of the previous histogram are done
            for (int i = tid; i < kT2Bins; i += kT2Threads) h[i] = 0;
            __syncthreads();
#pragma unroll
            for (int j = 0; j < KPT; ++j)
                if (key[j] && (key[j] & pmask) == prefix) atomicAdd(&h[(key[j] >> shift) & (bins - 1)], 1u);
            cluster.sync();
            t2_merge_hist(cluster, nct, h, S.tot);  // (bins beyond `bins` are zero everywhere)
            __syncthreads();
            t2_find_bin(S.tot, kr, S);
            kr -= S.res[1];
            if (pass == 3) ties = S.tot[S.res[0]];
            prefix |= S.res[0] << shift;
            pmask |= (uint32_t)(bins - 1) << shift;
        }
        T = prefix;
        keep_ties = kr;
    }

    // ---- 5. compaction in index order ----
    FIER_TRACE(8);
    // Common case: every T-valued key is kept -> kept iff key >= T, one ballot per slot.
    // Otherwise ties are ranked by index: kept iff key > T or (key == T and tie rank < keep_ties).
    const bool all_ties = keep_ties >= ties;  // cluster-uniform
    uint32_t g = 0, e = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        if (all_ties) {
            g += __popc(__ballot_sync(0xffffffffu, key[j] >= T));
        } else {
            g += __popc(__ballot_sync(0xffffffffu, key[j] > T));
            e += __popc(__ballot_sync(0xffffffffu, key[j] == T));
        }
    }
    if (lane == 0) {
        S.wg[warp] = g;
        S.we[warp] = e;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive prefix of the warp counts, and the CTA totals pushed to every CTA
        const uint32_t a = lane < kT2Warps ? S.wg[lane] : 0u, b = lane < kT2Warps ? S.we[lane] : 0u;
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
        if (lane < kT2Warps) {
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
    FIER_TRACE(9);
    uint32_t gb = 0, eb = 0;
    for (int r = 0; r < rank; ++r) {
        gb += S.cgt[r];
        eb += S.ceq[r];
    }
    uint32_t gt_run = gb + S.wsum[warp], eq_run = eb + S.wsuf[warp];
    int32_t* out = sel + (int64_t)row * k;
    const uint32_t lt = t2_lanemask_lt();
    if (all_ties) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const bool gg = key[j] >= T;
            const uint32_t mg = __ballot_sync(0xffffffffu, gg);
            if (gg) out[gt_run + __popc(mg & lt)] = s0 + wbase + 32 * j + lane;
            gt_run += __popc(mg);
        }
    } else {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const bool gg = key[j] > T, ee = key[j] == T;
            const uint32_t mg = __ballot_sync(0xffffffffu, gg);
            const uint32_t me = __ballot_sync(0xffffffffu, ee);
            const uint32_t my_gt = gt_run + __popc(mg & lt);
            const uint32_t my_eq = eq_run + __popc(me & lt);
            if (gg || (ee && my_eq < keep_ties)) out[my_gt + min(my_eq, keep_ties)] = s0 + wbase + 32 * j + lane;
            gt_run += __popc(mg);
            eq_run += __popc(me);
        }
    }
    FIER_TRACE(10);
}

template <int KPT>
static int launch_t2(int cluster, int rows, cudaStream_t st, const float* scores, int tokens, int64_t ld, int k,
                     int slice, int32_t* sel) {
    auto kern = topk2_kernel<KPT>;
    const size_t smem = sizeof(T2Shared);
    static bool attr = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(kT2Threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cluster;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, scores, tokens, ld, k, slice, sel);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

// Rows up to kT2MaxCluster * 512 * 32 keys.  Returns -1 if the row is too long.
int topk2_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st) {
    int c = 1;
    // grow the cluster until the grid covers the chip (or slices reach 8 keys per thread),
    // then until the slice fits the 32 registers per thread
    static const int max_c = [] {  // FIER_TOPK_CLUSTER caps the first growth step (tuning only)
        const char* e = getenv("FIER_TOPK_CLUSTER");
        return e ? atoi(e) : 8;
    }();
    while (c < max_c && (int64_t)rows * c < 2 * num_sms() && ceil_div(tokens, c) > 8 * kT2Threads) c *= 2;
    while (c < kT2MaxCluster && ceil_div(tokens, c) > 32 * kT2Threads) c *= 2;
    const int64_t slice = ceil_div(tokens, c);
    if (slice > 32 * kT2Threads) return -1;
    const int kpt = (int)ceil_div(slice, kT2Threads);
    if (kpt <= 1) return launch_t2<1>(c, rows, st, scores, tokens, ld, k, kT2Threads, sel);
    if (kpt <= 2) return launch_t2<2>(c, rows, st, scores, tokens, ld, k, 2 * kT2Threads, sel);
    if (kpt <= 4) return launch_t2<4>(c, rows, st, scores, tokens, ld, k, 4 * kT2Threads, sel);
    if (kpt <= 8) return launch_t2<8>(c, rows, st, scores, tokens, ld, k, 8 * kT2Threads, sel);
    if (kpt <= 16) return launch_t2<16>(c, rows, st, scores, tokens, ld, k, 16 * kT2Threads, sel);
    return launch_t2<32>(c, rows, st, scores, tokens, ld, k, 32 * kT2Threads, sel);
}

}  // namespace fier_cuda
