// topk_long.cu -- K3 for rows too long to keep on chip (C5: 1M tokens per row).
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores, ties to
// the LOWER index, ascending output.  One cluster of 16 CTAs (512 threads) per row;
// CTA r owns a contiguous slice of the row and streams it from memory three times:
//   pass 1  order-preserving keys -> 12-bit digit histogram (select_radix.cuh digit 1)
//           [cluster barrier] one warp merges the 64 coarse sums, then the 64 fine bins
//           of the coarse bin holding the k-th largest (DSMEM) -> bin b1, krem
//   pass 2  count the keys above b1; keys in b1 are candidates -> published list
//           [cluster barrier] every CTA gathers all candidates and refines them by
//           8-bit digits to the exact (T, idx_T) (index refinement for big tie groups);
//           kept counts of every CTA from the published lists -> this CTA's offset
//   pass 3  ordered emit: tiles of 2048 keys (4 consecutive per thread), block scan
//           of the kept flags, indices written at offset + running position.
// Three reads of the row (the C5 scores are 134 MB, beyond L2) instead of the old
// streaming kernel's eight.  Measured at C5 (32 x 1M, k = 4096): 347 us vs 361 us --
// only 7 clusters of 16 are co-resident (five waves), and each CTA's 65536 histogram
// atomics collide on the few hot bins of a 12-bit digit (~4000 keys share the k-th's
// bin); a 14-bit digit and fewer, larger clusters are the next step.  Candidate overflow (a digit-1 bin with > kTlCand keys)
// takes an exact streaming MSD radix select (9/9/9/5-bit digits) with index-ordered
// tie ranking instead.
#include <string>

#include "select_radix.cuh"

namespace fier_cuda {

constexpr int kTlThreads = 512;
constexpr int kTlCluster = 16;
constexpr int kTlCtaCand = 1024;
constexpr int kTlCand = 6144;
constexpr int kTlTile = 4 * kTlThreads;

struct TlShared {
    alignas(16) uint32_t hist[kRxBins + 4];
    alignas(16) uint32_t coarse[64];
    alignas(16) uint32_t tot[kT2Bins];
    uint32_t mkey[2][kTlCand];
    int32_t midx[2][kTlCand];
    uint32_t cn[kT2MaxCluster], ca[kT2MaxCluster], ck[kT2MaxCluster], ce[kT2MaxCluster];
    uint32_t wsum[32], wsuf[32];
    uint32_t res[8];
};

struct TlPublished {
    uint32_t pub[4];  // [0] candidates, [1] keys above b1 (fallback: [1] keys > T, [2] keys == T)
    uint32_t ckey[kTlCtaCand];
    int32_t cidx[kTlCtaCand];
};

// key of position i of a row ending at s1 (0: empty slot past the end)
__device__ __forceinline__ uint32_t tl_key(float v, int i, int s1) { return i < s1 ? score_key(v) : 0u; }

constexpr int kTlDepth = 8;  // tiles of loads in flight per thread (64 KB per SM)

// (an explicit branch: a select let the compiler issue the guarded scalar loads next to
// every vector load)
__device__ __forceinline__ float4 tl_load4(const float* srow, int i, int s1) {
    if (i + 3 < s1) return ldg_stream_f4(srow + i);
    float4 x = make_float4(__int_as_float(0x7fffffff), __int_as_float(0x7fffffff), __int_as_float(0x7fffffff),
                           __int_as_float(0x7fffffff));
    if (i < s1) x.x = srow[i];
    if (i + 1 < s1) x.y = srow[i + 1];
    if (i + 2 < s1) x.z = srow[i + 2];
    return x;
}

// f(key, index) for every key of [s0, s1) (s0 % 4 == 0), 4 consecutive keys per thread
// per tile, kTlDepth tiles of loads in flight (one CTA per SM: the latency needs them).
template <typename F>
__device__ __forceinline__ void tl_stream(const float* srow, int s0, int s1, F&& f) {
    for (int t0 = s0; t0 < s1; t0 += kTlDepth * kTlTile) {
        float4 v[kTlDepth];
#pragma unroll
        for (int u = 0; u < kTlDepth; ++u) v[u] = tl_load4(srow, t0 + u * kTlTile + 4 * threadIdx.x, s1);
#pragma unroll
        for (int u = 0; u < kTlDepth; ++u) {
            const int i = t0 + u * kTlTile + 4 * threadIdx.x;
            f(tl_key(v[u].x, i, s1), i);
            f(tl_key(v[u].y, i + 1, s1), i + 1);
            f(tl_key(v[u].z, i + 2, s1), i + 2);
            f(tl_key(v[u].w, i + 3, s1), i + 3);
        }
    }
}

// Block-wide exclusive scan of one count per thread; returns the prefix, the tile total in *tot.
__device__ __forceinline__ uint32_t tl_scan(uint32_t v, TlShared& S, uint32_t* tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) S.wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < kTlThreads / 32 ? S.wsum[lane] : 0u;
        uint32_t z = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < kTlThreads / 32) S.wsuf[lane] = z - w;
        if (lane == kTlThreads / 32 - 1) S.res[7] = z;
    }
    __syncthreads();
    *tot = S.res[7];
    const uint32_t r = S.wsuf[warp] + x - v;
    __syncthreads();  // wsum / wsuf / res[7] are rewritten by the next tile
    return r;
}

// Pass 3: kept(key, index, eq_rank) -> ascending positions from `base`.  RANKED: the rule
// needs eq_rank = index-order rank among the row's T-valued keys (eq_base = those of
// earlier CTAs); else eq_rank is not computed.
template <bool RANKED, typename Kept>
__device__ __forceinline__ void tl_emit(const float* srow, int s0, int s1, uint32_t T, uint32_t base,
                                        uint32_t eq_base, TlShared& S, int32_t* out, Kept&& kept) {
    uint32_t run = 0, eq_run = eq_base;
    constexpr int DEP = 4;  // tiles loaded ahead
    for (int b0 = s0; b0 < s1; b0 += DEP * kTlTile) {
      float4 vv[DEP];
#pragma unroll
      for (int u = 0; u < DEP; ++u) vv[u] = tl_load4(srow, b0 + u * kTlTile + 4 * threadIdx.x, s1);
#pragma unroll 1
      for (int u = 0; u < DEP; ++u) {
        const int t0 = b0 + u * kTlTile;
        if (t0 >= s1) break;  // block-uniform
        const int i = t0 + 4 * threadIdx.x;
        float4 v = vv[0];
#pragma unroll
        for (int w = 1; w < DEP; ++w) v = u == w ? vv[w] : v;
        const uint32_t kk[4] = {tl_key(v.x, i, s1), tl_key(v.y, i + 1, s1), tl_key(v.z, i + 2, s1),
                                tl_key(v.w, i + 3, s1)};
        uint32_t tot = 0, eq_pre = 0;
        if constexpr (RANKED) {
            uint32_t neq = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) neq += kk[j] == T && kk[j] != 0u;
            eq_pre = eq_run + tl_scan(neq, S, &tot);
            eq_run += tot;
        }
        uint32_t flags = 0, cnt = 0, e = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool isT = kk[j] == T && kk[j] != 0u;
            const bool kb = kk[j] != 0u && kept(kk[j], i + j, eq_pre + e);
            e += isT;
            flags |= (uint32_t)kb << j;
            cnt += kb;
        }
        const uint32_t pos = run + tl_scan(cnt, S, &tot);
        run += tot;
        uint32_t o = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((flags >> j) & 1u) out[base + pos + o++] = i + j;
      }
    }
}

// Exact streaming MSD radix select (9/9/9/5-bit digits) -> (T, kept ties); the candidate-
// overflow path.
__device__ __noinline__ void tl_radix(cg::cluster_group& cluster, const float* srow, int s0, int s1, int k,
                                      TlShared& S, uint32_t* T_out, uint32_t* keep_out) {
    const int nct = (int)cluster.num_blocks();
    uint32_t prefix = 0, pmask = 0, kr = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 23 - 9 * pass > 0 ? 23 - 9 * pass : 0;
        const int bins = pass == 3 ? 32 : 512;
        cluster.sync();  // remote readers of the previous histogram are done
        for (int i = threadIdx.x; i < kT2Bins; i += kTlThreads) S.hist[i] = 0;
        __syncthreads();
        tl_stream(srow, s0, s1, [&](uint32_t kj, int) {
            if (kj && (kj & pmask) == prefix) atomicAdd(&S.hist[(kj >> shift) & (bins - 1)], 1u);
        });
        cluster.sync();
        t2_merge_hist(cluster, nct, S.hist, S.tot);
        __syncthreads();
        t2_find_bin<kTlThreads>(S.tot, kr, S);
        kr -= S.res[1];
        prefix |= S.res[0] << shift;
        pmask |= (uint32_t)(bins - 1) << shift;
    }
    *T_out = prefix;
    *keep_out = kr;
}

__global__ void __launch_bounds__(kTlThreads, 1) topk_long_kernel(const float* __restrict__ scores, int tokens,
                                                                  int64_t ld, int k, int slice,
                                                                  int32_t* __restrict__ sel) {
    cg::cluster_group cluster = cg::this_cluster();
    const int nct = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s0 = min(rank * slice, tokens), s1 = min(s0 + slice, tokens);
    const float* srow = scores + (int64_t)row * ld;
    int32_t* out = sel + (int64_t)row * k;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    TlShared& S = *reinterpret_cast<TlShared*>(smem_raw);
    TlPublished& P = *reinterpret_cast<TlPublished*>(smem_raw + (sizeof(TlShared) + 15) / 16 * 16);

    // ---- pass 1: digit-1 histogram ----
    for (int i = tid; i < kRxBins + 4; i += kTlThreads) S.hist[i] = 0u;
    if (tid < kT2MaxCluster) S.ck[tid] = 0u;
    if (tid == 0) P.pub[0] = 0u;
    __syncthreads();
    tl_stream(srow, s0, s1, [&](uint32_t kj, int) { atomicAdd(&S.hist[kj ? kj >> 20 : kRxBins], 1u); });
    __syncthreads();
    for (int c = warp; c < 64; c += kTlThreads / 32) {
        const uint2 v = reinterpret_cast<const uint2*>(S.hist + 64 * c)[lane];
        uint32_t x = v.x + v.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S.coarse[c] = x;
    }
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
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
    const uint32_t b1 = S.res[0];
    uint32_t krem = S.res[1];

    // ---- pass 2: keys above b1, candidates in b1 ----
    uint32_t above = 0;
    tl_stream(srow, s0, s1, [&](uint32_t kj, int i) {
        const uint32_t d = kj >> 20;
        above += (kj != 0u && d > b1 && b1 != ~0u);
        const bool c = kj != 0u && d == b1;
        const uint32_t m = __ballot_sync(0xffffffffu, c);
        if (m) {
            uint32_t slot0 = 0;
            if (lane == __ffs(m) - 1) slot0 = atomicAdd(&P.pub[0], (uint32_t)__popc(m));
            slot0 = __shfl_sync(0xffffffffu, slot0, __ffs(m) - 1);
            const uint32_t slot = slot0 + __popc(m & t2_lanemask_lt());
            if (c && slot < kTlCtaCand) {
                P.ckey[slot] = kj;
                P.cidx[slot] = i;
            }
        }
    });
    above = __reduce_add_sync(0xffffffffu, above);
    if (lane == 0) S.wsum[warp] = above;
    __syncthreads();
    if (tid == 0) {
        uint32_t a = 0;
        for (int w = 0; w < kTlThreads / 32; ++w) a += S.wsum[w];
        P.pub[1] = a;
    }
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    if (tid < nct) {
        const uint32_t* pp = cluster.map_shared_rank(P.pub, tid);
        S.cn[tid] = pp[0];
        S.ca[tid] = pp[1];
    }
    __syncthreads();
    uint32_t n = 0;
    bool over = b1 == ~0u;
    for (int r = 0; r < nct; ++r) {
        over |= S.cn[r] > kTlCtaCand;
        n += S.cn[r];
    }
    over |= n > kTlCand;  // cluster-uniform
    if (over) {
        uint32_t T = 0, keep = 0;
        tl_radix(cluster, srow, s0, s1, k, S, &T, &keep);
        // per-CTA (> T, == T) counts -> offsets; then the tie-ranked emit
        uint32_t gt = 0, eq = 0;
        tl_stream(srow, s0, s1, [&](uint32_t kj, int) {
            gt += kj != 0u && kj > T;
            eq += kj != 0u && kj == T;
        });
        gt = __reduce_add_sync(0xffffffffu, gt);
        eq = __reduce_add_sync(0xffffffffu, eq);
        if (lane == 0) {
            S.wsum[warp] = gt;
            S.wsuf[warp] = eq;
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t a = 0, e = 0;
            for (int w = 0; w < kTlThreads / 32; ++w) {
                a += S.wsum[w];
                e += S.wsuf[w];
            }
            P.pub[1] = a;
            P.pub[2] = e;
        }
        cluster.sync();
        if (tid < nct) {
            const uint32_t* pp = cluster.map_shared_rank(P.pub, tid);
            S.ca[tid] = pp[1];
            S.ce[tid] = pp[2];
        }
        __syncthreads();
        uint32_t gb = 0, eb = 0;
        for (int r = 0; r < rank; ++r) {
            gb += S.ca[r];
            eb += S.ce[r];
        }
        // kept before this CTA: every key > T, and the first `keep` T-valued keys
        tl_emit<true>(srow, s0, s1, T, gb + min(eb, keep), eb, S, out,
                      [T, keep](uint32_t kk, int, uint32_t er) { return kk > T || (kk == T && er < keep); });
        cluster.sync();  // peers' pub reads are done
        return;
    }
    // ---- all candidates (identical list everywhere), refinement, exact threshold ----
    {
        uint32_t base = 0;
        for (int r = 0; r < nct; ++r) {
            const uint32_t* rk = cluster.map_shared_rank(P.ckey, r);
            const int32_t* ri = cluster.map_shared_rank(P.cidx, r);
            for (uint32_t i = tid; i < S.cn[r]; i += kTlThreads) {
                S.mkey[0][base + i] = rk[i];
                S.midx[0][base + i] = ri[i];
            }
            base += S.cn[r];
        }
    }
    __syncthreads();
    const uint32_t* ck = S.mkey[0];
    const int32_t* ci = S.midx[0];
    int buf = 1;
#pragma unroll 1
    for (int lvl = 0; lvl < 3 && n > 32u; ++lvl) {  // key bits 19..12, 11..4, 3..0
        const int sh = lvl == 0 ? 12 : (lvl == 1 ? 4 : 0);
        const uint32_t msk = lvl == 2 ? 0xFu : 0xFFu;
        n = rx_refine<kTlThreads, 256>(S, ck, ci, n, S.mkey[buf], S.midx[buf], krem,
                                       [sh, msk](uint32_t kk, int32_t) { return (kk >> sh) & msk; });
        ck = S.mkey[buf];
        ci = S.midx[buf];
        buf ^= 1;
    }
    if (n > 32u) {  // > 32 keys equal to T: keep the krem lowest indices
        const uint32_t Tk = ck[0];
#pragma unroll 1
        for (int lvl = 0; lvl < 4 && n > 1u; ++lvl) {
            const int sh = 24 - 8 * lvl;
            n = rx_refine<kTlThreads, 256>(S, ck, ci, n, S.mkey[buf], S.midx[buf], krem,
                                           [sh](uint32_t, int32_t ii) { return (~(uint32_t)ii >> sh) & 0xFFu; });
            ck = S.mkey[buf];
            ci = S.midx[buf];
            buf ^= 1;
        }
        if (tid == 0) {
            S.res[4] = Tk;
            S.res[5] = (uint32_t)ci[0];
        }
        __syncthreads();
    } else {
        rx_rank32(S, ck, ci, n, krem);
    }
    const uint32_t T = S.res[4];
    const int32_t idxT = (int32_t)S.res[5];
    // kept candidates of every CTA, from the published lists
    for (int r = 0; r < nct; ++r) {
        const uint32_t* rk = cluster.map_shared_rank(P.ckey, r);
        const int32_t* ri = cluster.map_shared_rank(P.cidx, r);
        uint32_t c = 0;
        for (uint32_t i = tid; i < S.cn[r]; i += kTlThreads) c += rk[i] > T || (rk[i] == T && ri[i] <= idxT);
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0 && c) atomicAdd(&S.ck[r], c);
    }
    // peers may still read this CTA's list: arrive now, wait before exiting
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
    __syncthreads();
    uint32_t base = 0;
    for (int r = 0; r < rank; ++r) base += S.ca[r] + S.ck[r];
    // ---- pass 3: ordered emit ----
    tl_emit<false>(srow, s0, s1, T, base, 0u, S, out,
                   [T, idxT](uint32_t kk, int idx, uint32_t) { return kk > T || (kk == T && idx <= idxT); });
    asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
}

static size_t topk_long_smem() {
    return (sizeof(TlShared) + 15) / 16 * 16 + sizeof(TlPublished);
}

// Rows longer than the register / shared-memory select paths.  Returns -1 if not applicable
// (unaligned scores: the float4 streaming needs 16-byte rows).
int topk_long_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st) {
    if (rows > 65535 || (ld & 3) || (reinterpret_cast<uintptr_t>(scores) & 15)) return -1;
    const int cluster = kTlCluster;
    const int slice = (int)(ceil_div(ceil_div(tokens, cluster), kTlTile) * kTlTile);
    static const bool attr = [] {
        cudaFuncSetAttribute(topk_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)topk_long_smem());
        cudaFuncSetAttribute(topk_long_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(kTlThreads, 1, 1);
    cfg.dynamicSmemBytes = topk_long_smem();
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cluster;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, topk_long_kernel, scores, tokens, ld, k, slice, sel);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    return FIER_OK;
}

}  // namespace fier_cuda
