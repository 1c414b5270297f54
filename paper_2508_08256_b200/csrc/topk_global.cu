// topk_global.cu -- K3 for many keys per launch (C3, C4, C5): a radix select whose
// per-row state lives in global memory, so the grid is as wide as the data instead of
// one thread-block cluster per row.
//
// Replaces topk_oracle (reference core.hpp:134-148): the k largest scores, ties to the
// LOWER index, ascending output.  Same keys as every K3 path (common.cuh score_key:
// order-preserving u32, NaN ranks lowest) and the same digit 1 as select_radix.cuh (the
// top 12 bits of the key).  Four launches:
//   memset    the per-row histograms and counters
//   K3g-1     CTA (slice, row) streams 8192 scores -> shared-memory digit-1 histogram ->
//             global per-row histogram (atomics on the non-empty bins only); the last
//             CTA of a row (a done counter) finds bin b1 of the k-th largest and its rank
//             krem inside the bin
//   K3g-2     the same CTAs stream their slices again (in reverse order: the tail of the
//             previous pass is still in L2): keys above b1 -> the row's "above" list
//             (< k of them), keys in b1 -> the row's candidate list
//   K3g-3     one CTA per row: the candidates (L2-resident) refined by 8-bit digits of
//             the key, then of the index for big tie groups -> (T, idx_T); the kept set =
//             above + candidates (key > T or key == T and index <= idx_T), placed in
//             ascending order through a shared-memory bitmap of the row's indices
//             (popcount prefix sums, 2^18 indices per window), written to sel.
// Two reads of the scores instead of three for topk_long.cu, and a grid of
// rows x tokens / 8192 CTAs.  A row whose candidate bin overflows the buffers (very
// narrow or tied score ranges) is finished by K3g-3 with an exact streaming MSD radix
// select of its own (9/9/9/5-bit digits, index-ordered tie ranking).
#include <climits>
#include <string>

#include "select_radix.cuh"

namespace fier_cuda {

constexpr int kTgSlice = 8192;     // keys per chunk of the streaming passes (8 float4 per thread)
constexpr int kTgChunks = 4;       // chunks per CTA of K3g-1 (fewer global histogram atomics)
constexpr int kTgChunksC = 1;      // chunks per CTA of K3g-2 (more CTAs in flight: C5 collect 96 -> 82 us)
constexpr int kTgThreads = 256;    // streaming passes: 32 keys per thread, all loads in flight
constexpr int kTgRowThreads = 512; // K3g-3
constexpr int kTgBins = kRxBins;   // digit 1 (4096 bins)
constexpr int kTgWin = 1 << 18;    // index window of K3g-3's ordering bitmap (32 KB)
constexpr int kTgRefine = 2048;    // candidates surviving the first refinement level

struct TgRow {  // per-row state (zeroed with the histograms)
    uint32_t done, b1, krem, nabove, ncand, pad[3];
};

struct TgLayout {
    size_t hist, state, above, ckey, cidx, total;
    int cap;
};

static TgLayout tg_layout(int rows, int tokens, int k) {
    TgLayout L;
    L.cap = (int)std::min<int64_t>(tokens, std::max<int64_t>(std::max(4096, 2 * k), tokens / 64));
    size_t o = 0;
    auto take = [&](size_t b) {
        const size_t at = o;
        o += (b + 255) / 256 * 256;
        return at;
    };
    L.hist = take((size_t)rows * kTgBins * 4);
    L.state = take((size_t)rows * sizeof(TgRow));
    L.above = take((size_t)rows * k * 4);
    L.ckey = take((size_t)rows * L.cap * 4);
    L.cidx = take((size_t)rows * L.cap * 4);
    L.total = o;
    return L;
}

// 32 consecutive-in-tile keys of this thread's slice part: 8 float4 per thread, all loads
// issued before any key is formed.  f(key, index) for every position < s1.
// The slice's loads: a full slice (every CTA but a row's last) without bounds checks -- a
// per-float4 select made the compiler issue the guarded scalar loads next to every
// vector load.
template <int U>
__device__ __forceinline__ void tg_load(const float* srow, int s0, int s1, float4 (&v)[U]) {
    constexpr int TILE = 4 * kTgThreads;
    if (s0 + U * TILE <= s1) {
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_stream_f4(srow + s0 + u * TILE + 4 * threadIdx.x);
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = s0 + u * TILE + 4 * threadIdx.x;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i < s1) x.x = srow[i];
            if (i + 1 < s1) x.y = srow[i + 1];
            if (i + 2 < s1) x.z = srow[i + 2];
            if (i + 3 < s1) x.w = srow[i + 3];
            v[u] = x;
        }
    }
}

template <typename F>
__device__ __forceinline__ void tg_slice(const float* srow, int s0, int s1, F&& f) {
    constexpr int TILE = 4 * kTgThreads;
    float4 v[kTgSlice / TILE];
    tg_load(srow, s0, s1, v);
#pragma unroll
    for (int u = 0; u < kTgSlice / TILE; ++u) {
        const int i = s0 + u * TILE + 4 * threadIdx.x;
        const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j < s1) f(score_key(e[j]), i + j);
    }
}

struct TgFindShared {
    uint32_t tot[kTgBins];
    uint32_t wsum[32], wsuf[32], res[8];
    uint32_t last;
};

__global__ void __launch_bounds__(kTgThreads, 4) tg_hist_kernel(const float* __restrict__ scores, int tokens,
                                                              int64_t ld, int k, uint32_t* __restrict__ hist,
                                                              TgRow* __restrict__ state) {
    __shared__ uint32_t h[kTgBins];
    __shared__ TgFindShared F;
    const int row = blockIdx.y, tid = threadIdx.x;
    for (int i = tid; i < kTgBins; i += kTgThreads) h[i] = 0u;
    __syncthreads();
    const float* srow = scores + (int64_t)row * ld;
    for (int c = 0; c < kTgChunks; ++c) {
        const int s0 = (blockIdx.x * kTgChunks + c) * kTgSlice, s1 = min(s0 + kTgSlice, tokens);
        if (s0 >= s1) break;
        tg_slice(srow, s0, s1, [&](uint32_t kj, int) { atomicAdd(&h[kj >> 20], 1u); });
    }
    __syncthreads();
    uint32_t* gh = hist + (size_t)row * kTgBins;
    for (int i = tid; i < kTgBins; i += kTgThreads)
        if (h[i]) atomicAdd(&gh[i], h[i]);
    __syncthreads();  // every bin of this CTA is in; one fence orders them before the ticket
    if (tid == 0) {
        __threadfence();
        F.last = atomicAdd(&state[row].done, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (!F.last) return;
    // the last CTA of the row: bin b1 of the k-th largest and its rank inside the bin
    __threadfence();
    {  // 16 KB of L2: every load in flight before the first store
        constexpr int V4 = kTgBins / 4 / kTgThreads;
        uint4 x[V4];
#pragma unroll
        for (int j = 0; j < V4; ++j) x[j] = __ldcg(reinterpret_cast<const uint4*>(gh) + tid + j * kTgThreads);
#pragma unroll
        for (int j = 0; j < V4; ++j) reinterpret_cast<uint4*>(F.tot)[tid + j * kTgThreads] = x[j];
    }
    __syncthreads();
    t2_find_bin<kTgThreads, kTgBins>(F.tot, (uint32_t)k, F);
    if (tid == 0) {
        state[row].b1 = F.res[0];
        state[row].krem = (uint32_t)k - F.res[1];
    }
}

__global__ void __launch_bounds__(kTgThreads, 4) tg_collect_kernel(const float* __restrict__ scores, int tokens,
                                                                 int64_t ld, int k, int cap, TgRow* __restrict__ state,
                                                                 int32_t* __restrict__ above,
                                                                 uint32_t* __restrict__ ckey,
                                                                 int32_t* __restrict__ cidx) {
    constexpr int TILE = 4 * kTgThreads, U = kTgSlice / TILE, NW = kTgThreads / 32;
    __shared__ uint32_t wa[NW], wc[NW], base[2];
    const int row = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int cc = kTgChunksC - 1; cc >= 0; --cc) {  // reverse order: the last pass's tail is in L2
        const int slice = (gridDim.x - 1 - blockIdx.x) * kTgChunksC + cc;
        const int s0 = slice * kTgSlice, s1 = min(s0 + kTgSlice, tokens);
        if (s0 >= s1) continue;  // block-uniform
        TgRow& st = state[row];
        const uint32_t b1 = __ldcg(&st.b1);
        const float* srow = scores + (int64_t)row * ld;
        // the slice's 32 keys per thread stay in registers: count first, one global atomic per
        // list and CTA reserves the output ranges, then write
        float4 v[U];
        tg_load(srow, s0, s1, v);
        uint32_t fa = 0, fc = 0;  // bit 4u + j: key j of tile u is above b1 / a candidate
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = s0 + u * TILE + 4 * tid;
            const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t d = score_key(e[j]) >> 20;
                const bool ok = i + j < s1;
                fa |= (uint32_t)(ok && d > b1) << (4 * u + j);
                fc |= (uint32_t)(ok && d == b1) << (4 * u + j);
            }
        }
        // per-warp counts, one CTA reservation per list, then each lane writes its own flagged
        // keys (few: a loop over set bits; the candidates' keys are re-read from L2) at its
        // warp-exclusive offset -- a 32-step ballot loop per chunk cost ~10 instructions per key
        uint32_t pa = __popc(fa), pc = __popc(fc);  // -> inclusive prefix over lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, pa, o), yc = __shfl_up_sync(0xffffffffu, pc, o);
            if (lane >= o) {
                pa += ya;
                pc += yc;
            }
        }
        if (lane == 31) {
            wa[warp] = pa;
            wc[warp] = pc;
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t ta = 0, tc = 0;
            for (int w = 0; w < NW; ++w) {
                const uint32_t x = wa[w], y = wc[w];
                wa[w] = ta;
                wc[w] = tc;
                ta += x;
                tc += y;
            }
            base[0] = ta ? atomicAdd(&st.nabove, ta) : 0u;
            base[1] = tc ? atomicAdd(&st.ncand, tc) : 0u;
        }
        __syncthreads();
        uint32_t oa = base[0] + wa[warp] + pa - __popc(fa), oc = base[1] + wc[warp] + pc - __popc(fc);
        int32_t* ab = above + (size_t)row * k;
        uint32_t* ck = ckey + (size_t)row * cap;
        int32_t* ci = cidx + (size_t)row * cap;
        auto index_of = [&](int b) { return s0 + (b >> 2) * TILE + 4 * tid + (b & 3); };
        for (uint32_t m = fa; m; m &= m - 1) ab[oa++] = index_of(__ffs(m) - 1);  // < k by the choice of b1
        for (uint32_t m = fc; m; m &= m - 1, ++oc) {
            if (oc < (uint32_t)cap) {
                const int ix = index_of(__ffs(m) - 1);
                ck[oc] = score_key(__ldg(srow + ix));
                ci[oc] = ix;
            }
        }
        __syncthreads();  // wa / wc / base are reused by the next chunk
    }
}

struct TgRowShared {
    uint32_t tot[kT2Bins];
    uint32_t wsum[32], wsuf[32], res[8];
    uint32_t nkept;
    uint32_t rk[2][kTgRefine];
    int32_t ri[2][kTgRefine];
    uint32_t bm[kTgWin / 32];  // bitmap of kept indices, one window
};

// Survivors of src[0..n) whose digit equals the bin of the krem-th largest (BINS = 256),
// written to dst (at most cap; the count is returned either way).
template <int NT, typename SH, typename Digit>
__device__ __forceinline__ uint32_t tg_refine(SH& S, const uint32_t* sk, const int32_t* si, uint32_t n,
                                              uint32_t* dk, int32_t* di, uint32_t cap, uint32_t& krem,
                                              Digit&& digit) {
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 256; i += NT) S.tot[i] = 0u;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += NT) atomicAdd(&S.tot[digit(sk[i], si[i])], 1u);
    __syncthreads();
    t2_find_bin<NT, 256>(S.tot, krem, S);
    const uint32_t b = S.res[0];
    krem -= S.res[1];
    __syncthreads();
    if (tid == 0) S.res[2] = 0;
    __syncthreads();
    for (uint32_t i0 = 0; i0 < n; i0 += NT) {
        const uint32_t i = i0 + tid;
        const bool c = i < n && digit(sk[i], si[i]) == b;
        const uint32_t m = __ballot_sync(0xffffffffu, c);
        if (m) {
            uint32_t base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&S.res[2], (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            const uint32_t slot = base + __popc(m & t2_lanemask_lt());
            if (c && slot < cap) {
                dk[slot] = sk[i];
                di[slot] = si[i];
            }
        }
    }
    __syncthreads();
    return S.res[2];
}

// Block-wide exclusive scan of one count per thread (NT threads); *tot = the sum.
template <int NT, typename SH>
__device__ __forceinline__ uint32_t tg_scan(uint32_t v, SH& S, uint32_t* tot) {
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
        const uint32_t w = lane < NT / 32 ? S.wsum[lane] : 0u;
        uint32_t z = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < NT / 32) S.wsuf[lane] = z - w;
        if (lane == 31) S.res[7] = z;
    }
    __syncthreads();
    *tot = S.res[7];
    const uint32_t r = S.wsuf[warp] + x - v;
    __syncthreads();
    return r;
}

// The exact path for a row whose candidates overflowed: MSD radix select on the key
// (9/9/9/5-bit digits) streaming the row, then an index-ordered emit (keys > T, and the
// first `keep` T-valued keys).
template <int NT, typename SH>
__device__ __noinline__ void tg_row_exact(const float* srow, int tokens, int k, int32_t* out, SH& S) {
    const int tid = threadIdx.x;
    uint32_t prefix = 0, pmask = 0, kr = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = pass < 3 ? 23 - 9 * pass : 0;
        const int bins = pass == 3 ? 32 : 512;
        for (int i = tid; i < 512; i += NT) S.tot[i] = 0u;
        __syncthreads();
        for (int i = tid; i < tokens; i += NT) {
            const uint32_t kj = score_key(srow[i]);
            if ((kj & pmask) == prefix) atomicAdd(&S.tot[(kj >> shift) & (bins - 1)], 1u);
        }
        __syncthreads();
        t2_find_bin<NT, 512>(S.tot, kr, S);
        kr -= S.res[1];
        prefix |= S.res[0] << shift;
        pmask |= (uint32_t)(bins - 1) << shift;
        __syncthreads();
    }
    const uint32_t T = prefix, keep = kr;
    uint32_t run = 0, eq_run = 0;
    for (int t0 = 0; t0 < tokens; t0 += NT) {
        const int i = t0 + tid;
        const uint32_t kj = i < tokens ? score_key(srow[i]) : 0u;
        const bool eq = i < tokens && kj == T;
        uint32_t te = 0, tk = 0;
        const uint32_t er = eq_run + tg_scan<NT>(eq ? 1u : 0u, S, &te);
        const bool kept = i < tokens && (kj > T || (eq && er < keep));
        const uint32_t pos = run + tg_scan<NT>(kept ? 1u : 0u, S, &tk);
        if (kept) out[pos] = i;
        run += tk;
        eq_run += te;
    }
}

__global__ void __launch_bounds__(kTgRowThreads) tg_row_kernel(const float* __restrict__ scores, int tokens,
                                                                int64_t ld, int k, int cap,
                                                                const TgRow* __restrict__ state,
                                                                const int32_t* __restrict__ above,
                                                                const uint32_t* __restrict__ ckey,
                                                                const int32_t* __restrict__ cidx,
                                                                int32_t* __restrict__ sel) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    TgRowShared& S = *reinterpret_cast<TgRowShared*>(smem_raw);
    constexpr int NT = kTgRowThreads;
    const int row = blockIdx.y, tid = threadIdx.x;  // blockIdx.x: this CTA's index window
    const TgRow st = state[row];
    int32_t* out = sel + (int64_t)row * k;
    const uint32_t nab = st.nabove, nc = st.ncand;
    if (st.b1 == ~0u || nc > (uint32_t)cap || nab + nc < (uint32_t)k) {  // no bin / overflow
        tg_row_exact<NT>(scores + (int64_t)row * ld, tokens, k, out, S);
        return;
    }
    const uint32_t* gk = ckey + (size_t)row * cap;
    const int32_t* gi = cidx + (size_t)row * cap;
    // ---- (T, idx_T): the krem-th largest candidate by (key desc, index asc) ----
    uint32_t krem = st.krem, n = nc;
    const uint32_t* ck = gk;
    const int32_t* ci = gi;
    int buf = 0;
    bool overflow = false;
#pragma unroll 1
    for (int lvl = 0; lvl < 3 && n > 32u; ++lvl) {  // key bits 19..12, 11..4, 3..0
        const int sh = lvl == 0 ? 12 : (lvl == 1 ? 4 : 0);
        const uint32_t msk = lvl == 2 ? 0xFu : 0xFFu;
        n = tg_refine<NT>(S, ck, ci, n, S.rk[buf], S.ri[buf], kTgRefine, krem,
                      [sh, msk](uint32_t kk, int32_t) { return (kk >> sh) & msk; });
        if (n > (uint32_t)kTgRefine) {
            overflow = true;
            break;
        }
        ck = S.rk[buf];
        ci = S.ri[buf];
        buf ^= 1;
    }
    if (!overflow && n > 32u) {  // > 32 keys equal to T: the krem lowest indices (digits of ~idx)
#pragma unroll 1
        for (int lvl = 0; lvl < 4 && n > 1u; ++lvl) {
            const int sh = 24 - 8 * lvl;
            n = tg_refine<NT>(S, ck, ci, n, S.rk[buf], S.ri[buf], kTgRefine, krem,
                          [sh](uint32_t, int32_t ii) { return (~(uint32_t)ii >> sh) & 0xFFu; });
            ck = S.rk[buf];
            ci = S.ri[buf];
            buf ^= 1;
        }
        if (tid == 0) {
            S.res[4] = ck[0];
            S.res[5] = (uint32_t)ci[0];
        }
        __syncthreads();
    } else if (!overflow) {
        rx_rank32<CtaBar>(S, ck, ci, n, krem);
    }
    if (overflow) {  // block-uniform
        tg_row_exact<NT>(scores + (int64_t)row * ld, tokens, k, out, S);
        return;
    }
    const uint32_t T = S.res[4];
    const int32_t idxT = (int32_t)S.res[5];
    // ---- ascending output: the kept indices (the above list and the kept candidates) in
    // this CTA's window of kTgWin indices set bits of a bitmap; the kept indices below the
    // window give its first output slot; popcount prefix sums place the rest.  One CTA per
    // window (every CTA of a row redoes the small threshold search above). ----
    const int32_t* ab = above + (size_t)row * k;
    constexpr int WPT = kTgWin / 32 / NT;  // bitmap words per thread of a full window
    const int wpt = min(WPT, ((tokens + 31) / 32 + NT - 1) / NT);  // short rows: a smaller window
    const int win = 32 * NT * wpt;
    const int w0 = blockIdx.x * win;
    if (w0 >= tokens) return;  // block-uniform
    for (int i = tid; i < win / 32; i += NT) S.bm[i] = 0u;
    __syncthreads();
    uint32_t below = 0;
    for (uint32_t i = tid; i < nab; i += NT) {
        const int32_t x = ab[i] - w0;
        below += x < 0;
        if (x >= 0 && x < win) atomicOr(&S.bm[x >> 5], 1u << (x & 31));
    }
    for (uint32_t i = tid; i < nc; i += NT) {
        const uint32_t kk = gk[i];
        const int32_t ix = gi[i], x = ix - w0;
        const bool kept = kk > T || (kk == T && ix <= idxT);
        below += kept && x < 0;
        if (kept && x >= 0 && x < win) atomicOr(&S.bm[x >> 5], 1u << (x & 31));
    }
    uint32_t run = 0;
    tg_scan<NT>(below, S, &run);  // (the scan's total = the kept indices below the window)
    uint32_t wv[WPT], c = 0;
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
        wv[j] = j < wpt ? S.bm[tid * wpt + j] : 0u;
        c += __popc(wv[j]);
    }
    uint32_t tot = 0;
    uint32_t o = run + tg_scan<NT>(c, S, &tot);
#pragma unroll
    for (int j = 0; j < WPT; ++j)
        for (uint32_t m = wv[j]; m; m &= m - 1) out[o++] = w0 + 32 * (tid * wpt + j) + __ffs(m) - 1;
}

// ---- K3r: one CTA per row, for launches of many short rows (C4: 1024 rows x 32768) ----
// The whole select of a row in one small CTA (256 threads, ~42 KB of shared memory), so
// every row of a C4 launch is in flight at once instead of one cluster wave after another:
//   pass 1  digit-1 histogram of the row (8 float4 loads in flight per thread) -> b1, krem
//   pass 2  the row again (recently read: mostly L2): keys above b1 set bits of an index
//           bitmap of the row, keys in b1 go to a shared-memory candidate list
//   then    candidates refined to (T, idx_T) (tg_refine), the kept ones set their bits,
//           and popcount prefix sums of the bitmap write the ascending selection.
// (Measured at C4: 122 us against 153 us for the 2-CTA cluster select; a sampled-threshold
// variant -- 2048 sampled keys bound the collection, no full histogram -- needed 75 KB of
// shared memory for the collected keys and ran 150 us.)
constexpr int kTrThreads = 256;
#ifndef FIER_TR_CAND
#define FIER_TR_CAND 1024
#endif
constexpr int kTrCand = FIER_TR_CAND;      // candidates of a row (digit 1 == b1); more: exact fallback
constexpr int kTrRefine = kTrCand / 2;     // survivors of the first refinement level
constexpr int kTrMaxTokens = 32768;        // bitmap of the row's indices (4 KB)
// Six CTAs per SM (30 KB of shared memory, <= 40 registers): 888 rows in flight, and the
// smaller carveout leaves L1 for the second pass's re-reads.  C4 K3 by footprint: 42 KB / 48
// registers (5 per SM) 88.9 us; 34 KB (1536 candidates), 6 per SM 87.9 us; 30 KB (1024), 6 per
// SM 82.2 us; 7 per SM (36 registers, 184 B of spill) 99 us; no register cap (84 registers,
// 3 per SM) 111 us.  A row with more candidates in its digit-1 bin takes the exact fallback.
constexpr int kTrMinBlocks = 6;

struct TrShared {
    union {
        uint32_t hist[kTgBins];  // pass 1
        struct {
            uint32_t rk[2][kTrRefine];
            int32_t ri[2][kTrRefine];
        } r;                     // refinement, after the histogram is dead
    } u;
    uint32_t ck[kTrCand];
    int32_t ci[kTrCand];
    uint32_t bm[kTrMaxTokens / 32];
    uint32_t tot[kT2Bins];
    uint32_t wsum[32], wsuf[32], res[8];
    uint32_t ncand;
};

__global__ void __launch_bounds__(kTrThreads, kTrMinBlocks) tr_row_kernel(const float* __restrict__ scores, int tokens, int64_t ld,
                                                             int k, int32_t* __restrict__ sel) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    TrShared& S = *reinterpret_cast<TrShared*>(smem_raw);
    constexpr int NT = kTrThreads, CH = kTgSlice;  // keys per chunk (8 float4 per thread)
    const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const float* srow = scores + (int64_t)row * ld;
    int32_t* out = sel + (int64_t)row * k;
    const int words = (tokens + 31) / 32;
    for (int i = tid; i < kTgBins; i += NT) S.u.hist[i] = 0u;
    for (int i = tid; i < words; i += NT) S.bm[i] = 0u;
    if (tid == 0) S.ncand = 0u;
    __syncthreads();
    for (int c0 = 0; c0 < tokens; c0 += CH) {
        float4 v[CH / (4 * NT)];
        tg_load(srow, c0, min(c0 + CH, tokens), v);
#pragma unroll
        for (int u = 0; u < CH / (4 * NT); ++u) {
            const int i = c0 + u * 4 * NT + 4 * tid;
            const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (i + j < tokens) atomicAdd(&S.u.hist[score_key(e[j]) >> 20], 1u);
        }
    }
    __syncthreads();
    t2_find_bin<NT, kTgBins>(S.u.hist, (uint32_t)k, S);
    const uint32_t b1 = S.res[0];
    uint32_t krem = (uint32_t)k - S.res[1];
    __syncthreads();
    if (b1 == ~0u) {
        tg_row_exact<NT>(srow, tokens, k, out, S);
        return;
    }
    for (int c0 = 0; c0 < tokens; c0 += CH) {
        constexpr int U = CH / (4 * NT);
        float4 v[U];
        tg_load(srow, c0, min(c0 + CH, tokens), v);
        uint32_t fa = 0, fc = 0;  // bit 4u + j: key j of float4 u is above b1 / a candidate
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = c0 + u * 4 * NT + 4 * tid;
            const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t d = score_key(e[j]) >> 20;
                const bool ok = i + j < tokens;
                fa |= (uint32_t)(ok && d > b1) << (4 * u + j);
                fc |= (uint32_t)(ok && d == b1) << (4 * u + j);
            }
        }
        // above b1: a float4's 4 tokens share one bitmap word -- one atomic per nibble
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t nib = (fa >> (4 * u)) & 0xFu;
            const int i = c0 + u * 4 * NT + 4 * tid;
            if (nib) atomicOr(&S.bm[i >> 5], nib << (i & 31));
        }
        // candidates: each lane writes its own (few) at a warp-exclusive offset; keys re-read (L2)
        uint32_t pc = __popc(fc);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, pc, o);
            if (lane >= o) pc += y;
        }
        uint32_t base = 0;
        if (lane == 31 && pc) base = atomicAdd(&S.ncand, pc);
        base = __shfl_sync(0xffffffffu, base, 31);
        uint32_t slot = base + pc - __popc(fc);
        for (uint32_t m = fc; m; m &= m - 1, ++slot) {
            const int b = __ffs(m) - 1;
            const int ix = c0 + (b >> 2) * 4 * NT + 4 * tid + (b & 3);
            if (slot < (uint32_t)kTrCand) {
                S.ck[slot] = score_key(__ldg(srow + ix));
                S.ci[slot] = ix;
            }
        }
    }
    __syncthreads();
    uint32_t n = S.ncand;
    const uint32_t nc = n;
    if (n > (uint32_t)kTrCand) {
        tg_row_exact<NT>(srow, tokens, k, out, S);
        return;
    }
    // ---- (T, idx_T) among the candidates ----
    const uint32_t* ck = S.ck;
    const int32_t* ci = S.ci;
    int buf = 0;
    bool overflow = false;
#pragma unroll 1
    for (int lvl = 0; lvl < 3 && n > 32u; ++lvl) {  // key bits 19..12, 11..4, 3..0
        const int sh = lvl == 0 ? 12 : (lvl == 1 ? 4 : 0);
        const uint32_t msk = lvl == 2 ? 0xFu : 0xFFu;
        n = tg_refine<NT>(S, ck, ci, n, S.u.r.rk[buf], S.u.r.ri[buf], kTrRefine, krem,
                          [sh, msk](uint32_t kk, int32_t) { return (kk >> sh) & msk; });
        if (n > (uint32_t)kTrRefine) {
            overflow = true;
            break;
        }
        ck = S.u.r.rk[buf];
        ci = S.u.r.ri[buf];
        buf ^= 1;
    }
    if (!overflow && n > 32u) {  // > 32 keys equal to T: the krem lowest indices
#pragma unroll 1
        for (int lvl = 0; lvl < 4 && n > 1u; ++lvl) {
            const int sh = 24 - 8 * lvl;
            n = tg_refine<NT>(S, ck, ci, n, S.u.r.rk[buf], S.u.r.ri[buf], kTrRefine, krem,
                              [sh](uint32_t, int32_t ii) { return (~(uint32_t)ii >> sh) & 0xFFu; });
            ck = S.u.r.rk[buf];
            ci = S.u.r.ri[buf];
            buf ^= 1;
        }
        if (tid == 0) {
            S.res[4] = ck[0];
            S.res[5] = (uint32_t)ci[0];
        }
        __syncthreads();
    } else if (!overflow) {
        rx_rank32<CtaBar>(S, ck, ci, n, krem);
    }
    if (overflow) {  // block-uniform
        tg_row_exact<NT>(srow, tokens, k, out, S);
        return;
    }
    const uint32_t T = S.res[4];
    const int32_t idxT = (int32_t)S.res[5];
    for (uint32_t i = tid; i < nc; i += NT) {
        const uint32_t kk = S.ck[i];
        const int32_t ix = S.ci[i];
        if (kk > T || (kk == T && ix <= idxT)) atomicOr(&S.bm[ix >> 5], 1u << (ix & 31));
    }
    __syncthreads();
    // ---- ascending output from the bitmap ----
    constexpr int WPT = kTrMaxTokens / 32 / NT;
    const int wpt = (words + NT - 1) / NT;
    uint32_t wv[WPT], c = 0;
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
        const int w = tid * wpt + j;
        wv[j] = (j < wpt && w < words) ? S.bm[w] : 0u;
        c += __popc(wv[j]);
    }
    uint32_t tot = 0;
    uint32_t o = tg_scan<NT>(c, S, &tot);
    if (tot <= (uint32_t)kTgBins) {
        // staged in the dead histogram / refinement union, then written out coalesced (each
        // thread's run of ~k/256 scattered stores was 13% of the kernel's warp samples)
        int32_t* stage = reinterpret_cast<int32_t*>(S.u.hist);
#pragma unroll
        for (int j = 0; j < WPT; ++j)
            for (uint32_t m = wv[j]; m; m &= m - 1) stage[o++] = 32 * (tid * wpt + j) + __ffs(m) - 1;
        __syncthreads();
        for (uint32_t i = tid; i < tot; i += NT) out[i] = stage[i];
    } else {
#pragma unroll
        for (int j = 0; j < WPT; ++j)
            for (uint32_t m = wv[j]; m; m &= m - 1) out[o++] = 32 * (tid * wpt + j) + __ffs(m) - 1;
    }
}

bool topk_rows_applies(int rows, int tokens, int k) {
    (void)k;
    return rows >= 4 * num_sms() && tokens <= kTrMaxTokens && rows <= 65535 && tokens >= 1024;
}

int topk_rows_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel, cudaStream_t st) {
    if (!topk_rows_applies(rows, tokens, k) || (ld & 3) || (reinterpret_cast<uintptr_t>(scores) & 15)) return -1;
    static const bool attr = [] {
        cudaFuncSetAttribute(tr_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TrShared));
        return true;
    }();
    (void)attr;
    tr_row_kernel<<<rows, kTrThreads, sizeof(TrShared), st>>>(scores, tokens, ld, k, sel);
    return check_launch("fier_topk");
}

// ---- host side -------------------------------------------------------------------

bool topk_rows_applies(int rows, int tokens, int k);

bool topk_global_applies(int rows, int tokens, int k) {
    // a wide grid pays off once the launch holds millions of keys in few rows (C5); many
    // short rows take the CTA-per-row kernel
    // (C3's 4M keys in 32 rows: the cluster select is faster, 26.2 vs 34.7 us)
    return (int64_t)rows * tokens >= (int64_t)16 << 20 && rows <= 65535 && !topk_rows_applies(rows, tokens, k);
}

size_t topk_global_workspace(int rows, int tokens, int k) {
    if (!topk_global_applies(rows, tokens, k)) return 0;
    return tg_layout(rows, tokens, k).total;
}

int topk_global_dispatch(const float* scores, int rows, int tokens, int64_t ld, int k, int32_t* sel,
                         void* workspace, size_t workspace_bytes, cudaStream_t st) {
    if (!topk_global_applies(rows, tokens, k) || !workspace) return -1;
    const TgLayout L = tg_layout(rows, tokens, k);
    if (workspace_bytes < L.total) return -1;
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
    TgRow* state = reinterpret_cast<TgRow*>(ws + L.state);
    int32_t* above = reinterpret_cast<int32_t*>(ws + L.above);
    uint32_t* ckey = reinterpret_cast<uint32_t*>(ws + L.ckey);
    int32_t* cidx = reinterpret_cast<int32_t*>(ws + L.cidx);
    cudaError_t e = cudaMemsetAsync(ws + L.hist, 0, L.above - L.hist, st);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_topk: ") + cudaGetErrorString(e));
    const dim3 grid((unsigned)ceil_div(tokens, (int64_t)kTgSlice * kTgChunks), (unsigned)rows);
    tg_hist_kernel<<<grid, kTgThreads, 0, st>>>(scores, tokens, ld, k, hist, state);
    if (int rc = check_launch("fier_topk")) return rc;
    const dim3 gridc((unsigned)ceil_div(tokens, (int64_t)kTgSlice * kTgChunksC), (unsigned)rows);
    tg_collect_kernel<<<gridc, kTgThreads, 0, st>>>(scores, tokens, ld, k, L.cap, state, above, ckey, cidx);
    if (int rc = check_launch("fier_topk")) return rc;
    static const bool attr = [] {
        cudaFuncSetAttribute(tg_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TgRowShared));
        return true;
    }();
    (void)attr;
    const int wins = (int)ceil_div(tokens, (int64_t)kTgWin);  // CTAs per row: one per index window
    tg_row_kernel<<<dim3((unsigned)wins, (unsigned)rows), kTgRowThreads, sizeof(TgRowShared), st>>>(scores, tokens, ld, k, L.cap, state, above,
                                                                    ckey, cidx, sel);
    return check_launch("fier_topk");
}

}  // namespace fier_cuda
