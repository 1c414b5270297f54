// step_fused.cu -- the whole decode step of an MHA layer in ONE launch:
// append -> score -> Top-n -> sparse attention, one thread-block cluster per
// (sequence, head).
//
// Reference: fier_attend (retrieval.hpp:136-146) = approx_scores
// (quant1bit.hpp:121-140) -> topk_oracle (core.hpp:134-148) -> gather_attention
// (core.hpp:152-179), for every (sequence, head) of a layer, after the decode-time
// append of the new token to the packed index (quantize's short-group rule,
// quant1bit.hpp:84).  The separate-kernel path (score.cu -> topk2.cu ->
// attention_tc.cu) computes the same thing with the scores and the selection
// round-tripping through memory; here they stay on chip:
//
//   phase A  the CTA whose slice holds `pos` writes the new k/v row and re-packs
//            the open group (K1 append, pack.cuh)
//   phase B  CTA r of the cluster scores tokens [r*S, (r+1)*S) into shared-memory
//            keys (S = 256*kpt; lane = token, the layout select.cuh wants).
//            Scorer: a per-group nibble table.  For each 4-channel nibble
//            position p the 16 entries hold  sum_{i in p} q_i (z_i - s_i)
//            + sum_{i in p, bit i set} 2 q_i s_i,  so a token's score is the sum
//            of 32 table reads, one per nibble of its 128-bit row: per nibble one
//            PRMT (address), one LDS, one FADD -- ~3.5 lane-instructions per 4
//            bits instead of ~2.5 per bit (score.cu).  Tables are rebuilt per
//            32-token slab (lane p builds position p), one table per warp.
//   phase C  cluster Top-k on the shared-memory keys (select_radix.cuh: a fixed
//            12-bit radix histogram counted by the scorer, merged over DSMEM,
//            candidate refinement by further digits, exact rank; two cluster
//            barriers), then the emit pass writes the ascending selection to `sel`
//            and this CTA's own selected tokens to shared memory.
//   phase D  8 warps gather the CTA's selected K/V rows through cp.async rings
//            and run the tensor-core online softmax (attn_tc.cuh); warp partials
//            merge in shared memory, CTA partials are pushed to rank 0 over DSMEM
//            and merged there by log-sum-exp.
//
// Only one kernel boundary per step, no score or index round trip through HBM,
// and no split/merge workspace.  Every phase runs once per CTA, so the code is
// kept as compact loops (a fully unrolled version streamed ~300 KB of SASS
// through a cold instruction cache and ran 3x slower).  Applies to MHA (Hq == Hkv), d = 128, 32 | g,
// 16-bit caches, rows up to 16 * 8192 tokens; other shapes use the
// separate-kernel path.
#include <climits>
#include <cstdlib>
#include <string>

#include "common.cuh"

#ifdef FIER_STEP_TRACE
// debug build only (build.py --trace): globaltimer at the phase boundaries, per CTA
namespace fier_cuda {
constexpr int kFsTraceCtas = 4096;
constexpr int kFsTraceMarks = 24;
__device__ unsigned long long g_fs_trace[kFsTraceCtas][kFsTraceMarks];
}  // namespace fier_cuda
#define FS_MARK_T(i, thr)                                                                     \
    do {                                                                                      \
        if (threadIdx.x == (thr)) {                                                           \
            const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                             \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)::"memory");                            \
            if (cta_ < ::fier_cuda::kFsTraceCtas) ::fier_cuda::g_fs_trace[cta_][i] = t_;                                \
        }                                                                                     \
    } while (0)
#else
#define FS_MARK_T(i, thr) \
    do {                  \
    } while (0)
#endif
#define FS_MARK(i) FS_MARK_T(i, 0)
#define T2_MARK(i) FS_MARK(i)

#include "attn_tc.cuh"
#include "nibble.cuh"
#include "pack.cuh"
#include "rope.cuh"
#include "select_radix.cuh"

namespace fier_cuda {

constexpr int kFsThreads = 512;  // 16 warps: ALU/LDS latency in the scorer needs the warps
constexpr int kFsWarps = kFsThreads / 32;
constexpr int kFsD = 128;
#ifndef FIER_FS_GATHER_WARPS
#define FIER_FS_GATHER_WARPS 8
#endif
#ifndef FIER_FS_NST
#define FIER_FS_NST 2
#endif
constexpr int kFsGatherWarps = FIER_FS_GATHER_WARPS;  // phase D: the last warps attend (tensor cores, cp.async rings),
constexpr int kFsSelWarps = kFsWarps - kFsGatherWarps;  // the first resolve the candidates and write the selection
constexpr int kFsSelThreads = kFsSelWarps * 32;
constexpr int kFsNst = FIER_FS_NST;
constexpr int kFsMaxKpt = 16;  // slice <= 8192 tokens (u16 slots in sidx)
#ifndef FS_SCORE_WARPS
#define FS_SCORE_WARPS 16
#endif
constexpr int kFsScoreWarps = FS_SCORE_WARPS;  // warps that score in phase B
#ifndef FIER_FS_APPEND_SLABS
#define FIER_FS_APPEND_SLABS 2
#endif
constexpr int kFsAppendSlabs = FIER_FS_APPEND_SLABS;  // sealed slabs the append warps hand to the others (~ the append's time)
constexpr int kFsLutBytes = kNibTableBytes;
// Shared memory map (bytes from a 256-aligned base).  RxShared's tail (the digit-1
// histogram, dead after cluster barrier 2) opens the ring area; the scorer's LUTs and
// keys (dead after the partition pass) follow it inside the ring area.
constexpr int cmax(int x, int y) { return x > y ? x : y; }
constexpr int kFsRx = 0;
constexpr int kFsRing = kFsRx + (int)offsetof(RxShared, hist);                     // phase D rings
constexpr int kFsRingBytes = kFsGatherWarps * kFsNst * 2 * tc_stage_bytes<kFsD>();
constexpr int kFsLut = (kFsRx + (int)sizeof(RxShared) + 255) / 256 * 256;          // phase B (in the ring area)
constexpr int kFsKeys = kFsLut + kFsWarps * kFsLutBytes;                      // phase B/C keys (ditto)
constexpr int kFsRingArea = cmax(kFsRingBytes, kFsKeys + kFsThreads * kFsMaxKpt * 4 - kFsRing);
constexpr int kFsSidx = kFsRing + kFsRingArea;                                    // u16 gather list
constexpr int kFsMasks = kFsSidx + kFsThreads * kFsMaxKpt * 2;                    // amask, kmask
constexpr int kFsPub = kFsMasks + 2 * kFsWarps * kFsMaxKpt * 4;                   // RxPublished (read by peers)
constexpr int kFsWres = kFsPub + ((int)sizeof(RxPublished) + 15) / 16 * 16;        // warp partials
constexpr int kFsCres = kFsWres + kFsGatherWarps * (kFsD + 2) * 4;                // CTA partials (rank 0)
constexpr int kFsQrot = kFsCres + kT2MaxCluster * (kFsD + 2) * 4;                 // fp32 (rotated) query
constexpr int kFsCbar = kFsQrot + kFsD * 4;                                       // 4 cluster mbarriers + kready
constexpr int kFsSmem = kFsCbar + 5 * 8 + 256;                                    // + base alignment
static_assert(kFsRing % 256 == 0, "");
static_assert(sizeof(T2Shared) <= sizeof(RxShared), "");
static_assert(kFsSmem <= 227 * 1024, "fused step exceeds shared memory");

struct FsArgs {
    const void* q;
    void* K;
    void* V;
    const void* k_new;
    const void* v_new;
    uint32_t* bits;
    __half2* sz;
    float* scores;  // optional
    float* out;
    int32_t* sel;
    int64_t ld;
    int pos, tokens, cap, G, hq, g, g_shift, k, kpt;  // g_shift = log2(g) or -1
    float scale_log2;
    RopeTable rope;  // rd = 0: no rotary embedding
    int32_t* nonfinite;  // FIER_NONFINITE_KEY / _QUERY (may be null)
};

// The degenerate-row path, out of line: its code would otherwise sit between the hot
// phases and be streamed through the instruction cache every step.
__device__ __noinline__ void fused_fallback_select(cg::cluster_group& cluster, const SmemKeys& keys, int k,
                                                   RxShared& S, int32_t* selrow, uint16_t* sidx, int s0,
                                                   int wbase, uint32_t* cbase, uint32_t* ccount) {
    const int lane = threadIdx.x & 31;
    const T2Threshold th = t2_radix_select<kFsThreads>(cluster, keys, k, S);
    t2_compact<kFsThreads>(cluster, keys, th, S, cbase, ccount, [&](uint32_t slot, int j) {
        const int local = wbase + 32 * j + lane;
        selrow[slot] = s0 + local;
        sidx[slot - *cbase] = (uint16_t)local;
    });
}

template <typename T>
__global__ void __launch_bounds__(kFsThreads, 1) step_fused_kernel(const FsArgs a) {
    constexpr int D = kFsD;
#ifndef FIER_FS_PF
#define FIER_FS_PF 2
#endif
    // slabs in flight per warp in the register ring (A/B x3, C2 us: 1 30.99, 2 29.64, 3 30.01,
    // 4 30.24, 6 33.15 -- fewer live registers next to the L2 prefetch at kernel entry)
    constexpr int PF = FIER_FS_PF;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int nct = (int)cluster.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = blockIdx.y;  // b * hq + h; MHA: kv head = h, sequence index = row
    const int64_t seq = row;
    const int kpt = a.kpt;  // slabs (keys) per thread
    const int slice = kFsThreads * kpt;
    const int s0 = rank * slice;
    const int wbase = warp * 32 * kpt;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 255u) & ~255u;
    uint8_t* smem = smem_raw + (base - raw);
    RxShared& S = *reinterpret_cast<RxShared*>(smem + kFsRx);
    RxPublished& P = *reinterpret_cast<RxPublished*>(smem + kFsPub);
    uint16_t* sidx = reinterpret_cast<uint16_t*>(smem + kFsSidx);
    float* wres = reinterpret_cast<float*>(smem + kFsWres);
    float* cres = reinterpret_cast<float*>(smem + kFsCres);
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(smem + kFsKeys);

    // Cluster barriers of phases C and D: one mbarrier each per CTA (nct arrivals).  The
    // launch-phase cluster barrier makes every CTA's initialisation visible before the
    // first remote arrive; only warp 0 waits on it (the others never use barrier.cluster
    // again, except on the degenerate-row path).
    uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + kFsCbar);
    // The appending CTA (its slice holds pos): warps 0..3 load the open group's rows first,
    // before the scoring streams queue up in the memory system.
    const bool appender = a.pos / slice == rank;  // CTA-uniform
    const int open_lo = appender ? (a.pos / a.g) * a.g : INT_MAX;  // first token of the open group
    // Raw registers: nothing waits on these loads before phase A uses them.
    T vpre[32];             // g <= 32: the open group's rows, channel tid
    T knr{}, knp{}, vnr{};  // the new k row's channels tid and rope_partner(tid), the new v
    if (appender && tid < kFsD) {
        const T* kn = static_cast<const T*>(a.k_new) + seq * kFsD;
        knr = kn[tid];
        knp = kn[rope_partner(a.rope, tid)];
        vnr = static_cast<const T*>(a.v_new)[seq * kFsD + tid];
        if (a.g <= 32)
            open_group_preload<T>(static_cast<const T*>(a.K) + seq * a.cap * kFsD, kFsD, open_lo,
                                  min(open_lo + a.g, a.pos + 1), vpre);
    }
    uint64_t* kready = cbar + 4;  // the select warps' kept candidates are listed (kFsSelThreads arrivals)
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(cbar + i, (uint32_t)nct);
        mbar_init(kready, (uint32_t)kFsSelThreads);
        S.gclaim = 0u;
    }
    rx_clear<kFsThreads>(S);  // the scorer counts every key into the digit-1 histogram
    T* Kseq = static_cast<T*>(a.K) + seq * a.cap * D;
    T* Vseq = static_cast<T*>(a.V) + seq * a.cap * D;
    uint32_t* bseq = a.bits + seq * a.cap * 4;
    __half2* zseq = a.sz + seq * a.G * D;

    // Scoring is assigned per slab (32 tokens), independently of which warp owns the
    // slab's keys in phase C (keys are stored token-ordered: slab sl -> keys_s[32 sl ..]).
    // Sealed slabs are split into contiguous per-warp ranges; in the appending CTA the
    // four append warps take kFsAppendSlabs fewer and also score the open (and empty)
    // slabs, right after the named barrier that publishes the re-packed group.
    const int nsl = slice / 32;
    const int ntok = max(0, min(a.tokens, s0 + slice) - s0);
    const int nsealed = appender ? (open_lo - s0) / 32 : (ntok + 31) / 32;
    int start, cnt;
    {
        const int per = nsealed / kFsScoreWarps;
        const int na = appender ? max(0, per - kFsAppendSlabs) : per;  // warps 0..3
        const int rest = nsealed - 4 * na, nb = kFsScoreWarps - 4;
        if (warp >= kFsScoreWarps) {
            start = nsealed;
            cnt = 0;
        } else if (warp < 4) {
            start = warp * na;
            cnt = na;
        } else {
            const int w = warp - 4, q = rest / nb, r = rest % nb;
            start = 4 * na + w * q + min(w, r);
            cnt = q + (w < r ? 1 : 0);
        }
    }
#ifndef FIER_FS_L2PF
#define FIER_FS_L2PF 4
#endif
#if FIER_FS_L2PF > 0
    // The first slabs of every non-append warp are prefetched into L2 before the query read
    // (a PCIe round trip when q is host-resident): one bulk prefetch of their bit rows and
    // one of their groups' (s, z) rows per warp, nothing held in registers (loads into
    // registers here spilled at the 128-register cap).  A/B x3 on one box, C2 step / e2e us:
    // none 31.01 / 33.90, 3 slabs 30.71 / 33.64, 4 30.65 / 33.39, 6 30.73 / 33.29, 8 30.82 / 33.17.
    if (lane == 0 && !(appender && warp < 4) && cnt > 0 && a.g_shift >= 0) {
        const int nf = min(cnt, FIER_FS_L2PF);
        const int t0 = s0 + 32 * start;
        if (t0 + 32 * nf <= a.tokens) {
            const int g0 = t0 >> a.g_shift, g1 = (t0 + 32 * nf - 1) >> a.g_shift;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(bseq + (int64_t)t0 * 4),
                         "r"((uint32_t)nf * 512u) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(zseq + (int64_t)g0 * D),
                         "r"((uint32_t)(g1 - g0 + 1) * 512u) : "memory");
        }
    }
#endif
    float* qrot = reinterpret_cast<float*>(smem + kFsQrot);  // this head's query, rotated (RoPE)
    if (tid < kFsD) {
        const T* qh = static_cast<const T*>(a.q) + (int64_t)row * kFsD;
        // rotated in fp32, rounded to the cache dtype like the rotated k row (rope.cuh)
        qrot[tid] = to_f32(T(rope_channel(a.rope, tid, [&](int j) { return to_f32(qh[j]); })));
        // the query's logits cannot be finite ("softmax: non-finite logit", core.hpp:122)
        if (a.nonfinite && rank == 0 && __any_sync(0xffffffffu, !isfinite(qrot[tid])) && (tid & 31) == 0)
            atomicOr(a.nonfinite, 2);
    }
    __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    if (warp == 0) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    FS_MARK(0);

    // ---- phase A: append (the CTA whose slice holds pos; warps 0..3 re-pack the open
    // group while the other warps start scoring; the open group's slabs are scored last) ----
    if (appender && tid < D) {
        const T kv = T(rope_channel(a.rope, tid, [&](int j) { return to_f32(j == tid ? knr : knp); }));
        const T vv = vnr;
        // "quantize: non-finite key entry" (quant1bit.hpp:68) for the appended row
        if (a.nonfinite && __any_sync(0xffffffffu, !isfinite(to_f32(kv))) && (tid & 31) == 0) atomicOr(a.nonfinite, 1);
        FS_MARK(16);
        if (a.g <= 32)
            pack_open_group32<T>(D, a.g, a.pos / a.g, a.pos + 1, bseq, zseq, to_f32(kv), a.pos, vpre);
        else  // (an out-of-line call here measured +1 us on the whole step: register ABI)
            pack_open_group<T>(Kseq, D, a.g, a.pos / a.g, a.pos + 1, bseq, zseq, to_f32(kv), a.pos);
        FS_MARK(21);
        Kseq[(int64_t)a.pos * D + tid] = kv;  // after the re-pack: its loads do not queue behind this store
        Vseq[(int64_t)a.pos * D + tid] = vv;
    }

    FS_MARK(1);
    // ---- phase B: score this CTA's slice into shared-memory keys ----
    float qv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) qv[i] = qrot[4 * lane + i];
    const uint32_t tab0 = base + kFsLut + warp * kFsLutBytes;  // one table per warp (trace: 10.75 vs 11.0 us double-buffered)
    float* srow = a.scores ? a.scores + (int64_t)row * a.ld : nullptr;
    auto score_slab = [&](int sl, int u, const uint4& p, const uint4& bw) {
        const int t0 = s0 + 32 * sl, t = t0 + lane;
        uint32_t key = 0u;  // 0 = empty slot (past the row end, or NaN)
        if (t0 < a.tokens) {  // warp-uniform
            build_nibble_table(tab0, p, qv);
            __syncwarp();
            const float sc = nibble_score(tab0, bw);
            __syncwarp();  // every lane read the table before the next slab rebuilds it
            if (t < a.tokens) {
                key = score_key(sc);
                if (srow) srow[t] = sc;
            }
        }
        keys_s[32 * sl + lane] = key;
        rx_count(S, key);
    };
    auto load = [&](int sl, uint4& p, uint4& bw) {
        const int t0 = s0 + 32 * sl;
        p = make_uint4(0, 0, 0, 0);
        bw = make_uint4(0, 0, 0, 0);
        if (t0 < a.tokens) {
            const int gi = a.g_shift >= 0 ? t0 >> a.g_shift : t0 / a.g;
            p = ld_cg16(zseq + (int64_t)gi * D + 4 * lane);
            if (t0 + lane < a.tokens) bw = ld_cg16(bseq + (int64_t)(t0 + lane) * 4);
        }
    };
    if (appender && warp < 4) {
        // the append warps re-packed the open group: a named barrier over those four
        // warps publishes it, and they score the open (and empty) slabs first
        asm volatile("bar.sync 1, 128;" ::: "memory");
        FS_MARK(22);
        for (int sl = nsealed + warp; sl < nsl; sl += 4) {
            uint4 p, bw;
            load(sl, p, bw);
            score_slab(sl, sl, p, bw);
        }
        FS_MARK(23);
    }
    uint4 pb[PF], bb[PF];  // register ring: (s, z) and bit rows of the next PF slabs
    // Fast path: whole chunks of PF full, sealed slabs -- no per-slab bounds checks, a
    // compile-time inner loop (trace: the per-slab checks cost ~1 us of the C2 score phase).
    int nfast = 0;
    if (a.g_shift >= 0 && cnt >= PF) {
        const int full = min(cnt, (a.tokens - s0) / 32 - start);  // slabs whose 32 tokens all exist
        nfast = max(0, full) / PF * PF;
    }
    if (nfast > 0) {
        const uint32_t* bw0 = bseq + (int64_t)(s0 + 32 * start + lane) * 4;
        const int t00 = s0 + 32 * start;
        auto ld = [&](int j, uint4& p, uint4& bw) {
            p = ld_cg16(zseq + (int64_t)((t00 + 32 * j) >> a.g_shift) * D + 4 * lane);
            bw = ld_cg16(bw0 + (int64_t)j * 128);
        };
#pragma unroll
        for (int u = 0; u < PF; ++u) ld(u, pb[u], bb[u]);
        for (int j0 = 0; j0 < nfast; j0 += PF) {
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const int j = j0 + u;
                const uint4 p = pb[u], bw = bb[u];
                if (j + PF < nfast) ld(j + PF, pb[u], bb[u]);
                build_nibble_table(tab0, p, qv);
                __syncwarp();
                const float sc = nibble_score(tab0, bw);
                __syncwarp();  // every lane read the table before the next slab rebuilds it
                const uint32_t key = score_key(sc);
                if (srow) srow[s0 + 32 * (start + j) + lane] = sc;
                keys_s[32 * (start + j) + lane] = key;
                rx_count(S, key);
            }
        }
        start += nfast;
        cnt -= nfast;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u)
        if (u < cnt) load(start + u, pb[u], bb[u]);
    for (int j0 = 0; j0 < cnt; j0 += PF) {
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int j = j0 + u;
            if (j < cnt) {  // warp-uniform
                const uint4 p = pb[u], bw = bb[u];
                if (j + PF < cnt) load(start + j + PF, pb[u], bb[u]);
                score_slab(start + j, u, p, bw);
            }
        }
    }

    // ---- phase C: digit-1 bin over the cluster, partition of this CTA's keys ----
    FS_MARK(2);
    const SmemKeys keys{keys_s + wbase, kpt};  // phase C ownership: warp w, slot j, lane L
    uint32_t* amask = reinterpret_cast<uint32_t*>(smem + kFsMasks);
    uint32_t* kmask = amask + kFsWarps * kFsMaxKpt;
    int32_t* selrow = a.sel + (int64_t)row * a.k;
    const RxFind f = rx_find<kFsThreads>(nct, a.k, S, P, cbar);
    int nlist;  // gather-list rows known to every warp at the split
    if (!f.over) {
        rx_partition<kFsThreads>(keys, s0, wbase, f.b1, S, P, amask, kmask, sidx);
        T2_MARK(10);
        __syncthreads();  // P and the gather list complete: cluster barrier 2 (as in rx_find)
        if (warp == 0) {
            if (lane < nct) mbar_arrive_remote(smem_u32(cbar + 1), lane);
            mbar_wait(cbar + 1, 0);
        }
        // only the select warps read the peers' candidates; the gather warps start on the
        // rows above b1 as soon as no peer reads this CTA's histogram any more (cbar[3])
        if (warp < kFsSelWarps) NamedBar<2, kFsSelThreads>::sync();
        T2_MARK(11);
        nlist = (int)S.nabove;
    } else {  // candidate overflow (very narrow score range): exact MSD radix select, all warps
        if (warp != 0) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // (its cluster.sync)
        uint32_t cbase = 0, ccount = 0;
        fused_fallback_select(cluster, keys, a.k, S, selrow, sidx, s0, wbase, &cbase, &ccount);
        __syncthreads();  // (the fallback select's shared state overlays RxShared)
        if (tid == 0) S.gclaim = 0u;
        __syncthreads();
        nlist = (int)ccount;
    }

    // ---- phase D: the gather warps attend over the keys above b1 while the select warps
    // resolve the candidates, append the kept ones to the list and write the selection ----
    if (warp >= kFsSelWarps) {
        const int gw = warp - kFsSelWarps;
        uint32_t qb[D / 16][2];
        tc_load_q_f32<T, D, 1>(qrot, qb);
        TcState<D> st;
        st.init();
        const uint32_t ring = base + kFsRing + (uint32_t)gw * kFsNst * 2 * tc_stage_bytes<D>();
        auto tok = [&](int r) { return s0 + (int)sidx[r]; };
        // The granules (16 rows) form one CTA-wide queue: the rows above b1, then the kept
        // candidates once the select warps have listed them (mbarrier kready).  Each warp
        // claims its next granule from a shared counter one ring stage ahead, so the warps
        // whose rows come back early take more, and no warp waits for the others.
        const int nga = (nlist + kTcRows - 1) / kTcRows;  // granules above b1
        int nk = -1;                                       // kept candidates, once listed
        int m0 = -1, m0r = 0, m0n = 0, m1 = -1, m1r = 0, m1n = 0;  // claims of granules sg (even, odd)
        auto gran = [&](int sg, int& r0) {
            if (sg & 1) {
                if (m1 == sg) return r0 = m1r, m1n;
            } else if (m0 == sg) {
                return r0 = m0r, m0n;
            }
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd(&S.gclaim, 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            int nr;
            if ((int)c < nga) {
                r0 = (int)c * kTcRows;
                nr = min(kTcRows, nlist - r0);
            } else {
                if (nk < 0) {  // first claim past the rows above b1: wait for the list
                    nk = 0;
                    if (!f.over) {
                        mbar_wait(kready, 0);
                        nk = (int)S.nkept;
                    }
                    FS_MARK_T(15, kFsSelThreads);
                }
                r0 = nlist + ((int)c - nga) * kTcRows;
                nr = min(kTcRows, nlist + nk - r0);
            }
            if (sg & 1) {
                m1 = sg, m1r = r0, m1n = nr;
            } else {
                m0 = sg, m0r = r0, m0n = nr;
            }
            return nr;
        };
        if (!f.over) mbar_wait(cbar + 3, 0);  // the rings overlay the histogram the peers read
        tc_stream_granules<T, D, true, kFsNst>(qb, Kseq, Vseq, ring, a.scale_log2, gran, tok, st);
        tc_store_state<D, 1>(st, wres + gw * (D + 2));
        FS_MARK_T(5, kFsSelThreads);
    } else if (!f.over) {
        using SelBar = NamedBar<2, kFsSelThreads>;
        const RxResult rx = rx_resolve<kFsSelThreads, SelBar>(cluster, s0, slice, f.krem, S, P, kmask, sidx + nlist);
        FS_MARK(3);
        mbar_arrive_local(kready);  // release: this thread's kept-list entries and S.nkept
        rx_emit_masks<kFsSelThreads, kFsWarps, kFsMaxKpt, SelBar>(rx, kpt, amask, kmask, S, [&](uint32_t slot, int kw, int j) {
            selrow[slot] = s0 + kw * 32 * kpt + 32 * j + lane;
        });
        FS_MARK(4);
    }
    __syncthreads();
    // CTA partial -> rank 0's cres[rank] over DSMEM
    float* dst = cluster.map_shared_rank(cres, 0) + rank * (D + 2);
    if (tid < D) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kFsGatherWarps; ++w) M = fmaxf(M, wres[w * (D + 2) + D]);
        float oo = 0.f, L = 0.f;
#pragma unroll
        for (int w = 0; w < kFsGatherWarps; ++w) {
            const float* xx = wres + w * (D + 2);
            const float sc = xx[D] == -INFINITY ? 0.f : exp2f(xx[D] - M);
            oo = fmaf(xx[tid], sc, oo);
            L = fmaf(xx[D + 1], sc, L);
        }
        dst[tid] = oo;
        if (tid == 0) {
            dst[D] = M;
            dst[D + 1] = L;
        }
    }
    __syncthreads();  // partial written: cluster barrier 3, after which no CTA reads a peer
    if (warp == 0) {
        if (lane < nct) mbar_arrive_remote(smem_u32(cbar + 2), lane);
        mbar_wait(cbar + 2, 0);
    }
    FS_MARK(6);
    if (rank != 0) return;
    __syncthreads();  // rank 0: every partial is in cres
    if (tid >= D) return;
    float M = -INFINITY;
    for (int r = 0; r < nct; ++r) M = fmaxf(M, cres[r * (D + 2) + D]);
    float oo = 0.f, L = 0.f;
    for (int r = 0; r < nct; ++r) {
        const float* xx = cres + r * (D + 2);
        if (xx[D] == -INFINITY) continue;
        const float sc = exp2f(xx[D] - M);
        oo = fmaf(xx[tid], sc, oo);
        L = fmaf(xx[D + 1], sc, L);
    }
    a.out[(int64_t)row * D + tid] = L > 0.f ? oo / L : 0.f;
    FS_MARK(7);
}

// ---- host side -------------------------------------------------------------------

template <typename T>
static int launch_fused(int cluster, int rows, const FsArgs& args, cudaStream_t st) {
    auto kern = step_fused_kernel<T>;
    static const bool ok = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kFsSmem);
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return true;
    }();
    (void)ok;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, rows, 1);
    cfg.blockDim = dim3(kFsThreads, 1, 1);
    cfg.dynamicSmemBytes = kFsSmem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cluster;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args);
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string("fier_decode_step: ") + cudaGetErrorString(e));
    return FIER_OK;
}

// Cluster size and keys per thread for `tokens` per row: one CTA per SM (the
// smem footprint), the whole grid in one wave when it fits, >= 2 slabs per warp.
static bool fused_plan(int rows, int tokens, int g, int* cluster, int* kpt) {
    int c = 1;
    while (c < kT2MaxCluster && ceil_div(tokens, c) > (int64_t)kFsThreads * kFsMaxKpt) c *= 2;
    if (ceil_div(tokens, c) > (int64_t)kFsThreads * kFsMaxKpt) return false;
    while (c < kT2MaxCluster && (int64_t)rows * c * 2 <= num_sms() && ceil_div(tokens, 2 * c) >= 2 * kFsThreads) c *= 2;
    int k = (int)ceil_div(ceil_div(tokens, c), kFsThreads);
    while (((int64_t)kFsThreads * k) % g != 0) ++k;  // the open group lies inside one CTA's slice
    if (k > kFsMaxKpt) return false;
    *kpt = k;
    *cluster = (int)ceil_div(tokens, (int64_t)kFsThreads * k);
    return true;
}

static bool fused_shape_ok(const fier_shape* s) {
    if (s->q_heads != s->kv_heads || s->dim != kFsD || s->group % 32 != 0) return false;
    return s->dtype == FIER_BF16 || s->dtype == FIER_F16;
}

bool fused_step_applies(const fier_shape* s, int tokens) {
    int cluster = 0, kpt = 0;
    return fused_shape_ok(s) && s->batch * s->q_heads <= 65535 &&
           fused_plan(s->batch * s->q_heads, tokens, s->group, &cluster, &kpt);
}

// Returns -1 when the shape is not covered (the caller runs the separate kernels).
int fused_step_dispatch(const fier_shape* s, const void* q, const void* k_new, const void* v_new, int pos, void* K,
                        void* V, uint32_t* bits, void* params, int n, float scale, const fier_rope* rope,
                        float* out, int32_t* sel, float* scores_out, int64_t ld, int32_t* nonfinite,
                        cudaStream_t st) {
    if (!fused_shape_ok(s)) return -1;
    const int tokens = pos + 1, rows = s->batch * s->q_heads;
    if (rows > 65535) return -1;
    int cluster = 0, kpt = 0;
    if (!fused_plan(rows, tokens, s->group, &cluster, &kpt)) return -1;
    FsArgs args;
    args.q = q;
    args.K = K;
    args.V = V;
    args.k_new = k_new;
    args.v_new = v_new;
    args.bits = bits;
    args.sz = static_cast<__half2*>(params);
    args.scores = scores_out;
    args.out = out;
    args.sel = sel;
    args.ld = ld;
    args.pos = pos;
    args.tokens = tokens;
    args.cap = s->capacity;
    args.G = (int)ceil_div(s->capacity, s->group);
    args.hq = s->q_heads;
    args.g = s->group;
    args.g_shift = (s->group & (s->group - 1)) == 0 ? __builtin_ctz(s->group) : -1;
    args.k = n;
    args.kpt = kpt;
    args.scale_log2 = scale * kLog2e;
    args.rope = rope_table(rope, pos);
    args.nonfinite = nonfinite;
    if (s->dtype == FIER_BF16) return launch_fused<__nv_bfloat16>(cluster, rows, args, st);
    return launch_fused<__half>(cluster, rows, args, st);
}

}  // namespace fier_cuda

#ifdef FIER_STEP_TRACE
// max co-resident clusters of the bf16 instance at this cluster size
extern "C" FIER_API int fier_debug_step_occupancy(int cluster) {
    auto kern = fier_cuda::step_fused_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, fier_cuda::kFsSmem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, 64, 1);
    cfg.blockDim = dim3(fier_cuda::kFsThreads, 1, 1);
    cfg.dynamicSmemBytes = fier_cuda::kFsSmem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cluster;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = -1;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return -1;
    return n;
}

extern "C" FIER_API int fier_debug_step_trace_clear(void) {
    static unsigned long long zeros[fier_cuda::kFsTraceCtas][fier_cuda::kFsTraceMarks];
    return cudaMemcpyToSymbol(fier_cuda::g_fs_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 3;
}

extern "C" FIER_API int fier_debug_step_trace(unsigned long long* host, int ctas) {
    const int n = ctas < fier_cuda::kFsTraceCtas ? ctas : fier_cuda::kFsTraceCtas;
    return cudaMemcpyFromSymbol(host, fier_cuda::g_fs_trace, (size_t)n * fier_cuda::kFsTraceMarks * sizeof(unsigned long long)) ==
                   cudaSuccess
               ? 0
               : 3;
}
#endif
