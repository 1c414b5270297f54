// topk64.cu -- topk_oracle (reference core.hpp:134-148) on fp64 scores, exact.
//
// The decode path ranks fp32 scores (K2's output, topk2.cu).  The reference's own
// ScoreVector holds doubles, and distinct doubles can round to the same float, so the
// C++ drop-in (fier_cuda.hpp topk_oracle / select_for_policy's oracle branch) ranks
// fp64 scores here instead: order-preserving u64 keys, an exact MSD radix select of the
// k-th largest key (six 11-bit digits, one CTA per row, shared-memory histograms), then
// one ordered pass keeping every key above the threshold and the lowest-index ties
// (ascending output, core.hpp:139-146).  -0.0 and +0.0 tie, as doubles compare.  Not a
// hot path: the drop-in's fp64 inputs only.
#include "common.cuh"

namespace fier_cuda {

constexpr int kT64Threads = 1024;
constexpr int kT64Bits = 11;
constexpr int kT64Bins = 1 << kT64Bits;

__device__ __forceinline__ uint64_t double_key(double x) {
    if (isnan(x)) return 0ull;  // NaN ranks below everything
    uint64_t u = __double_as_longlong(x);
    if (x == 0.0) u = 0ull;
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(kT64Threads) topk64_kernel(const double* __restrict__ scores, int tokens,
                                                             int64_t ld, int k, int32_t* __restrict__ sel) {
    __shared__ uint32_t hist[kT64Bins];
    __shared__ uint32_t wsum[kT64Threads / 32];
    __shared__ uint64_t s_prefix;
    __shared__ uint32_t s_krem, s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* row = scores + (int64_t)blockIdx.x * ld;
    int32_t* out = sel + (int64_t)blockIdx.x * k;
    uint64_t prefix = 0, mask = 0;  // the threshold's digits found so far
    uint32_t krem = (uint32_t)k;    // rank of the threshold among the keys matching prefix
    for (int shift = 64 - kT64Bits; shift > -kT64Bits; shift -= kT64Bits) {
        const int sh = shift < 0 ? 0 : shift;
        const int width = shift < 0 ? kT64Bits + shift : kT64Bits;  // the last digit is narrower
        const uint64_t dmask = ((1ull << width) - 1) << sh;
        for (int i = tid; i < kT64Bins; i += kT64Threads) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < tokens; i += kT64Threads) {
            const uint64_t key = double_key(row[i]);
            if ((key & mask) == prefix) atomicAdd(&hist[(key & dmask) >> sh], 1u);
        }
        __syncthreads();
        if (warp == 0) {  // bin of the krem-th largest: scan from the top bin down
            uint32_t above = 0;
            int found = -1;
            uint32_t kr = krem;
            for (int base = kT64Bins - 32; base >= 0 && found < 0; base -= 32) {
                const uint32_t c = hist[base + lane];
                // suffix sums within the 32 bins (bins above this lane's, in this chunk)
                uint32_t suf = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_down_sync(0xffffffffu, suf, o);
                    if (lane + o < 32) suf += y;
                }
                const uint32_t hi = above + suf - c;  // keys in bins above this lane's
                const bool hit = c > 0 && hi < kr && kr <= hi + c;
                const uint32_t m = __ballot_sync(0xffffffffu, hit);
                if (m) {
                    const int l = 31 - __clz(m);
                    found = base + l;
                    kr -= __shfl_sync(0xffffffffu, hi, l);
                }
                above += __shfl_sync(0xffffffffu, suf, 0);
            }
            if (lane == 0) {
                s_prefix = prefix | ((uint64_t)found << sh);
                s_krem = kr;
            }
        }
        __syncthreads();
        prefix = s_prefix;
        krem = s_krem;
        mask |= dmask;
    }
    // prefix = the k-th largest key T; krem = how many T-valued keys to keep (lowest indices)
    const uint64_t T = prefix;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    uint32_t ties_before = 0;  // T-valued keys in earlier chunks (identical in every thread)
    for (int c0 = 0; c0 < tokens; c0 += kT64Threads) {
        const int i = c0 + tid;
        const uint64_t key = i < tokens ? double_key(row[i]) : 0ull;
        const bool tie = i < tokens && key == T;
        // rank of this tie among the chunk's ties (block scan of the tie flags)
        const uint32_t tb = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) wsum[warp] = __popc(tb);
        __syncthreads();
        uint32_t tpre = 0, ttot = 0;
        for (int w = 0; w < kT64Threads / 32; ++w) {
            const uint32_t v = wsum[w];
            tpre += w < warp ? v : 0u;
            ttot += v;
        }
        const uint32_t trank = ties_before + tpre + __popc(tb & ((1u << lane) - 1u));
        const bool keep = i < tokens && (key > T || (tie && trank < krem));
        __syncthreads();
        const uint32_t kb = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[warp] = __popc(kb);
        __syncthreads();
        uint32_t kpre = 0, ktot = 0;
        for (int w = 0; w < kT64Threads / 32; ++w) {
            const uint32_t v = wsum[w];
            kpre += w < warp ? v : 0u;
            ktot += v;
        }
        if (keep) out[s_carry + kpre + __popc(kb & ((1u << lane) - 1u))] = i;
        __syncthreads();
        if (tid == 0) s_carry += ktot;
        ties_before += ttot;
        __syncthreads();
    }
}

}  // namespace fier_cuda

using namespace fier_cuda;

extern "C" int fier_topk_f64(const double* scores, int32_t rows, int32_t tokens, int64_t ld, int32_t k, int32_t* sel,
                             void* stream) {
    FIER_REQUIRE(rows >= 1, "topk_oracle: rows out of range");
    FIER_REQUIRE(k >= 1 && k <= tokens, "topk_oracle: k out of range");
    FIER_REQUIRE(ld >= tokens, "topk_oracle: score row stride shorter than tokens");
    FIER_REQUIRE(scores && sel, "topk_oracle: null buffer");
    topk64_kernel<<<rows, kT64Threads, 0, static_cast<cudaStream_t>(stream)>>>(scores, tokens, ld, k, sel);
    return check_launch("fier_topk_f64");
}
