// pack.cuh -- the 1-bit group packer shared by K1 (pack.cu) and the fused
// append+score launch (score.cu).  See pack.cu for the reference mapping.
#pragma once

#include "common.cuh"

namespace fier_cuda {

constexpr int kPackThreads = 128;  // 4 warps; warp w packs channel slices w, w+4, ...

// Arithmetic type of the packer: 16/32-bit keys are exact in fp32; fp64 keys (the
// reference's own KeyCache type) stay fp64 end to end.
template <typename T>
struct PackVal {
    using type = float;
    __device__ static float get(T x) { return to_f32(x); }
};
template <>
struct PackVal<double> {
    using type = double;
    __device__ static double get(double x) { return x; }
};
__device__ __forceinline__ bool pack_finite(float x) { return isfinite(x); }
__device__ __forceinline__ bool pack_finite(double x) { return isfinite(x); }

// Values of one 32-token chunk of this lane's channel, loaded together (one
// memory latency per chunk instead of one per token).  bf16/fp16/fp32 are
// exact in fp32; they are widened to fp64 for the arithmetic below.  Token
// tnew (the row a decode-time append is storing right now) takes the value
// xnew, read from the appended row itself, so the group's loads do not wait
// behind the store (the loaded copy of that row is discarded).
template <typename T, typename VT = typename PackVal<T>::type>
__device__ __forceinline__ void load_chunk(const T* Kseq, int d, int c, bool valid,
                                           int tc, int cnt, VT (&v)[32], VT xnew, int tnew) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        // read-only path: the only row this launch writes (tnew) is stored after the
        // re-pack, and its loaded copy is discarded
        const VT x = (valid && i < cnt) ? PackVal<T>::get(__ldg(Kseq + (int64_t)(tc + i) * d + c)) : VT(0);
        v[i] = tc + i == tnew ? xnew : x;
    }
}

template <typename T>
__device__ __forceinline__ void pack_group(const T* Kseq,  // no restrict: append re-reads its own store
                                           int d, int W, int g, int gi,
                                           int t_end, uint32_t* __restrict__ bits_seq,
                                           __half2* __restrict__ sz_seq, int32_t* nonfinite,
                                           const T* nrow = nullptr, int tnew = -1) {
    const int lane = threadIdx.x & 31;
    for (int warp = threadIdx.x >> 5; warp < W; warp += blockDim.x >> 5) {
    const int c = warp * 32 + lane;
    const bool valid = c < d;
    const int t0 = gi * g;
    const int t1 = min(t0 + g, t_end);  // short final group (quant1bit.hpp:84)
    using VT = typename PackVal<T>::type;
    VT v[32];
    const VT xnew = (nrow && valid) ? PackVal<T>::get(nrow[c]) : VT(0);
    // min/max on the exact values (fp32 holds every 16/32-bit key exactly, == its fp64
    // widening), sequential with std::min/std::max semantics: a tie keeps the
    // first-seen value (+0 vs -0).
    VT mn = 0, mx = 0;
    bool bad = false;
    for (int tc = t0; tc < t1; tc += 32) {
        const int cnt = min(32, t1 - tc);
        load_chunk<T>(Kseq, d, c, valid, tc, cnt, v, xnew, tnew);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            if (i < cnt) {
                const VT x = v[i];
                bad |= !pack_finite(x);
                if (tc == t0 && i == 0) {
                    mn = mx = x;
                } else {
                    mn = (x < mn) ? x : mn;
                    mx = (mx < x) ? x : mx;
                }
            }
        }
    }
    // z, s in fp64 exactly as the reference (quant1bit.hpp:90-93)
    const double z = ((double)mx + (double)mn) / 2.0;
    const double s = ((double)mx - (double)mn) / 2.0;
    if (valid) sz_seq[(int64_t)gi * d + c] = __halves2half2(__double2half(s), __double2half(z));
    if (bad && nonfinite) atomicOr(nonfinite, 1);  // FIER_NONFINITE_KEY
    // x >= z (fp64) <=> x >= zc for fp32 x, zc = the smallest float >= z (fp64 keys: z).
    VT zc;
    if constexpr (sizeof(VT) == 8) {
        zc = z;
    } else {
        zc = __double2float_rn(z);
        if ((double)zc < z) zc = nextafterf(zc, INFINITY);
    }
    const bool all_one = (s == 0.0);
    // pass 2: one ballot per token -> the word of (token, 32 channels); for
    // g <= 32 the chunk is still in registers.
    for (int tc = t0; tc < t1; tc += 32) {
        const int cnt = min(32, t1 - tc);
        if (g > 32) load_chunk<T>(Kseq, d, c, valid, tc, cnt, v, xnew, tnew);
        uint32_t mine = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            if (i < cnt) {
                const uint32_t word = __ballot_sync(0xffffffffu, valid && (all_one || v[i] >= zc));
                if (lane == i) mine = word;
            }
        }
        if (lane < cnt) bits_seq[(int64_t)(tc + lane) * W + warp] = mine;
    }
    }  // channel slices
}

// The open-group re-pack's two halves, shared by pack_open_group and pack_open_group32:
// z / s in fp64 from the first-seen min / max, stored as the group's half2 (s, z); returns
// zc, the smallest float >= z (x >= z in fp64 <=> x >= zc for fp32 x).
__device__ __forceinline__ float open_group_params(float mn, float mx, bool valid, __half2* dst, bool& all_one) {
    const double z = ((double)mx + (double)mn) / 2.0;
    const double s = ((double)mx - (double)mn) / 2.0;
    if (valid) *dst = __halves2half2(__double2half(s), __double2half(z));
    float zc = __double2float_rn(z);
    if ((double)zc < z) zc = nextafterf(zc, INFINITY);
    all_one = (s == 0.0);
    return zc;
}

// One ballot per token of a 32-token chunk -> lane i holds token i's word (its warp's 32
// channels); lanes < cnt store it.
__device__ __forceinline__ void open_group_bits(const float (&v)[32], int cnt, bool valid, float zc, bool all_one,
                                                uint32_t* words, int W) {
    const int lane = threadIdx.x & 31;
    uint32_t mine = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const uint32_t word = __ballot_sync(0xffffffffu, valid && (all_one || v[i] >= zc));
        mine = lane == i ? word : mine;
    }
    if (lane < cnt) words[(int64_t)lane * W] = mine;
}

// Decode-time re-pack of the open group [gi*g, t_end) (one group per launch, so
// the code stays small: no divergent unrolled paths).  Threads [0, 32*W) take
// part, thread c owns channel c; the same rules as pack_group (first-seen
// min/max, fp64 z/s, cvt.rn.f16.f64, compare against the unrounded z).  Token
// tnew takes the value xnew (this thread's channel of the row being appended,
// already rounded to T) instead of a load that would wait behind its store.
template <typename T>
__device__ __forceinline__ void pack_open_group(const T* Kseq,  // no restrict: re-reads the appended row
                                                int d, int g, int gi, int t_end, uint32_t* __restrict__ bits_seq,
                                                __half2* __restrict__ sz_seq, float xnew = 0.f,
                                                int tnew = -1) {
    const int W = (d + 31) / 32;
    const int c = threadIdx.x, w = c >> 5;
    if (w >= W) return;
    const bool valid = c < d;
    const int t0 = gi * g;
    const int t1 = min(t0 + g, t_end);  // short final group (quant1bit.hpp:84)
    float mn = 0.f, mx = 0.f;
    float v[32];  // the current chunk (g <= 32: the whole group, reused by the ballot pass)
    auto load = [&](int tc) {  // chunks of 32 tokens: 32 loads in flight
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int t = min(tc + i, t1 - 1);  // past the end: repeat the last token (no effect)
            v[i] = !valid ? 0.f : t == tnew ? xnew : to_f32(Kseq[(int64_t)t * d + c]);
        }
    };
    for (int tc = t0; tc < t1; tc += 32) {
        load(tc);
        if (tc == t0) mn = mx = v[0];
#pragma unroll
        for (int i = 0; i < 32; ++i) {  // std::min/max: a tie keeps the first-seen value
            mn = (v[i] < mn) ? v[i] : mn;
            mx = (mx < v[i]) ? v[i] : mx;
        }
    }
    bool all_one;
    const float zc = open_group_params(mn, mx, valid, sz_seq + (int64_t)gi * d + c, all_one);
    for (int tc = t0; tc < t1; tc += 32) {
        if (t1 - t0 > 32) load(tc);  // g > 32: reload this chunk
        open_group_bits(v, t1 - tc, valid, zc, all_one, bits_seq + (int64_t)tc * W + w, W);
    }
}

// The open group's first 32 rows, channel threadIdx.x (token t0 + i clamped to t1 - 1), raw:
// issued by a caller that wants them in flight before other traffic (step_fused.cu) and
// converted only where pack_open_group32 uses them, so the loads do not stall the caller.
template <typename T>
__device__ __forceinline__ void open_group_preload(const T* Kseq, int d, int t0, int t1, T (&raw)[32]) {
    const int c = threadIdx.x;
    if (c < d) {
#pragma unroll
        for (int i = 0; i < 32; ++i) raw[i] = Kseq[(int64_t)min(t0 + i, t1 - 1) * d + c];
    }
}

// pack_open_group for g <= 32 from open_group_preload's rows (token tnew -> xnew).
template <typename T>
__device__ __forceinline__ void pack_open_group32(int d, int g, int gi, int t_end, uint32_t* __restrict__ bits_seq,
                                                  __half2* __restrict__ sz_seq, float xnew, int tnew,
                                                  const T (&raw)[32]) {
    const int W = (d + 31) / 32;
    const int c = threadIdx.x, w = c >> 5;
    if (w >= W) return;
    const bool valid = c < d;
    const int t0 = gi * g;
    const int t1 = min(t0 + g, t_end);
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = !valid ? 0.f : min(t0 + i, t1 - 1) == tnew ? xnew : to_f32(raw[i]);
    float mn = v[0], mx = v[0];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        mn = (v[i] < mn) ? v[i] : mn;
        mx = (mx < v[i]) ? v[i] : mx;
    }
    bool all_one;
    const float zc = open_group_params(mn, mx, valid, sz_seq + (int64_t)gi * d + c, all_one);
    open_group_bits(v, t1 - t0, valid, zc, all_one, bits_seq + (int64_t)t0 * W + w, W);
}

}  // namespace fier_cuda
