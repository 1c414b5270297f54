// rope.cuh -- rotary position embedding inside the decode step (SURVEY §8(f) row 1:
// the KV write + RoPE + append-pack that precedes scoring in a real decode loop).
//
// The host evaluates cos/sin of pos * base^(-2i/rd) in double for the step's position
// and passes the table by value (RopeTable), so the kernels only multiply-add.
// Channel c < rd of a head vector x:
//   rotate_half (NeoX / Llama): c <  rd/2: x[c] cos_c - x[c + rd/2] sin_c
//                               c >= rd/2: x[c] cos_i + x[c - rd/2] sin_i,  i = c - rd/2
//   interleaved (GPT-J):        c even:    x[c] cos_i - x[c + 1] sin_i,      i = c / 2
//                               c odd:     x[c] cos_i + x[c - 1] sin_i
// Channels >= rd pass through.  The rotation is evaluated in fp32 and the rotated q and
// k rows are rounded to the cache dtype: the step then uses them exactly as if the
// model had applied RoPE before calling it (the cache stores the rounded k row).
#pragma once

#include "common.cuh"

namespace fier_cuda {

constexpr int kRopeMaxPairs = 64;  // rd <= 128

struct RopeTable {
    int rd;  // 0: no rotation
    int interleaved;
    float cs[kRopeMaxPairs];
    float sn[kRopeMaxPairs];
};

// Host: the table of one position (double-precision angles).
inline RopeTable rope_table(const fier_rope* r, int pos) {
    RopeTable t = {};
    if (!r) return t;
    t.rd = r->rotary_dim;
    t.interleaved = r->interleaved ? 1 : 0;
    for (int i = 0; i < t.rd / 2; ++i) {
        const double ang = (double)pos * pow((double)r->base, -2.0 * i / t.rd);
        t.cs[i] = (float)cos(ang);
        t.sn[i] = (float)sin(ang);
    }
    return t;
}

// Rotated channel c of x (x(j) = channel j of the unrotated vector, as float).
// The other channel rope_channel(t, c, x) reads (c itself when c is not rotated).
__device__ __forceinline__ int rope_partner(const RopeTable& t, int c) {
    if (c >= t.rd) return c;
    if (t.interleaved) return c ^ 1;
    const int h = t.rd >> 1;
    return c < h ? c + h : c - h;
}

template <typename Ld>
__device__ __forceinline__ float rope_channel(const RopeTable& t, int c, Ld&& x) {
    if (c >= t.rd) return x(c);
    if (t.interleaved) {
        const int i = c >> 1;
        return (c & 1) ? fmaf(x(c), t.cs[i], x(c - 1) * t.sn[i]) : fmaf(x(c), t.cs[i], -x(c + 1) * t.sn[i]);
    }
    const int h = t.rd >> 1;
    return c < h ? fmaf(x(c), t.cs[c], -x(c + h) * t.sn[c]) : fmaf(x(c), t.cs[c - h], x(c - h) * t.sn[c - h]);
}

}  // namespace fier_cuda
