// nibble.cuh -- the nibble-table scorer of the fused decode step (step_fused.cu):
// approx_scores (reference quant1bit.hpp:121-140) for one 32-token slab per warp,
// lane = token.  For each 4-channel nibble position p the 16 table entries hold
//     sum_{i in p} q_i (z_i - s_i) + sum_{i in p, bit i set} 2 q_i s_i,
// so a token's score is the sum of 32 table reads, one per nibble of its 128-bit
// row: one PRMT (address), one LDS, one FADD per 4 bits.
#pragma once

#include "common.cuh"

namespace fier_cuda {

constexpr int kNibTableBytes = 32 * 16 * 4;  // one table: 32 nibble positions x 16 fp32 entries

#ifndef FIER_NO_EVICT_FIRST
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
#endif

__device__ __forceinline__ uint4 ld_cg16(const void* p) {
    uint4 v;
#ifndef FIER_NO_EVICT_FIRST
    asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(l2_evict_first_policy()));
#else
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
#endif
    return v;
}

__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ void sts_v4(uint32_t a, float x, float y, float z, float w) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

// Table layout: position p owns the 64-byte row p; its 16-byte granule i (entries
// 4i..4i+3) is stored at granule i ^ h(p), h(p) = (p >> 1) & 3.  The build (lane p
// stores row p with 4 x 16-byte stores) then spreads every store instruction over all
// 32 banks (4 wavefronts instead of 16), and a lookup (all lanes read row p) still
// touches 16 distinct banks.  The swizzle of nibble byte i of a word is i << 4
// (positions 8w + 2i and 8w + 2i + 1 both have h = i), folded into the LOP3 mask.
constexpr uint32_t kFsSwz = 0x30201000u;

// Lane p builds nibble position p of the table at `tab`: channels 4p..4p+3,
// p4 = this lane's (s, z) half2 x 4, q = this lane's 4 query channels.
__device__ __forceinline__ void build_nibble_table(uint32_t tab, const uint4& p4, const float (&q)[4]) {
    const int lane = threadIdx.x & 31;
    const __half2* ph = reinterpret_cast<const __half2*>(&p4);
    float w[4], bz = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(ph[i]);  // (s, z)
        w[i] = 2.f * q[i] * f.x;
        bz = fmaf(q[i], f.y - f.x, bz);
    }
    float e[16];
    e[0] = bz;
    e[1] = bz + w[0];
    e[2] = bz + w[1];
    e[3] = e[1] + w[1];
#pragma unroll
    for (int i = 0; i < 4; ++i) e[4 + i] = e[i] + w[2];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[8 + i] = e[i] + w[3];
    const uint32_t a = tab + lane * 64;
    const uint32_t h = ((lane >> 1) & 3) << 4;
    sts_v4(a + (0u ^ h), e[0], e[1], e[2], e[3]);
    sts_v4(a + (16u ^ h), e[4], e[5], e[6], e[7]);
    sts_v4(a + (32u ^ h), e[8], e[9], e[10], e[11]);
    sts_v4(a + (48u ^ h), e[12], e[13], e[14], e[15]);
}

// Score of this lane's token from its 4-word bit row through the table at `tab`
// (tab % 256 == 0: PRMT splices the swizzled nibble offset into the address's low byte).
__device__ __forceinline__ float nibble_score(uint32_t tab, const uint4& bw) {
    const uint32_t words[4] = {bw.x, bw.y, bw.z, bw.w};
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
        const uint32_t x = words[wd];
        const uint32_t ev = ((x << 2) & 0x3C3C3C3Cu) ^ kFsSwz;  // nibbles 0,2,4,6 (x4) in bytes 0..3
        const uint32_t od = ((x >> 2) & 0x3C3C3C3Cu) ^ kFsSwz;  // nibbles 1,3,5,7 (x4)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int pe = wd * 8 + 2 * i;  // nibble position of ev byte i
            acc[i] += lds_f32(__byte_perm(ev, tab, 0x7650u + i) + pe * 64);
            acc[(i + 2) & 3] += lds_f32(__byte_perm(od, tab, 0x7650u + i) + (pe + 1) * 64);
        }
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

}  // namespace fier_cuda
