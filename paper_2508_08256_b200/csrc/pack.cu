// pack.cu -- K1: 1-bit key packer (bulk prefill + decode-time append).
//
// Replaces quantize (reference quant1bit.hpp:65-103).  One CTA per
// (group, kv head, sequence); warp w owns channels [32w, 32w+32), lane = channel.
//   * min/max scanned sequentially over the group's tokens in the input dtype
//     widened exactly to fp64 (fp64 keys -- the reference's own KeyCache type,
//     core.hpp:24-68 -- are taken as they are), first-seen wins ties (std::min/std::max at
//     quant1bit.hpp:85-89 -- matters for the sign of zero),
//   * z = (mx+mn)/2, s = (mx-mn)/2 in fp64 (:90-93), stored RNE to binary16
//     with cvt.rn.f16.f64 (= double_to_half, half.hpp:30-61),
//   * bit = (s == 0 || k >= z) against the UNROUNDED fp64 z (:96), produced
//     32 tokens-at-a-time by __ballot_sync over the channel lanes: one u32 word
//     per (token, 32 channels).
// The append variant first writes the new k/v row (the KV-cache update that
// precedes scoring in a decode step), then re-packs only the open group.
#include "pack.cuh"

namespace fier_cuda {

template <typename T>
__global__ void __launch_bounds__(kPackThreads) pack_kernel(const T* __restrict__ K, int cap, int d, int W,
                                                     int g, int G, int tokens, int hkv,
                                                     uint32_t* __restrict__ bits,
                                                     __half2* __restrict__ sz, int32_t* nonfinite) {
    const int gi = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int64_t seq = (int64_t)b * hkv + h;
    pack_group<T>(K + seq * cap * d, d, W, g, gi, tokens, bits + seq * cap * W, sz + seq * G * d,
                  nonfinite);
}

template <typename T>
__global__ void __launch_bounds__(kPackThreads) append_kernel(T* __restrict__ K, T* __restrict__ V,
                                                       const T* __restrict__ k_new,
                                                       const T* __restrict__ v_new, int pos, int cap,
                                                       int d, int W, int g, int G, int hkv,
                                                       uint32_t* __restrict__ bits,
                                                       __half2* __restrict__ sz, int32_t* nonfinite,
                                                       int* zero_words, int zero_n) {
    const int h = blockIdx.y, b = blockIdx.z;
    const int64_t seq = (int64_t)b * hkv + h;
    T* Kseq = K + seq * cap * d;
    if (zero_words) {  // the fused step's attention-merge counters (stream-ordered before K4)
        const int per = (zero_n + gridDim.y * gridDim.z - 1) / (gridDim.y * gridDim.z);
        for (int i = threadIdx.x; i < per; i += blockDim.x) {
            const int64_t j = seq * per + i;
            if (j < zero_n) zero_words[j] = 0;
        }
    }
    // The group re-pack takes token pos from k_new; the K/V row stores follow it,
    // so the group's loads do not queue behind them.
    pack_group<T>(Kseq, d, W, g, pos / g, pos + 1, bits + seq * cap * W, sz + seq * G * d,
                  nonfinite, k_new + seq * d, pos);
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        Kseq[(int64_t)pos * d + c] = k_new[seq * d + c];
        V[seq * cap * d + (int64_t)pos * d + c] = v_new[seq * d + c];
    }
}

template <typename T>
static int launch_pack(const fier_shape* s, const void* K, int32_t tokens, uint32_t* bits,
                       void* params, int32_t* nonfinite, cudaStream_t st) {
    const int W = (s->dim + 31) / 32;
    const int G = (int)ceil_div(s->capacity, s->group);
    const int groups = (int)ceil_div(tokens, s->group);
    dim3 grid(groups, s->kv_heads, s->batch);
    pack_kernel<T><<<grid, min(32 * W, kPackThreads), 0, st>>>(static_cast<const T*>(K), s->capacity, s->dim, W,
                                            s->group, G, tokens, s->kv_heads, bits,
                                            static_cast<__half2*>(params), nonfinite);
    return check_launch("fier_pack_keys");
}

template <typename T>
static int launch_append(const fier_shape* s, void* K, void* V, const void* k_new,
                         const void* v_new, int32_t pos, uint32_t* bits, void* params,
                         int32_t* nonfinite, int* zero_words, int zero_n, cudaStream_t st) {
    const int W = (s->dim + 31) / 32;
    const int G = (int)ceil_div(s->capacity, s->group);
    dim3 grid(1, s->kv_heads, s->batch);
    append_kernel<T><<<grid, min(32 * W, kPackThreads), 0, st>>>(static_cast<T*>(K), static_cast<T*>(V),
                                              static_cast<const T*>(k_new),
                                              static_cast<const T*>(v_new), pos, s->capacity,
                                              s->dim, W, s->group, G, s->kv_heads, bits,
                                              static_cast<__half2*>(params), nonfinite, zero_words,
                                              zero_n);
    return check_launch("fier_append");
}

int pack_dispatch(const fier_shape* s, const void* K, int32_t tokens, uint32_t* bits, void* params,
                  int32_t* nonfinite, cudaStream_t st) {
    switch (s->dtype) {
        case FIER_F32: return launch_pack<float>(s, K, tokens, bits, params, nonfinite, st);
        case FIER_F16: return launch_pack<__half>(s, K, tokens, bits, params, nonfinite, st);
        case FIER_BF16: return launch_pack<__nv_bfloat16>(s, K, tokens, bits, params, nonfinite, st);
        case FIER_F64: return launch_pack<double>(s, K, tokens, bits, params, nonfinite, st);
    }
    return fail(FIER_EINVAL, "fier_pack_keys: unknown dtype");
}

int append_dispatch(const fier_shape* s, void* K, void* V, const void* k_new, const void* v_new,
                    int32_t pos, uint32_t* bits, void* params, int32_t* nonfinite, int* zero_words,
                    int zero_n, cudaStream_t st) {
    switch (s->dtype) {
        case FIER_F32:
            return launch_append<float>(s, K, V, k_new, v_new, pos, bits, params, nonfinite, zero_words, zero_n, st);
        case FIER_F16:
            return launch_append<__half>(s, K, V, k_new, v_new, pos, bits, params, nonfinite, zero_words, zero_n, st);
        case FIER_BF16:
            return launch_append<__nv_bfloat16>(s, K, V, k_new, v_new, pos, bits, params,
                                                nonfinite, zero_words, zero_n, st);
        case FIER_F64:
            return launch_append<double>(s, K, V, k_new, v_new, pos, bits, params, nonfinite, zero_words, zero_n, st);
    }
    return fail(FIER_EINVAL, "fier_append: unknown dtype");
}

}  // namespace fier_cuda
