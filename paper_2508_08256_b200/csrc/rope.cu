// rope.cu -- RoPE for the separate-kernel decode step: rotate q (every q head) and
// k_new (every kv head) by the step's position into workspace copies that the
// append/score/attention launches then read.  The fused step (step_fused.cu) applies
// the same rotation in-kernel.  See rope.cuh for the convention.
#include "rope.cuh"

namespace fier_cuda {

// block b < nq: q head b; else kv head b - nq.  Thread c = channel c.
template <typename T>
__global__ void rope_kernel(const T* __restrict__ q, const T* __restrict__ k_new, int nq, int d, RopeTable t,
                            T* __restrict__ q_out, T* __restrict__ k_out) {
    const int b = blockIdx.x;
    const T* src = b < nq ? q + (int64_t)b * d : k_new + (int64_t)(b - nq) * d;
    T* dst = b < nq ? q_out + (int64_t)b * d : k_out + (int64_t)(b - nq) * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x)
        dst[c] = T(rope_channel(t, c, [&](int j) { return to_f32(src[j]); }));
}

int rope_dispatch(const fier_shape* s, const void* q, const void* k_new, int pos, const fier_rope* rope, void* q_out,
                  void* k_out, cudaStream_t st) {
    const RopeTable t = rope_table(rope, pos);
    const int nq = s->batch * s->q_heads, nk = s->batch * s->kv_heads;
    const int threads = s->dim < 128 ? ((s->dim + 31) / 32) * 32 : 128;
    switch (s->dtype) {
        case FIER_F32:
            rope_kernel<float><<<nq + nk, threads, 0, st>>>(static_cast<const float*>(q), static_cast<const float*>(k_new),
                                                            nq, s->dim, t, static_cast<float*>(q_out),
                                                            static_cast<float*>(k_out));
            break;
        case FIER_F16:
            rope_kernel<__half><<<nq + nk, threads, 0, st>>>(static_cast<const __half*>(q),
                                                             static_cast<const __half*>(k_new), nq, s->dim, t,
                                                             static_cast<__half*>(q_out), static_cast<__half*>(k_out));
            break;
        default:
            rope_kernel<__nv_bfloat16><<<nq + nk, threads, 0, st>>>(
                static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k_new), nq, s->dim, t,
                static_cast<__nv_bfloat16*>(q_out), static_cast<__nv_bfloat16*>(k_out));
    }
    return check_launch("fier_decode_step (rope)");
}

}  // namespace fier_cuda
