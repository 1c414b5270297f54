// capi.cu -- the C ABI (include/fier_cuda.h): argument validation with the
// reference's error texts, workspace sizing, the fused decode step, and the
// host-side FIER format conversion.
#include <cmath>
#include <cstring>
#include <string>

#include "common.cuh"

namespace fier_cuda {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(FIER_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return FIER_OK;
}

// kernels (pack.cu, score.cu, topk.cu, attention.cu)
int pack_dispatch(const fier_shape*, const void*, int32_t, uint32_t*, void*, int32_t*, cudaStream_t);
int append_dispatch(const fier_shape*, void*, void*, const void*, const void*, int32_t, uint32_t*,
                    void*, int32_t*, int*, int, cudaStream_t);
int score_dispatch(const fier_shape*, const void*, const uint32_t*, const void*, int, float*, int64_t,
                   cudaStream_t);
int topk_dispatch(const float*, int, int, int64_t, int, int32_t*, cudaStream_t);
int topk_dispatch_ws(const float*, int, int, int64_t, int, int32_t*, void*, size_t, cudaStream_t);
size_t topk_workspace(int, int, int);
size_t sparse_workspace(const fier_shape*, int);
size_t full_workspace(const fier_shape*, int);
int sparse_dispatch(const fier_shape*, const void*, const void*, const void*, const int32_t*, int, int,
                    float, float*, void*, bool, cudaStream_t, const int32_t*, float*);
int full_dispatch(const fier_shape*, const void*, const void*, const void*, int, float, float*, void*,
                  cudaStream_t);
size_t sparse_counter_offset(const fier_shape*, int);
int append_score_dispatch(const fier_shape*, const void*, void*, void*, const void*, const void*, int,
                          uint32_t*, void*, float*, int64_t, int*, int, int32_t*, cudaStream_t);
int fused_step_dispatch(const fier_shape*, const void*, const void*, const void*, int, void*, void*, uint32_t*,
                        void*, int, float, const fier_rope*, float*, int32_t*, float*, int64_t, int32_t*,
                        cudaStream_t);
int rope_dispatch(const fier_shape*, const void*, const void*, int, const fier_rope*, void*, void*, cudaStream_t);
bool fused_step_applies(const fier_shape*, int tokens);
bool attn_fused_merge(const fier_shape*);

static int check_shape(const fier_shape* s, const char* fn, bool allow_f64 = false) {
    const std::string f(fn);
    if (!s) return fail(FIER_EINVAL, f + ": null shape");
    if (s->batch < 1 || s->q_heads < 1 || s->kv_heads < 1 || s->capacity < 1)
        return fail(FIER_EINVAL, f + ": batch, heads and capacity must be >= 1");
    if (s->q_heads % s->kv_heads != 0)
        return fail(FIER_EINVAL, f + ": q_heads must be a multiple of kv_heads");
    if (s->dim < 1 || s->dim > 1024) return fail(FIER_EINVAL, f + ": head dim must be in [1, 1024]");
    if (s->group < 1) return fail(FIER_EINVAL, "quantize: group size must be >= 1");
    if (s->dtype == FIER_F64 && !allow_f64)
        return fail(FIER_EINVAL, f + ": FIER_F64 keys are accepted by fier_pack_keys / fier_append only");
    if (s->dtype != FIER_F32 && s->dtype != FIER_F16 && s->dtype != FIER_BF16 && s->dtype != FIER_F64)
        return fail(FIER_EINVAL, f + ": unknown dtype");
    return FIER_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static size_t elem_size(int dtype) { return dtype == FIER_F64 ? 8 : dtype == FIER_F32 ? 4 : 2; }

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace fier_cuda

using namespace fier_cuda;

extern "C" {

const char* fier_last_error(void) { return g_last_error.c_str(); }

int fier_version(void) { return 1; }

size_t fier_bits_bytes(const fier_shape* s) {
    if (check_shape(s, "fier_bits_bytes", true)) return 0;
    return (size_t)s->batch * s->kv_heads * s->capacity * ((s->dim + 31) / 32) * 4;
}

size_t fier_params_bytes(const fier_shape* s) {
    if (check_shape(s, "fier_params_bytes", true)) return 0;
    return (size_t)s->batch * s->kv_heads * ceil_div(s->capacity, s->group) * s->dim * 4;
}

size_t fier_payload_bytes(int32_t tokens, int32_t dim, int32_t group) {
    if (tokens < 1 || dim < 1 || group < 1) return 0;
    return (size_t)tokens * ((dim + 7) / 8) + (size_t)dim * ceil_div(tokens, group) * 4;
}

int fier_load_ratio_fier(int64_t tokens, int64_t group, int64_t* numerator_bits, int64_t* denominator_bits,
                         int32_t* formula) {
    FIER_REQUIRE(tokens >= 1 && group >= 1, "load_ratio_fier: l and g must be >= 1");
    FIER_REQUIRE(numerator_bits && denominator_bits && formula, "load_ratio_fier: null output");
    const int64_t groups = (tokens + group - 1) / group;
    *numerator_bits = tokens + groups * 2 * 16;
    *denominator_bits = tokens * 16;
    *formula = tokens % group == 0 ? 1 : 0;
    return FIER_OK;
}

int fier_pack_keys(const fier_shape* s, const void* K, int32_t tokens, uint32_t* bits, void* params,
                   int32_t* nonfinite, void* stream) {
    if (int rc = check_shape(s, "quantize", true)) return rc;
    FIER_REQUIRE(tokens >= 1, "quantize: empty key cache");
    FIER_REQUIRE(tokens <= s->capacity, "quantize: tokens exceed cache capacity");
    FIER_REQUIRE(K && bits && params, "quantize: null buffer");
    return pack_dispatch(s, K, tokens, bits, params, nonfinite, static_cast<cudaStream_t>(stream));
}

int fier_append(const fier_shape* s, void* K, void* V, const void* k_new, const void* v_new,
                int32_t pos, uint32_t* bits, void* params, int32_t* nonfinite, void* stream) {
    if (int rc = check_shape(s, "fier_append", true)) return rc;
    FIER_REQUIRE(pos >= 0 && pos < s->capacity, "fier_append: position outside cache capacity");
    FIER_REQUIRE(K && V && k_new && v_new && bits && params, "fier_append: null buffer");
    return append_dispatch(s, K, V, k_new, v_new, pos, bits, params, nonfinite, nullptr, 0,
                           static_cast<cudaStream_t>(stream));
}

int fier_score(const fier_shape* s, const void* q, const uint32_t* bits, const void* params,
               int32_t tokens, float* scores, int64_t ld, void* stream) {
    if (int rc = check_shape(s, "approx_scores")) return rc;
    FIER_REQUIRE(tokens >= 1 && tokens <= s->capacity, "approx_scores: tokens out of range");
    FIER_REQUIRE(ld >= tokens, "approx_scores: score row stride shorter than tokens");
    FIER_REQUIRE(q && bits && params && scores, "approx_scores: null buffer");
    FIER_REQUIRE(aligned16(bits) && aligned16(params), "approx_scores: index buffers must be 16-byte aligned");
    return score_dispatch(s, q, bits, params, tokens, scores, ld, static_cast<cudaStream_t>(stream));
}

size_t fier_topk_workspace(int32_t rows, int32_t tokens, int32_t k) { return topk_workspace(rows, tokens, k); }

int fier_topk(const float* scores, int32_t rows, int32_t tokens, int64_t ld, int32_t k, int32_t* sel,
              void* workspace, size_t workspace_bytes, void* stream) {
    FIER_REQUIRE(rows >= 1 && rows <= 65535, "topk_oracle: rows out of range");
    FIER_REQUIRE(k >= 1 && k <= tokens, "topk_oracle: k out of range");
    FIER_REQUIRE(ld >= tokens, "topk_oracle: score row stride shorter than tokens");
    FIER_REQUIRE(scores && sel, "topk_oracle: null buffer");
    return topk_dispatch_ws(scores, rows, tokens, ld, k, sel, workspace, workspace ? workspace_bytes : 0,
                            static_cast<cudaStream_t>(stream));
}

size_t fier_sparse_attention_workspace(const fier_shape* s, int32_t n) {
    if (check_shape(s, "gather_attention") || n < 1) return 0;
    return sparse_workspace(s, n);
}

int fier_sparse_attention(const fier_shape* s, const void* q, const void* K, const void* V,
                          const int32_t* sel, int32_t n, int32_t tokens, float scale, float* out,
                          void* workspace, size_t workspace_bytes, void* stream) {
    if (int rc = check_shape(s, "gather_attention")) return rc;
    FIER_REQUIRE(n >= 1, "gather_attention: empty selection");
    FIER_REQUIRE(n <= (1 << 19), "gather_attention: selection longer than 2^19 rows");
    FIER_REQUIRE(tokens >= 1 && tokens <= s->capacity && n <= tokens,
                 "gather_attention: selection invalid for cache");
    FIER_REQUIRE(q && K && V && sel && out, "gather_attention: null buffer");
    FIER_REQUIRE(aligned16(K) && aligned16(V), "gather_attention: K/V must be 16-byte aligned");
    FIER_REQUIRE(workspace && workspace_bytes >= sparse_workspace(s, n),
                 "gather_attention: workspace too small");
    return sparse_dispatch(s, q, K, V, sel, n, tokens, scale, out, workspace, false,
                           static_cast<cudaStream_t>(stream), nullptr, nullptr);
}

int fier_sparse_attention_ragged(const fier_shape* s, const void* q, const void* K, const void* V,
                                 const int32_t* sel, const int32_t* counts, int32_t n, int32_t tokens,
                                 float scale, float* out, float* lse, void* workspace,
                                 size_t workspace_bytes, void* stream) {
    if (int rc = check_shape(s, "gather_attention")) return rc;
    FIER_REQUIRE(n >= 1, "gather_attention: empty selection");
    FIER_REQUIRE(tokens >= 1 && tokens <= s->capacity, "gather_attention: selection invalid for cache");
    FIER_REQUIRE(q && K && V && sel && counts && out && lse, "gather_attention: null buffer");
    FIER_REQUIRE(aligned16(K) && aligned16(V), "gather_attention: K/V must be 16-byte aligned");
    FIER_REQUIRE(workspace && workspace_bytes >= sparse_workspace(s, n),
                 "gather_attention: workspace too small");
    return sparse_dispatch(s, q, K, V, sel, n, tokens, scale, out, workspace, false,
                           static_cast<cudaStream_t>(stream), counts, lse);
}

size_t fier_full_attention_workspace(const fier_shape* s, int32_t tokens) {
    if (check_shape(s, "gather_attention") || tokens < 1) return 0;
    return full_workspace(s, tokens);
}

int fier_full_attention(const fier_shape* s, const void* q, const void* K, const void* V,
                        int32_t tokens, float scale, float* out, void* workspace,
                        size_t workspace_bytes, void* stream) {
    if (int rc = check_shape(s, "gather_attention")) return rc;
    FIER_REQUIRE(tokens >= 1 && tokens <= s->capacity, "gather_attention: empty selection");
    FIER_REQUIRE(q && K && V && out, "gather_attention: null buffer");
    FIER_REQUIRE(aligned16(K) && aligned16(V), "gather_attention: K/V must be 16-byte aligned");
    FIER_REQUIRE(workspace && workspace_bytes >= full_workspace(s, tokens),
                 "gather_attention: workspace too small");
    return full_dispatch(s, q, K, V, tokens, scale, out, workspace, static_cast<cudaStream_t>(stream));
}

int64_t fier_step_scores_ld(int32_t tokens) { return ceil_div(tokens, 32) * 32; }

// workspace: [scores][attention partials + counters][top-k][q, k_new, v_new: rotated (RoPE) or
// staged from host memory (separate kernels)]
static size_t rope_bytes(const fier_shape* s) {
    return align_up((size_t)s->batch * (s->q_heads + 2 * s->kv_heads) * s->dim * elem_size(s->dtype));
}

// One launch copies the step's inputs out of (pinned, mapped) host memory, so the separate
// kernels' CTAs read them from HBM instead of each paying its own PCIe round trips.
__global__ void stage_inputs_kernel(const uint8_t* a, uint8_t* da, int64_t na, const uint8_t* b, uint8_t* db,
                                    int64_t nb, const uint8_t* c, uint8_t* dc, int64_t nc) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    auto copy = [&](const uint8_t* src, uint8_t* dst, int64_t n) {
        if ((((uintptr_t)src | (uintptr_t)dst | (uintptr_t)n) & 15) == 0) {
            for (int64_t i = tid; i < n / 16; i += nt)
                reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
        } else {
            for (int64_t i = tid; i < n; i += nt) dst[i] = src[i];
        }
    };
    copy(a, da, na);
    copy(b, db, nb);
    copy(c, dc, nc);
}

size_t fier_decode_workspace(const fier_shape* s, int32_t tokens, int32_t n) {
    if (check_shape(s, "fier_decode_step") || tokens < 1 || n < 1) return 0;
    const size_t scores = (size_t)s->batch * s->q_heads * fier_step_scores_ld(tokens) * sizeof(float);
    return align_up(scores) + align_up(sparse_workspace(s, n)) +
           align_up(topk_workspace(s->batch * s->q_heads, tokens, n)) + rope_bytes(s);
}

int fier_decode_step(const fier_shape* s, const void* q, const void* k_new, const void* v_new,
                     int32_t pos, void* K, void* V, uint32_t* bits, void* params, int32_t n,
                     float scale, float* out, int32_t* sel, float* scores_out, void* workspace,
                     size_t workspace_bytes, void* stream) {
    return fier_decode_step_ex(s, q, k_new, v_new, pos, K, V, bits, params, n, scale, nullptr, 0u, nullptr, out, sel,
                               scores_out, workspace, workspace_bytes, stream);
}

int fier_decode_step_ex(const fier_shape* s, const void* q, const void* k_new, const void* v_new,
                        int32_t pos, void* K, void* V, uint32_t* bits, void* params, int32_t n,
                        float scale, const fier_rope* rope, uint32_t flags, int32_t* nonfinite, float* out,
                        int32_t* sel, float* scores_out, void* workspace, size_t workspace_bytes, void* stream) {
    if (int rc = check_shape(s, "fier_decode_step")) return rc;
    const int32_t tokens = pos + 1;
    FIER_REQUIRE(pos >= 0 && pos < s->capacity, "fier_append: position outside cache capacity");
    FIER_REQUIRE(n >= 1 && n <= tokens, "fier_select: budget out of range");
    FIER_REQUIRE(q && k_new && v_new && K && V && bits && params && out && sel, "fier_decode_step: null buffer");
    FIER_REQUIRE(aligned16(K) && aligned16(V) && aligned16(bits) && aligned16(params),
                 "fier_decode_step: K, V and the index buffers must be 16-byte aligned");
    FIER_REQUIRE((int64_t)s->batch * s->q_heads <= 65535, "fier_decode_step: batch * q_heads exceeds 65535 rows");
    FIER_REQUIRE((flags & ~(uint32_t)(FIER_STEP_HOST_INPUTS | FIER_STEP_SEPARATE)) == 0,
                 "fier_decode_step: unknown flags");
    FIER_REQUIRE(workspace && workspace_bytes >= fier_decode_workspace(s, tokens, n),
                 "fier_decode_step: workspace too small");
    if (rope) {
        FIER_REQUIRE(rope->rotary_dim >= 2 && rope->rotary_dim % 2 == 0 && rope->rotary_dim <= s->dim &&
                         rope->rotary_dim <= 128,
                     "fier_decode_step: rotary_dim must be even, >= 2 and <= min(dim, 128)");
        FIER_REQUIRE(rope->base > 0.f && std::isfinite(rope->base), "fier_decode_step: rope base must be > 0");
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t ld = fier_step_scores_ld(tokens);
    // MHA, d = 128: the whole step (RoPE included) in one cluster launch (step_fused.cu)
    if (!(flags & FIER_STEP_SEPARATE)) {
        const int frc = fused_step_dispatch(s, q, k_new, v_new, pos, K, V, bits, params, n, scale, rope, out, sel,
                                            scores_out, ld, nonfinite, st);
        if (frc >= 0) return frc;
    }
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    float* scores = scores_out ? scores_out : reinterpret_cast<float*>(ws);
    uint8_t* attn_ws = ws + align_up((size_t)s->batch * s->q_heads * ld * sizeof(float));
    int* counters = reinterpret_cast<int*>(attn_ws + sparse_counter_offset(s, n));
    uint8_t* rws = attn_ws + align_up(sparse_workspace(s, n)) +
                   align_up(topk_workspace(s->batch * s->q_heads, tokens, n));
    const size_t qb = (size_t)s->batch * s->q_heads * s->dim * elem_size(s->dtype);
    const size_t kb = (size_t)s->batch * s->kv_heads * s->dim * elem_size(s->dtype);
    // (with RoPE the rope kernel already moves q / k_new out of host memory once)
    if (!rope && (flags & FIER_STEP_HOST_INPUTS)) {
        const int64_t words = (int64_t)(qb + 2 * kb) / 16;
        const int blocks = (int)std::min<int64_t>(num_sms(), std::max<int64_t>(1, ceil_div(words, 256)));
        stage_inputs_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint8_t*>(q), rws, (int64_t)qb,
                                                    static_cast<const uint8_t*>(k_new), rws + qb, (int64_t)kb,
                                                    static_cast<const uint8_t*>(v_new), rws + qb + kb, (int64_t)kb);
        if (int rc = check_launch("fier_decode_step (staging)")) return rc;
        q = rws;
        k_new = rws + qb;
        v_new = rws + qb + kb;
    }
    if (rope) {  // rotated copies of q and k_new for the separate kernels
        void* q_rot = rws;
        void* k_rot = rws + qb;
        if (int rc = rope_dispatch(s, q, k_new, pos, rope, q_rot, k_rot, st)) return rc;
        q = q_rot;
        k_new = k_rot;
    }
    int rc = append_score_dispatch(s, q, K, V, k_new, v_new, pos, bits, params, scores, ld, counters,
                                   s->batch * s->q_heads, nonfinite, st);
    if (rc) return rc;
    uint8_t* tws = attn_ws + align_up(sparse_workspace(s, n));
    rc = topk_dispatch_ws(scores, s->batch * s->q_heads, tokens, ld, n, sel, tws,
                          topk_workspace(s->batch * s->q_heads, tokens, n), st);
    if (rc) return rc;
    return sparse_dispatch(s, q, K, V, sel, n, tokens, scale, out, attn_ws, true, st, nullptr, nullptr);
}

int32_t fier_decode_step_launches(const fier_shape* s, int32_t tokens, int32_t n, uint32_t flags,
                                  int32_t with_rope) {
    if (check_shape(s, "fier_decode_step") || tokens < 1 || n < 1 || n > tokens) return 0;
    if (!(flags & FIER_STEP_SEPARATE) && fused_step_applies(s, tokens)) return 1;
    // append+score, Top-k, sparse attention (+ a separate LSE merge on the generic attention path)
    int launches = attn_fused_merge(s) ? 3 : 4;
    if (with_rope) return launches + 1;  // the RoPE kernel (it also reads host-resident inputs once)
    return launches + ((flags & FIER_STEP_HOST_INPUTS) ? 1 : 0);  // staging of host-resident inputs
}

// ---- host-side FIER conversion (io.hpp:197-277) ------------------------------------

int fier_index_to_fier(const uint32_t* bits, const uint16_t* params, int32_t tokens, int32_t dim,
                       int32_t group, uint8_t* out, size_t out_bytes) {
    FIER_REQUIRE(tokens >= 1 && dim >= 1 && group >= 1, "serialize_packed_keys: invalid dims");
    const size_t need = 18 + fier_payload_bytes(tokens, dim, group);
    FIER_REQUIRE(out && out_bytes >= need, "serialize_packed_keys: output buffer too small");
    const int W = (dim + 31) / 32;
    const int64_t G = ceil_div(tokens, group);
    uint8_t* p = out;
    std::memcpy(p, "FIER", 4);
    p += 4;
    *p++ = 1;
    *p++ = 0;
    const uint32_t hdr[3] = {(uint32_t)tokens, (uint32_t)dim, (uint32_t)group};
    for (uint32_t v : hdr)
        for (int i = 0; i < 4; ++i) *p++ = (uint8_t)((v >> (8 * i)) & 0xFF);
    for (int j = 0; j < dim; ++j) {
        for (int64_t gi = 0; gi < G; ++gi) {
            const uint16_t s = params[(gi * dim + j) * 2], z = params[(gi * dim + j) * 2 + 1];
            *p++ = s & 0xFF;
            *p++ = s >> 8;
            *p++ = z & 0xFF;
            *p++ = z >> 8;
        }
    }
    const int row_bytes = (dim + 7) / 8;
    for (int64_t t = 0; t < tokens; ++t) {
        for (int bb = 0; bb < row_bytes; ++bb) {
            uint8_t byte = 0;
            for (int bit = 0; bit < 8; ++bit) {
                const int j = bb * 8 + bit;
                if (j < dim && ((bits[t * W + j / 32] >> (j % 32)) & 1u)) byte |= (uint8_t)(1u << bit);
            }
            *p++ = byte;
        }
    }
    return FIER_OK;
}

static uint32_t rd_u32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

int fier_fier_to_index(const uint8_t* buf, size_t len, int32_t* tokens, int32_t* dim, int32_t* group,
                       uint32_t* bits, size_t bits_cap, uint16_t* params, size_t params_cap) {
    // Diagnostics follow parse_packed_keys / ByteReader (io.hpp:110-134, 227-277).
    if (len < 4) return fail(FIER_EDATA, "truncated file while reading magic");
    if (std::memcmp(buf, "FIER", 4) != 0) return fail(FIER_EDATA, "bad magic: expected FIER");
    if (len < 6) return fail(FIER_EDATA, "truncated file while reading version");
    const uint16_t version = (uint16_t)(buf[4] | (buf[5] << 8));
    if (version != 1) return fail(FIER_EDATA, "unsupported version: " + std::to_string(version));
    if (len < 10) return fail(FIER_EDATA, "truncated file while reading l");
    if (len < 14) return fail(FIER_EDATA, "truncated file while reading d");
    if (len < 18) return fail(FIER_EDATA, "truncated file while reading g");
    const uint32_t l = rd_u32(buf + 6), d = rd_u32(buf + 10), g = rd_u32(buf + 14);
    if (l == 0) return fail(FIER_EDATA, "invalid l: must be >= 1");
    if (d == 0) return fail(FIER_EDATA, "invalid d: must be >= 1");
    if (g == 0) return fail(FIER_EDATA, "invalid g: must be >= 1");
    if (l > 0x7FFFFFFFu || d > 1024u || g > 0x7FFFFFFFu)
        return fail(FIER_EDATA, "index dimensions exceed the device layout");
    const size_t expect = fier_payload_bytes((int32_t)l, (int32_t)d, (int32_t)g);
    if (len - 18 != expect)
        return fail(FIER_EDATA, "payload length mismatch: header declares " + std::to_string(expect) +
                                    " bytes, found " + std::to_string(len - 18));
    *tokens = (int32_t)l;
    *dim = (int32_t)d;
    *group = (int32_t)g;
    const int W = ((int)d + 31) / 32;
    const int64_t G = ceil_div(l, g);
    if (!bits || !params) return FIER_OK;  // size query
    if (bits_cap < (size_t)l * W || params_cap < (size_t)G * d * 2)
        return fail(FIER_EINVAL, "parse_packed_keys: output buffers too small");
    const uint8_t* p = buf + 18;
    for (uint32_t j = 0; j < d; ++j) {
        for (int64_t gi = 0; gi < G; ++gi) {
            params[(gi * d + j) * 2] = (uint16_t)(p[0] | (p[1] << 8));
            params[(gi * d + j) * 2 + 1] = (uint16_t)(p[2] | (p[3] << 8));
            p += 4;
        }
    }
    std::memset(bits, 0, (size_t)l * W * 4);
    const int row_bytes = ((int)d + 7) / 8;
    for (uint32_t t = 0; t < l; ++t) {
        for (int bb = 0; bb < row_bytes; ++bb) {
            const uint8_t byte = p[bb];
            for (int bit = 0; bit < 8; ++bit) {
                const uint32_t j = (uint32_t)(bb * 8 + bit);
                if (j < d && (byte & (1u << bit))) bits[(size_t)t * W + j / 32] |= 1u << (j % 32);
            }
        }
        p += row_bytes;
    }
    return FIER_OK;
}

}  // extern "C"
