/*
 * fier_cuda.h -- C ABI of the B200 (sm_100a) Fier decode-time KV retrieval path.
 *
 * This is the drop-in boundary for the reference's hot path (arxiv 2508.08256,
 * reference at proj/include/fier/).  Every entry point below replaces one
 * reference function; the citation names the reference interface.  A C++
 * shim with the reference's own signatures (fier::cuda::quantize,
 * approx_scores, topk_oracle, gather_attention, fier_select, fier_attend)
 * lives in fier_cuda.hpp; see INTEGRATION.md for ctypes / C++ bindings.
 *
 * Conventions
 *  - Plain C: device pointers, sizes and a cudaStream_t passed as void*.
 *  - Nothing allocates: the caller owns every buffer and workspace
 *    (size-query functions below).  Calls are stream-ordered, never block,
 *    and are CUDA-graph capturable.
 *  - Return 0 on success, else FIER_EINVAL (1, the reference's
 *    std::invalid_argument from require(), core.hpp:19-21), FIER_EDATA (2,
 *    fier::DataError, io.hpp:29-31) or FIER_ECUDA (3).  fier_last_error()
 *    returns the thread's last message, using the reference's message text.
 *  - Data races: concurrent calls need distinct output/workspace buffers.
 *
 * Device layouts (one "layer" of a batch of B sequences):
 *   K, V   : dtype [B][Hkv][cap][d]           token rows contiguous
 *   bits   : uint32 [B][Hkv][cap][W], W=ceil(d/32); bit i of word w is channel
 *            32w+i, 1 <=> code +1.  Byte-identical to the reference's in-memory
 *            code_words (quant1bit.hpp:38-49) and FIER bit plane when 32 | d.
 *   params : half2 [B][Hkv][ceil(cap/g)][d] = (s, z) as IEEE binary16
 *            (the on-disk precision of io.hpp:205-211), group-major like the
 *            in-memory scales/zeros [gi*d + j] (quant1bit.hpp:39-42).
 *   q      : dtype [B][Hq][d];  scores : float [B][Hq][ld];  sel : int32 [B][Hq][n]
 *            ascending (core.hpp:146);  out : float [B][Hq][d].
 *   GQA    : q head h reads kv head h / (Hq/Hkv); selection is per q head.
 */
#ifndef FIER_CUDA_H_
#define FIER_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FIER_API __attribute__((visibility("default")))
#else
#define FIER_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum fier_status { FIER_OK = 0, FIER_EINVAL = 1, FIER_EDATA = 2, FIER_ECUDA = 3 };
/* FIER_F64: the reference's own key type (KeyCache is an fp64 Matrix, core.hpp:24-68);
 * accepted by fier_pack_keys, fier_append (bit-exact quantize of fp64 keys) and
 * fier_exact_scores (the C++ drop-in's oracle / full policies) only. */
enum fier_dtype { FIER_F32 = 0, FIER_F16 = 1, FIER_BF16 = 2, FIER_F64 = 3 };

/* Shape of one layer's cache.  All fields are plain integers. */
typedef struct fier_shape {
    int32_t batch;     /* B sequences                               */
    int32_t q_heads;   /* Hq (multiple of kv_heads)                 */
    int32_t kv_heads;  /* Hkv                                       */
    int32_t capacity;  /* allocated tokens per sequence (cap)       */
    int32_t dim;       /* head dim d (1..1024)                      */
    int32_t group;     /* g, tokens per quantization group (>= 1)   */
    int32_t dtype;     /* enum fier_dtype of K, V, q                */
} fier_shape;

/* ---- errors / sizes --------------------------------------------------------- */
FIER_API const char* fier_last_error(void);
FIER_API int fier_version(void);
/* Bytes of the bit plane / the (s,z) table for the whole layer. */
FIER_API size_t fier_bits_bytes(const fier_shape* s);
FIER_API size_t fier_params_bytes(const fier_shape* s);
/* Exact accounted payload of one (sequence, kv head) index at `tokens`
 * (PackedKeys::payload_bytes, quant1bit.hpp:60-62). */
FIER_API size_t fier_payload_bytes(int32_t tokens, int32_t dim, int32_t group);
/* load_ratio_fier (quant1bit.hpp:176-184): exact estimation cost per channel against a
 * 16-bit key cache, l code bits + ceil(l/g) * 2 * 16 parameter bits over l * 16 bits,
 * as the unreduced bit counts of LoadRatio (numerator_bits, denominator_bits) and
 * formula = (g divides l).  Reduce with gcd for LoadRatio::ratio().  Host-only. */
FIER_API int fier_load_ratio_fier(int64_t tokens, int64_t group, int64_t* numerator_bits,
                                  int64_t* denominator_bits, int32_t* formula);

/* ---- K1: 1-bit key packer ---------------------------------------------------- */
/* quantize (quant1bit.hpp:65-103) of tokens [0, tokens) of every (b, kv head).
 * Bits compare against the fp64 midpoint; (s, z) stored RNE to binary16
 * (half.hpp:30-61).  *nonfinite (device int, may be NULL) is set to 1 if any
 * key is not finite ("quantize: non-finite key entry", quant1bit.hpp:68). */
FIER_API int fier_pack_keys(const fier_shape* s, const void* K, int32_t tokens, uint32_t* bits,
                   void* params, int32_t* nonfinite, void* stream);

/* Decode-time append: write k_new/v_new ([B][Hkv][d]) as token `pos` of K/V
 * and re-pack the open group [floor(pos/g)*g, pos] so the index equals
 * quantize(K[0:pos+1]) bit for bit (quant1bit.hpp:84 short final group). */
FIER_API int fier_append(const fier_shape* s, void* K, void* V, const void* k_new, const void* v_new,
                int32_t pos, uint32_t* bits, void* params, int32_t* nonfinite, void* stream);

/* ---- K2: packed-key scorer --------------------------------------------------- */
/* approx_scores (quant1bit.hpp:121-140) for all (b, q head): scores[b][h][t],
 * t < tokens, row stride ld >= tokens.  fp32 accumulation. */
FIER_API int fier_score(const fier_shape* s, const void* q, const uint32_t* bits, const void* params,
               int32_t tokens, float* scores, int64_t ld, void* stream);

/* ---- K3: Top-k selector -------------------------------------------------------- */
/* topk_oracle (core.hpp:134-148) on `rows` rows of `tokens` fp32 scores
 * (row stride ld): the k largest, ties to the lower index, ascending output
 * in sel[row][0..k).  Requires 1 <= k <= tokens ("topk_oracle: k out of range").
 * With a device workspace of fier_topk_workspace() bytes (0 = none needed), launches
 * holding millions of keys take the wide-grid radix select (histogram pass, collect pass,
 * per-row resolve + sort: 3 kernels and a memset); without one (NULL, 0), the per-row
 * cluster select.  Both return identical selections. */
FIER_API size_t fier_topk_workspace(int32_t rows, int32_t tokens, int32_t k);
FIER_API int fier_topk(const float* scores, int32_t rows, int32_t tokens, int64_t ld, int32_t k,
              int32_t* sel, void* workspace, size_t workspace_bytes, void* stream);

/* topk_oracle on fp64 scores (the reference's own ScoreVector type, core.hpp:75-79):
 * exact on doubles that would tie after rounding to fp32.  One CTA per row, an exact
 * radix select on order-preserving u64 keys; not a decode-path kernel (the C++
 * drop-in's fp64 inputs).  Same tie rule and ascending output as fier_topk. */
FIER_API int fier_topk_f64(const double* scores, int32_t rows, int32_t tokens, int64_t ld, int32_t k,
                           int32_t* sel, void* stream);

/* ---- K4: sparse attention over the selected rows ------------------------------ */
/* gather_attention (core.hpp:152-179): out[b][h] = softmax(scale * q K[sel]^T) V[sel]
 * over the n ascending indices sel[b][h][0..n) (< tokens).  Partial softmaxes
 * of KV splits are merged by log-sum-exp.  scale = 1/sqrt(d) reproduces the
 * reference default (scaled=true, core.hpp:154). */
FIER_API size_t fier_sparse_attention_workspace(const fier_shape* s, int32_t n);
FIER_API int fier_sparse_attention(const fier_shape* s, const void* q, const void* K, const void* V,
                          const int32_t* sel, int32_t n, int32_t tokens, float scale, float* out,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Ragged variant for the sequence-sharded step: row (b, h) attends over the
 * first min(n, counts[b][h]) indices of sel[b][h][0..n) (row stride n).  Also
 * writes lse[b][h] = log2 sum_i exp2(scale*log2(e)*q.k_i) (the log-sum-exp of
 * this shard's logits in the log2 domain; -inf and out = 0 for an empty row),
 * the weight fier_lse_merge needs. */
FIER_API int fier_sparse_attention_ragged(const fier_shape* s, const void* q, const void* K, const void* V,
                                 const int32_t* sel, const int32_t* counts, int32_t n, int32_t tokens,
                                 float scale, float* out, float* lse, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ---- K0: full-KV decode attention (the in-house baseline) --------------------- */
/* gather_attention over all indices (the `full` policy, retrieval.hpp:159-166). */
FIER_API size_t fier_full_attention_workspace(const fier_shape* s, int32_t tokens);
FIER_API int fier_full_attention(const fier_shape* s, const void* q, const void* K, const void* V,
                        int32_t tokens, float scale, float* out, void* workspace,
                        size_t workspace_bytes, void* stream);

/* ---- fused decode step --------------------------------------------------------- */
/* fier_attend (retrieval.hpp:136-146) for a decode step of every (b, q head):
 * append(pos) -> score -> Top-n -> sparse attention, over tokens = pos + 1.
 * scores_out (may be NULL) receives the estimated logits (ld = tokens rounded
 * up to 32, see fier_step_scores_ld).  MHA layers with d = 128, 32 | g, 16-bit
 * caches and tokens <= 131072 run as ONE cluster kernel (step_fused.cu);
 * other shapes as append+score, Top-k and sparse-attention launches. */
FIER_API size_t fier_decode_workspace(const fier_shape* s, int32_t tokens, int32_t n);
FIER_API int64_t fier_step_scores_ld(int32_t tokens);
/* Kernel launches fier_decode_step_ex issues for this shape and flags (1 = the fused
 * kernel; the separate-kernel path adds one launch for FIER_STEP_HOST_INPUTS staging and
 * one for RoPE when with_rope != 0).  fier_decode_step = flags 0, no rope. */
FIER_API int32_t fier_decode_step_launches(const fier_shape* s, int32_t tokens, int32_t n, uint32_t flags,
                                           int32_t with_rope);

/* Rotary position embedding fused into the step (the KV write +
 * RoPE + append-pack that precedes scoring in a decode loop).  q (every q head) and
 * k_new (every kv head) are rotated by position pos before use: frequency i < rd/2
 * turns by pos * base^(-2i/rd) (angles evaluated in double on the host), channels
 * >= rd pass through.  interleaved = 0: pairs (i, i + rd/2) ("rotate_half", NeoX /
 * Llama); 1: pairs (2i, 2i + 1) (GPT-J).  v_new is not rotated.  The rotation is
 * evaluated in fp32 and rounded to the cache dtype; the rotated k row is what the
 * cache stores and the index packs. */
typedef struct fier_rope {
    float base;          /* e.g. 10000 */
    int32_t rotary_dim;  /* rd: even, 2 <= rd <= min(dim, 128) */
    int32_t interleaved;
} fier_rope;
/* Flags of fier_decode_step_ex.
 *  FIER_STEP_HOST_INPUTS: q / k_new / v_new live in pinned, mapped HOST memory.  The
 *  separate-kernel path then stages them into the workspace with one launch first (one
 *  PCIe round trip instead of one per CTA); the one-launch path reads them directly.
 *  The caller states residency once (no per-step pointer queries, and the choice is
 *  what a captured graph replays).
 *  FIER_STEP_SEPARATE: run the separate-kernel path even where the one-launch cluster
 *  kernel applies (same results; for A/B comparisons and tests). */
enum fier_step_flags { FIER_STEP_HOST_INPUTS = 1, FIER_STEP_SEPARATE = 2 };
/* Non-finite inputs of a step, OR-ed into *nonfinite (a device int the caller zeroes):
 *  FIER_NONFINITE_KEY   -- the appended key row (after RoPE) or its open group holds a
 *                          non-finite entry: "quantize: non-finite key entry" (quant1bit.hpp:68)
 *  FIER_NONFINITE_QUERY -- the query does: its logits cannot be finite,
 *                          "softmax: non-finite logit" (core.hpp:122). */
enum fier_nonfinite { FIER_NONFINITE_KEY = 1, FIER_NONFINITE_QUERY = 2 };
/* fier_decode_step with an optional rope (NULL: none), flags (fier_step_flags) and an
 * optional device status word nonfinite (NULL: not checked); same workspace. */
FIER_API int fier_decode_step_ex(const fier_shape* s, const void* q, const void* k_new, const void* v_new,
                        int32_t pos, void* K, void* V, uint32_t* bits, void* params, int32_t n,
                        float scale, const fier_rope* rope, uint32_t flags, int32_t* nonfinite, float* out,
                        int32_t* sel, float* scores_out, void* workspace, size_t workspace_bytes, void* stream);
FIER_API int fier_decode_step(const fier_shape* s, const void* q, const void* k_new, const void* v_new,
                     int32_t pos, void* K, void* V, uint32_t* bits, void* params, int32_t n,
                     float scale, float* out, int32_t* sel, float* scores_out, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ---- X1: sequence-sharded step -------------------------------- */
/* The whole-group token range [start, end) of shard `rank` of `shards` over a
 * context of `tokens` (boundaries multiples of g: each shard's index equals the
 * matching slice of quantize(), quant1bit.hpp:5-9).  Host-only. */
FIER_API int fier_shard_bounds(int64_t tokens, int32_t shards, int32_t group, int32_t rank, int64_t* start,
                      int64_t* end);
/* Candidate list of one shard: (scores[row][sel[row][i]], start + sel[row][i])
 * for i < k, padded to nc entries with (-inf, -1).  sel = the shard's local
 * Top-k (ascending), k = min(n, local tokens). */
FIER_API int fier_shard_candidates(const float* scores, int32_t rows, int64_t ld, const int32_t* sel, int32_t k,
                          int32_t nc, int32_t start, float* cand_scores, int32_t* cand_idx, void* stream);
/* Global Top-n (topk_oracle tie rule) from the all-gathered candidate lists
 * cand_*[shards][rows][nc]: sel_global[rows][n] (ascending global indices),
 * and this rank's run as local indices sel_local[rows][0..counts[row]) (each
 * output may be NULL). */
FIER_API size_t fier_shard_merge_workspace(int32_t shards, int32_t rows, int32_t nc, int32_t n);
FIER_API int fier_shard_merge(const float* cand_scores, const int32_t* cand_idx, int32_t shards, int32_t rows,
                     int32_t nc, int32_t n, int32_t rank, int32_t start, int32_t* sel_global,
                     int32_t* sel_local, int32_t* counts, void* workspace, size_t workspace_bytes,
                     void* stream);
/* Log-sum-exp merge of per-shard partials outs[shards][rows][dim], lses[shards][rows]
 * (from fier_sparse_attention_ragged) into out[rows][dim] (and lse[rows], may be NULL). */
FIER_API int fier_lse_merge(const float* outs, const float* lses, int32_t shards, int32_t rows, int32_t dim,
                   float* out, float* lse, void* stream);

/* ---- host-side format conversion (no GPU) -------------------------------------- */
/* serialize_packed_keys (io.hpp:197-225) of one (b, kv head) index copied to
 * host: bits [tokens][W] uint32, params [ceil(tokens/g)][d] (s, z) binary16
 * pairs.  out must hold 18 + fier_payload_bytes(tokens, d, g) bytes. */
FIER_API int fier_index_to_fier(const uint32_t* bits, const uint16_t* params, int32_t tokens, int32_t dim,
                       int32_t group, uint8_t* out, size_t out_bytes);
/* parse_packed_keys (io.hpp:227-277) into the device layout (host buffers).
 * Returns FIER_EDATA with the reference's diagnostics on malformed input. */
FIER_API int fier_fier_to_index(const uint8_t* buf, size_t len, int32_t* tokens, int32_t* dim,
                       int32_t* group, uint32_t* bits, size_t bits_cap, uint16_t* params,
                       size_t params_cap);

/* ---- device-side FIER / KVD1 byte streams --------------------- */
/* serialize_packed_keys (io.hpp:197-225) of one (sequence, kv head) index, written by
 * kernels into the DEVICE buffer out (18 + fier_payload_bytes(tokens, d, g) bytes):
 * bits = that head's [>= tokens][ceil(d/32)] words, params = its [ceil(tokens/g)][d]
 * (s, z) binary16 pairs.  Byte-identical to fier_index_to_fier. */
FIER_API int fier_index_export(const uint32_t* bits, const void* params, int32_t tokens, int32_t dim,
                      int32_t group, uint8_t* out, size_t out_bytes, void* stream);
/* parse_packed_keys (io.hpp:227-277) of a FIER stream in DEVICE memory into a device
 * index (bits_words >= l * ceil(d/32), param_pairs >= ceil(l/g) * d).  The 18-byte
 * header is read back (stream-synchronous) and checked with the reference's
 * diagnostics (FIER_EDATA); NULL bits/params = size query. */
FIER_API int fier_index_import(const uint8_t* in, size_t in_bytes, int32_t* tokens, int32_t* dim, int32_t* group,
                      uint32_t* bits, int64_t bits_words, void* params, int64_t param_pairs, void* stream);
/* parse_cache_dump (io.hpp:140-185) of a KVD1 stream in DEVICE memory into fp32 device
 * values [K (l x d) | V (l x d) | queries (nq x d)] (exact for both payload dtypes);
 * dtype = 0 (f16) or 1 (f32).  NULL values = size query. */
FIER_API int fier_kvd1_load(const uint8_t* in, size_t in_bytes, int32_t* tokens, int32_t* dim, int32_t* queries,
                   int32_t* dtype, float* values, int64_t values_cap, void* stream);
/* serialize_cache_dump (io.hpp:110-137) of device fp32 values laid out as above into the
 * DEVICE buffer out (20 + (2l + nq) * d * (dtype ? 4 : 2) bytes); f16 rounds to nearest even. */
FIER_API int fier_kvd1_store(const float* values, int32_t tokens, int32_t dim, int32_t queries, int32_t dtype,
                    uint8_t* out, size_t out_bytes, void* stream);

/* ---- Quest page retrieval (baselines.hpp) ------------------------ */
/* build_page_summaries (baselines.hpp:34-56): K [B][Hkv][capacity][d] (s->dtype) ->
 * kmax, kmin [B][Hkv][ceil(tokens/L)][d] fp32 (exact channel-wise extrema). */
FIER_API int fier_quest_summaries(const fier_shape* s, const void* K, int32_t tokens, int32_t page_size,
                         float* kmax, float* kmin, void* stream);
/* quest_page_scores (baselines.hpp:60-79) for q [B][Hq][d] (q head h reads kv head
 * h / (Hq/Hkv)): page_scores[B*Hq][pld], variant 1 = sum over channels, 0 = max;
 * evaluated in fp64, stored fp32. */
FIER_API int fier_quest_page_scores(const fier_shape* s, const void* q, const float* kmax, const float* kmin,
                           int32_t tokens, int32_t page_size, int32_t variant, float* page_scores,
                           int64_t pld, void* stream);
/* quest_select_quantized's page scores (baselines.hpp:131-139): the mean of each page's
 * approx_scores (K2 output scores[rows][ld]) -> page_scores[rows][pld]. */
FIER_API int fier_page_mean(const float* scores, int32_t rows, int32_t tokens, int64_t ld, int32_t page_size,
                   float* page_scores, int64_t pld, void* stream);
/* detail::select_by_page_scores (baselines.hpp:85-111): rank pages by (score desc, index
 * asc), take whole pages while they fit, then the next page's lowest indices:
 * sel[rows][n] ascending.  Workspace from fier_page_select_workspace (required). */
FIER_API size_t fier_page_select_workspace(int32_t rows, int32_t tokens, int32_t page_size, int32_t n);
FIER_API int fier_page_select(const float* page_scores, int32_t rows, int32_t tokens, int64_t pld, int32_t page_size,
                     int32_t n, int32_t* sel, void* workspace, size_t workspace_bytes, void* stream);

/* ---- recall / margin sweep diagnostics (evalharness.hpp) --------- */
/* exact_scores (core.hpp:98-112): scores[B*Hq][ld] = q . k_i in fp64 (scaled: / sqrt(d)),
 * GQA as above; scores32 (may be NULL) receives the same rounded to fp32.  FIER_F64
 * q and K (the reference's own types) are summed in the reference's channel order with
 * unfused products: bit-identical to exact_scores. */
FIER_API int fier_exact_scores(const fier_shape* s, const void* q, const void* K, int32_t tokens, int32_t scaled,
                      double* scores, float* scores32, int64_t ld, void* stream);
/* margin_and_errors (evalharness.hpp:63-83) per row: report[rows][5] = (margin, max_err,
 * l2_loss, hinge_loss, hinge_loss_symmetric) of err = exact - est; the order statistics
 * come from K3 on exact32 (exact unless fp32 rounding ties the boundary scores). */
FIER_API size_t fier_margin_errors_workspace(int32_t rows, int32_t k);
FIER_API int fier_margin_errors(const double* exact, const float* exact32, const float* est, int32_t rows,
                       int32_t tokens, int64_t ld, int32_t k, double* report, void* workspace,
                       size_t workspace_bytes, void* stream);
/* overlap_fraction (evalharness.hpp:40-48) per row of ascending lists: out[rows]. */
FIER_API int fier_overlap(const int32_t* sel, int32_t n, const int32_t* oracle, int32_t no, int32_t rows, double* out,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FIER_CUDA_H_ */
