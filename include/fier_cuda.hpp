// fier_cuda.hpp -- header-only C++ drop-in for the reference's Fier entry points,
// running on the sm_100a kernels behind the C ABI (fier_cuda.h).
//
// Same names, argument meaning and error behaviour as the reference
// (proj/include/fier/): precondition failures throw std::invalid_argument with the
// reference's message (require(), core.hpp:19-21), malformed FIER bytes throw
// fier::cuda::DataError (io.hpp:29-31), CUDA failures throw std::runtime_error.
//
//   fier::cuda::quantize(K, GroupSpec)          quantize          quant1bit.hpp:65-103
//   fier::cuda::approx_scores(q, pk)            approx_scores     quant1bit.hpp:121-140
//   fier::cuda::topk_oracle(scores, k)          topk_oracle       core.hpp:134-148
//   fier::cuda::gather_attention(q, K, V, sel)  gather_attention  core.hpp:152-179
//   fier::cuda::fier_select(q, pk, n)           fier_select       retrieval.hpp:130-133
//   fier::cuda::fier_attend(q, K, V, pk, n)     fier_attend       retrieval.hpp:136-146
//   fier::cuda::build_page_summaries(K, L)      build_page_summaries baselines.hpp:34-56
//   fier::cuda::quest_select(q, K, ps, n, v)    quest_select      baselines.hpp:113-118
//   fier::cuda::quest_select_quantized(q, pk, L, n) quest_select_quantized baselines.hpp:120-140
//   fier::cuda::exact_scores(q, K, scaled)      exact_scores      core.hpp:98-112
//   fier::cuda::select_for_policy(p, q, K, st)  select_for_policy retrieval.hpp:155-221
//   fier::cuda::run_policy(p, q, K, V, st)      run_policy        retrieval.hpp:223-233
//   fier::cuda::load_ratio_fier(l, g)           load_ratio_fier   quant1bit.hpp:176-184
//
// The functions are templates over the cache / index / result types and only use
// the reference's member names (K.tokens(), K.dim(), K.data.data(), pk.code_words,
// pk.scales, ...).  Standalone they default to the mirror types in
// fier::cuda::types; next to the reference headers a caller names the reference's
// own types, e.g. `fier::cuda::quantize<fier::PackedKeys>(K, fier::GroupSpec{32})`.
//
// Precision: quantize packs the fp64 keys themselves on the device (FIER_F64: fp64
// min/max/midpoint, bits against the unrounded fp64 z) and keeps (s, z) as binary16,
// the on-disk precision of the FIER format (io.hpp:205-211); the returned PackedKeys
// holds those half-rounded values, so serialize_packed_keys() of it is byte-identical
// to serialize_packed_keys(quantize(K)) of the reference for any fp64 K.  topk_oracle
// and exact_scores run in fp64 (bit-identical selections / scores).  approx_scores and
// gather_attention compute in fp32 on fp32 copies of q, K, V (the decode path's
// arithmetic): within 1e-3 / 1e-2 of the reference (BASELINE.json north star).
#ifndef FIER_CUDA_HPP_
#define FIER_CUDA_HPP_

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "fier_cuda.h"

namespace fier {
namespace cuda {

struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace types {  // mirrors of the reference's value types (core.hpp:24-94, quant1bit.hpp:28-63)
struct Matrix {
    std::size_t r = 0, c = 0;
    std::vector<double> v;
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, double fill = 0.0) : r(rows), c(cols), v(rows * cols, fill) {}
    std::size_t rows() const { return r; }
    std::size_t cols() const { return c; }
    double* row(std::size_t i) { return v.data() + i * c; }
    const double* row(std::size_t i) const { return v.data() + i * c; }
};
struct KeyCache {
    Matrix data;
    std::size_t tokens() const { return data.rows(); }
    std::size_t dim() const { return data.cols(); }
};
using ValueCache = KeyCache;
struct GroupSpec {
    std::size_t group_size = 32;
};
struct PackedKeys {
    std::size_t tokens = 0, dim = 0, group_size = 1, groups_per_channel = 0;
    std::vector<uint64_t> code_words;  // ceil(d/64) words per row, bit 1 <=> +1
    std::vector<double> scales, zeros;  // [gi * dim + j], binary16-rounded
    std::size_t payload_bytes() const { return tokens * ((dim + 7) / 8) + dim * groups_per_channel * 4; }
};
struct ScoreVector {
    std::vector<double> values;
    std::size_t size() const { return values.size(); }
};
struct Selection {
    std::vector<std::size_t> indices;
    std::size_t budget = 0;
};
struct RetrievalResult {
    Selection selection;
    std::vector<double> output;
    ScoreVector est_scores;
    uint64_t bytes_loaded_for_estimation = 0;
};
enum class QuestVariant { max_over_channels, sum_over_channels };  // baselines.hpp:28-31
// retrieval.hpp:20 (same enumerator order: the drop-in reads the reference's enum by value)
enum class PolicyKind { full, oracle, fier, quest, quest_quant, streaming_llm, h2o };
struct BudgetPolicy {  // retrieval.hpp:36-45 (the fields the device policies read)
    PolicyKind kind = PolicyKind::full;
    std::size_t budget = 0;
    std::size_t group_size = 32;
    std::size_t page_size = 16;
    QuestVariant variant = QuestVariant::sum_over_channels;
};
struct PolicySelection {  // retrieval.hpp:147-151
    Selection selection;
    ScoreVector est_scores;
    uint64_t bytes_loaded = 0;
};
struct LoadRatio {  // quant1bit.hpp:162-171
    long long numerator_bits = 0, denominator_bits = 1;
    bool formula = true;
};
struct PageSummaries {  // baselines.hpp:16-29
    std::size_t page_size = 16, tokens = 0, dim = 0;
    Matrix max_vecs, min_vecs;
    std::size_t page_count() const { return max_vecs.rows(); }
};
struct SideState {  // retrieval.hpp:88-103: the side state select_for_policy reads
    std::vector<std::pair<std::size_t, PackedKeys>> packed_by_group;
    std::vector<std::pair<std::size_t, PageSummaries>> pages_by_size;
    const PackedKeys& packed(std::size_t g) const {
        for (const auto& e : packed_by_group)
            if (e.first == g) return e.second;
        throw std::invalid_argument("run_policy: missing packed keys in side state");
    }
    const PageSummaries& pages(std::size_t L) const {
        for (const auto& e : pages_by_size)
            if (e.first == L) return e.second;
        throw std::invalid_argument("run_policy: missing page summaries in side state");
    }
};
}  // namespace types

namespace detail {

inline void check(int rc) {
    if (rc == FIER_OK) return;
    const std::string msg = fier_last_error();
    if (rc == FIER_EINVAL) throw std::invalid_argument(msg);
    if (rc == FIER_EDATA) throw DataError(msg);
    throw std::runtime_error(msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
template <typename T>
struct Dev {
    T* p = nullptr;
    std::size_t n = 0;
    explicit Dev(std::size_t count) : n(count) {
        cuda_check(cudaMalloc(&p, (count ? count : 1) * sizeof(T)), "cudaMalloc");
    }
    Dev(const T* host, std::size_t count) : Dev(count) {
        if (count) cuda_check(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy");
    }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    std::vector<T> host() const {
        std::vector<T> h(n);
        if (n) cuda_check(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy");
        return h;
    }
};

inline std::vector<float> to_f32(const double* x, std::size_t n) {
    std::vector<float> f(n);
    for (std::size_t i = 0; i < n; ++i) f[i] = static_cast<float>(x[i]);
    return f;
}

template <typename M>
inline const double* mat_data(const M& m) {  // KeyCache / ValueCache: row-major doubles (core.hpp:24-54)
    return m.data.row(0);
}

inline double half_to_double(uint16_t h) {  // exact widening (half.hpp:13-28)
    const int e = (h >> 10) & 0x1F, m = h & 0x3FF;
    const double sgn = (h & 0x8000) ? -1.0 : 1.0;
    if (e == 0) return sgn * std::ldexp((double)m, -24);
    if (e == 31) return m ? std::nan("") : sgn * INFINITY;
    return sgn * std::ldexp((double)(m | 0x400), e - 25);
}

inline fier_shape shape(int B, int Hq, int Hkv, int cap, int d, int g, int dtype = FIER_F32) {
    fier_shape s;
    s.batch = B;
    s.q_heads = Hq;
    s.kv_heads = Hkv;
    s.capacity = cap;
    s.dim = d;
    s.group = g;
    s.dtype = dtype;
    return s;
}

// device index of a single head (bits [l][W] u32, params [G][d] half2)
struct DevIndex {
    std::size_t l, d, g;
    Dev<uint32_t> bits;
    Dev<uint16_t> params;
    DevIndex(std::size_t l_, std::size_t d_, std::size_t g_)
        : l(l_), d(d_), g(g_), bits(l_ * ((d_ + 31) / 32)), params(((l_ + g_ - 1) / g_) * d_ * 2) {}
};

template <typename PK>
inline void upload(const PK& pk, DevIndex& di) {  // host PackedKeys -> device layout (u64 rows -> u32 words)
    const std::size_t W = (pk.dim + 31) / 32, W64 = (pk.dim + 63) / 64;
    std::vector<uint32_t> bits(pk.tokens * W, 0);
    for (std::size_t t = 0; t < pk.tokens; ++t)
        for (std::size_t w = 0; w < W; ++w)
            bits[t * W + w] = static_cast<uint32_t>(pk.code_words[t * W64 + w / 2] >> (32 * (w % 2)));
    std::vector<uint16_t> par(((pk.tokens + pk.group_size - 1) / pk.group_size) * pk.dim * 2);
    for (std::size_t i = 0; i < par.size() / 2; ++i) {
        const __half s = __double2half(pk.scales[i]), z = __double2half(pk.zeros[i]);
        std::memcpy(&par[2 * i], &s, 2);
        std::memcpy(&par[2 * i + 1], &z, 2);
    }
    cuda_check(cudaMemcpy(di.bits.p, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    cuda_check(cudaMemcpy(di.params.p, par.data(), par.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
}

}  // namespace detail

// quantize (quant1bit.hpp:65-103): the fp64 keys are packed as they are (FIER_F64)
template <typename PK = types::PackedKeys, typename KC, typename GS>
PK quantize(const KC& K, const GS& spec) {
    if (spec.group_size < 1) throw std::invalid_argument("quantize: group size must be >= 1");
    if (K.tokens() == 0 || K.dim() == 0) throw std::invalid_argument("quantize: empty key cache");
    const std::size_t l = K.tokens(), d = K.dim(), g = spec.group_size;
    detail::Dev<double> dk(detail::mat_data(K), l * d);
    detail::DevIndex di(l, d, g);
    detail::Dev<int32_t> flag(1);
    detail::cuda_check(cudaMemset(flag.p, 0, 4), "cudaMemset");
    fier_shape s = detail::shape(1, 1, 1, (int)l, (int)d, (int)g, FIER_F64);
    detail::check(fier_pack_keys(&s, dk.p, (int32_t)l, di.bits.p, di.params.p, flag.p, nullptr));
    detail::cuda_check(cudaDeviceSynchronize(), "quantize");
    if (flag.host()[0]) throw std::invalid_argument("quantize: non-finite key entry");
    const std::vector<uint32_t> bits = di.bits.host();
    const std::vector<uint16_t> par = di.params.host();
    PK pk;
    pk.tokens = l;
    pk.dim = d;
    pk.group_size = g;
    pk.groups_per_channel = (l + g - 1) / g;
    const std::size_t W = (d + 31) / 32, W64 = (d + 63) / 64;
    pk.code_words.assign(l * W64, 0);
    for (std::size_t t = 0; t < l; ++t)
        for (std::size_t w = 0; w < W; ++w)
            pk.code_words[t * W64 + w / 2] |= static_cast<uint64_t>(bits[t * W + w]) << (32 * (w % 2));
    pk.scales.resize(pk.groups_per_channel * d);
    pk.zeros.resize(pk.groups_per_channel * d);
    for (std::size_t i = 0; i < pk.scales.size(); ++i) {
        pk.scales[i] = detail::half_to_double(par[2 * i]);
        pk.zeros[i] = detail::half_to_double(par[2 * i + 1]);
    }
    return pk;
}

// approx_scores (quant1bit.hpp:121-140)
template <typename SV = types::ScoreVector, typename Q, typename PK>
SV approx_scores(const Q& q, const PK& pk) {
    if (q.size() != pk.dim) throw std::invalid_argument("approx_scores: query length does not match key dim");
    detail::DevIndex di(pk.tokens, pk.dim, pk.group_size);
    detail::upload(pk, di);
    const std::vector<float> qf = detail::to_f32(q.data(), q.size());
    detail::Dev<float> dq(qf.data(), qf.size());
    detail::Dev<float> ds(pk.tokens);
    fier_shape s = detail::shape(1, 1, 1, (int)pk.tokens, (int)pk.dim, (int)pk.group_size);
    detail::check(fier_score(&s, dq.p, di.bits.p, di.params.p, (int32_t)pk.tokens, ds.p, (int64_t)pk.tokens, nullptr));
    const std::vector<float> sc = ds.host();
    SV out;
    out.values.assign(sc.begin(), sc.end());
    return out;
}

// topk_oracle (core.hpp:134-148): the k largest, ties to the lower index, ascending --
// ranked on the fp64 scores themselves (fier_topk_f64)
template <typename SEL = types::Selection, typename SV>
SEL topk_oracle(const SV& scores, std::size_t k) {
    const std::size_t l = scores.values.size();
    if (k < 1 || k > l) throw std::invalid_argument("topk_oracle: k out of range");
    detail::Dev<double> ds(scores.values.data(), l);
    detail::Dev<int32_t> dsel(k);
    detail::check(fier_topk_f64(ds.p, 1, (int32_t)l, (int64_t)l, (int32_t)k, dsel.p, nullptr));
    const std::vector<int32_t> idx = dsel.host();
    SEL sel;
    sel.indices.assign(idx.begin(), idx.end());
    sel.budget = k;
    return sel;
}

// exact_scores (core.hpp:98-112): fp64 on the device in the reference's term order
template <typename SV = types::ScoreVector, typename Q, typename KC>
SV exact_scores(const Q& q, const KC& K, bool scaled = false) {
    if (q.size() != K.dim()) throw std::invalid_argument("exact_scores: query length does not match key dim");
    const std::size_t l = K.tokens(), d = K.dim();
    detail::Dev<double> dk(detail::mat_data(K), l * d), dq(q.data(), d), ds(l);
    fier_shape s = detail::shape(1, 1, 1, (int)l, (int)d, 1, FIER_F64);
    detail::check(fier_exact_scores(&s, dq.p, dk.p, (int32_t)l, scaled ? 1 : 0, ds.p, nullptr, (int64_t)l, nullptr));
    const std::vector<double> v = ds.host();
    SV out;
    out.values.assign(v.begin(), v.end());
    return out;
}

// load_ratio_fier (quant1bit.hpp:176-184)
template <typename LR = types::LoadRatio>
LR load_ratio_fier(std::size_t l, std::size_t g) {
    int64_t num = 0, den = 1;
    int32_t formula = 1;
    detail::check(fier_load_ratio_fier((int64_t)l, (int64_t)g, &num, &den, &formula));
    LR r;
    r.numerator_bits = num;
    r.denominator_bits = den;
    r.formula = formula != 0;
    return r;
}

// gather_attention (core.hpp:152-179)
template <typename OUT = std::vector<double>, typename Q, typename KC, typename VC, typename SEL>
OUT gather_attention(const Q& q, const KC& K, const VC& V, const SEL& sel, bool scaled = true) {
    if (K.tokens() != V.tokens() || K.dim() != V.dim())
        throw std::invalid_argument("gather_attention: K and V are not row-aligned");
    if (q.size() != K.dim()) throw std::invalid_argument("gather_attention: query length does not match key dim");
    if (sel.indices.empty()) throw std::invalid_argument("gather_attention: empty selection");
    for (std::size_t i = 0; i < sel.indices.size(); ++i)
        if (sel.indices[i] >= K.tokens() || (i > 0 && sel.indices[i] <= sel.indices[i - 1]))
            throw std::invalid_argument("gather_attention: selection invalid for cache");
    const std::size_t l = K.tokens(), d = K.dim(), n = sel.indices.size();
    const std::vector<float> kf = detail::to_f32(detail::mat_data(K), l * d), vf = detail::to_f32(detail::mat_data(V), l * d),
                             qf = detail::to_f32(q.data(), d);
    std::vector<int32_t> si(sel.indices.begin(), sel.indices.end());
    detail::Dev<float> dk(kf.data(), kf.size()), dv(vf.data(), vf.size()), dq(qf.data(), d), dout(d);
    detail::Dev<int32_t> dsel(si.data(), n);
    fier_shape s = detail::shape(1, 1, 1, (int)l, (int)d, 32);
    const std::size_t wsb = fier_sparse_attention_workspace(&s, (int32_t)n);
    detail::Dev<uint8_t> ws(wsb);
    const float scale = scaled ? 1.0f / std::sqrt((float)d) : 1.0f;
    detail::check(fier_sparse_attention(&s, dq.p, dk.p, dv.p, dsel.p, (int32_t)n, (int32_t)l, scale, dout.p, ws.p, wsb,
                                        nullptr));
    const std::vector<float> o = dout.host();
    return OUT(o.begin(), o.end());
}

// fier_select (retrieval.hpp:130-133)
template <typename SEL = types::Selection, typename Q, typename PK>
SEL fier_select(const Q& q, const PK& pk, std::size_t n) {
    if (n < 1 || n > pk.tokens) throw std::invalid_argument("fier_select: budget out of range");
    return ::fier::cuda::topk_oracle<SEL>(::fier::cuda::approx_scores(q, pk), n);
}

// fier_attend (retrieval.hpp:136-146)
template <typename RR = types::RetrievalResult, typename Q, typename KC, typename VC, typename PK>
RR fier_attend(const Q& q, const KC& K, const VC& V, const PK& pk, std::size_t n) {
    if (pk.tokens != K.tokens() || pk.dim != K.dim())
        throw std::invalid_argument("fier_attend: packed keys do not match cache");
    RR r;
    r.est_scores = ::fier::cuda::approx_scores<decltype(r.est_scores)>(q, pk);
    r.selection = ::fier::cuda::topk_oracle<decltype(r.selection)>(r.est_scores, n);
    r.output = ::fier::cuda::gather_attention<decltype(r.output)>(q, K, V, r.selection);
    r.bytes_loaded_for_estimation = pk.payload_bytes();
    return r;
}

// ---- Quest page retrieval (baselines.hpp) ----

namespace detail {
// detail::select_by_page_scores (baselines.hpp:85-111) of device page scores
template <typename SEL>
SEL page_select(const Dev<float>& dp, std::size_t tokens, std::size_t page_size, std::size_t n) {
    if (n < 1 || n > tokens) throw std::invalid_argument("page selection: budget out of range");
    const std::size_t P = (tokens + page_size - 1) / page_size;
    const std::size_t wsb = fier_page_select_workspace(1, (int32_t)tokens, (int32_t)page_size, (int32_t)n);
    Dev<uint8_t> ws(wsb);
    Dev<int32_t> dsel(n);
    check(fier_page_select(dp.p, 1, (int32_t)tokens, (int64_t)P, (int32_t)page_size, (int32_t)n, dsel.p, ws.p, wsb,
                           nullptr));
    const std::vector<int32_t> idx = dsel.host();
    SEL sel;
    sel.indices.assign(idx.begin(), idx.end());
    sel.budget = n;
    return sel;
}
}  // namespace detail

// build_page_summaries (baselines.hpp:34-56): channel-wise page extrema on the device
template <typename PS = types::PageSummaries, typename KC>
PS build_page_summaries(const KC& K, std::size_t page_size) {
    if (page_size < 1) throw std::invalid_argument("build_page_summaries: page size must be >= 1");
    const std::size_t l = K.tokens(), d = K.dim(), P = (l + page_size - 1) / page_size;
    const std::vector<float> kf = detail::to_f32(detail::mat_data(K), l * d);
    detail::Dev<float> dk(kf.data(), kf.size()), mx(P * d), mn(P * d);
    fier_shape s = detail::shape(1, 1, 1, (int)l, (int)d, 1);
    detail::check(fier_quest_summaries(&s, dk.p, (int32_t)l, (int32_t)page_size, mx.p, mn.p, nullptr));
    const std::vector<float> hx = mx.host(), hn = mn.host();
    PS ps;
    ps.page_size = page_size;
    ps.tokens = l;
    ps.dim = d;
    ps.max_vecs = decltype(ps.max_vecs)(P, d);
    ps.min_vecs = decltype(ps.min_vecs)(P, d);
    for (std::size_t p = 0; p < P; ++p)
        for (std::size_t j = 0; j < d; ++j) {
            ps.max_vecs.row(p)[j] = hx[p * d + j];
            ps.min_vecs.row(p)[j] = hn[p * d + j];
        }
    return ps;
}

// quest_select (baselines.hpp:113-118); variant: the reference's QuestVariant (max = 0, sum = 1)
template <typename SEL = types::Selection, typename Q, typename KC, typename PS, typename VAR>
SEL quest_select(const Q& q, const KC& K, const PS& ps, std::size_t n, VAR variant) {
    if (K.tokens() != ps.tokens || K.dim() != ps.dim)
        throw std::invalid_argument("quest_select: summaries do not match cache");
    if (q.size() != ps.dim) throw std::invalid_argument("quest_page_scores: query length does not match dim");
    const std::size_t P = ps.page_count(), d = ps.dim;
    std::vector<float> hx(P * d), hn(P * d);
    for (std::size_t p = 0; p < P; ++p)
        for (std::size_t j = 0; j < d; ++j) {
            hx[p * d + j] = static_cast<float>(ps.max_vecs.row(p)[j]);
            hn[p * d + j] = static_cast<float>(ps.min_vecs.row(p)[j]);
        }
    const std::vector<float> qf = detail::to_f32(q.data(), d);
    detail::Dev<float> mx(hx.data(), hx.size()), mn(hn.data(), hn.size()), dq(qf.data(), d), dp(P);
    fier_shape s = detail::shape(1, 1, 1, (int)ps.tokens, (int)d, 1);
    detail::check(fier_quest_page_scores(&s, dq.p, mx.p, mn.p, (int32_t)ps.tokens, (int32_t)ps.page_size,
                                         static_cast<int>(variant) == 1 ? 1 : 0, dp.p, (int64_t)P, nullptr));
    return detail::page_select<SEL>(dp, ps.tokens, ps.page_size, n);
}

// quest_select_quantized (baselines.hpp:120-140): pages scored by the mean 1-bit estimate
template <typename SEL = types::Selection, typename Q, typename PK>
SEL quest_select_quantized(const Q& q, const PK& pk, std::size_t page_size, std::size_t n) {
    if (page_size < 1) throw std::invalid_argument("quest_select_quantized: page size must be >= 1");
    if (q.size() != pk.dim) throw std::invalid_argument("approx_scores: query length does not match key dim");
    const std::size_t l = pk.tokens, P = (l + page_size - 1) / page_size;
    detail::DevIndex di(l, pk.dim, pk.group_size);
    detail::upload(pk, di);
    const std::vector<float> qf = detail::to_f32(q.data(), q.size());
    detail::Dev<float> dq(qf.data(), qf.size()), ds(l), dp(P);
    fier_shape s = detail::shape(1, 1, 1, (int)l, (int)pk.dim, (int)pk.group_size);
    detail::check(fier_score(&s, dq.p, di.bits.p, di.params.p, (int32_t)l, ds.p, (int64_t)l, nullptr));
    detail::check(fier_page_mean(ds.p, 1, (int32_t)l, (int64_t)l, (int32_t)page_size, dp.p, (int64_t)P, nullptr));
    return detail::page_select<SEL>(dp, l, page_size, n);
}

// ---- policy dispatch (retrieval.hpp:155-233): the device-side policies ----
//
// select_for_policy's branches for the policies on the device path -- full, oracle,
// fier (retrieval.hpp:177-183: the Fier index from state.packed(policy.group_size),
// approx_scores -> topk_oracle, bytes = payload_bytes), quest and quest_quant --
// with the reference's preconditions and messages.  streaming_llm and h2o are not on
// the Fier path (SURVEY §8 out of scope) and throw.  PS / the policy / the side state
// may be the reference's own types (PolicySelection, BudgetPolicy, SideState).
template <typename PS = types::PolicySelection, typename POL, typename Q, typename KC, typename ST>
PS select_for_policy(const POL& policy, const Q& q, const KC& K, const ST& state) {
    const std::size_t l = K.tokens();
    PS r;
    const int kind = static_cast<int>(policy.kind);  // PolicyKind enumerator order, retrieval.hpp:20
    if (kind == static_cast<int>(types::PolicyKind::full)) {  // pass-through: budget does not apply
        r.selection.budget = l;
        r.selection.indices.resize(l);
        for (std::size_t i = 0; i < l; ++i) r.selection.indices[i] = i;
        r.est_scores = ::fier::cuda::exact_scores<decltype(r.est_scores)>(q, K);
        return r;
    }
    const std::size_t n = policy.budget;
    if (n < 1 || n > l) throw std::invalid_argument("run_policy: budget out of range for cache");
    switch (static_cast<types::PolicyKind>(kind)) {
        case types::PolicyKind::oracle:
            r.est_scores = ::fier::cuda::exact_scores<decltype(r.est_scores)>(q, K);
            r.selection = ::fier::cuda::topk_oracle<decltype(r.selection)>(r.est_scores, n);
            r.bytes_loaded = static_cast<uint64_t>(l) * K.dim() * 2;
            break;
        case types::PolicyKind::fier: {
            const auto& pk = state.packed(policy.group_size);
            r.est_scores = ::fier::cuda::approx_scores<decltype(r.est_scores)>(q, pk);
            r.selection = ::fier::cuda::topk_oracle<decltype(r.selection)>(r.est_scores, n);
            r.bytes_loaded = pk.payload_bytes();
            break;
        }
        case types::PolicyKind::quest: {
            const auto& ps = state.pages(policy.page_size);
            r.selection = ::fier::cuda::quest_select<decltype(r.selection)>(q, K, ps, n, policy.variant);
            r.bytes_loaded = static_cast<uint64_t>(ps.page_count()) * ps.dim * 4;
            break;
        }
        case types::PolicyKind::quest_quant: {
            const auto& pk = state.packed(policy.group_size);
            r.selection = ::fier::cuda::quest_select_quantized<decltype(r.selection)>(q, pk, policy.page_size, n);
            r.est_scores = ::fier::cuda::approx_scores<decltype(r.est_scores)>(q, pk);
            r.bytes_loaded = pk.payload_bytes();
            break;
        }
        default:
            throw std::invalid_argument("run_policy: policy not on the device path (streaming_llm, h2o)");
    }
    return r;
}

// run_policy (retrieval.hpp:223-233): the selection, then gather_attention on it
template <typename RR = types::RetrievalResult, typename POL, typename Q, typename KC, typename VC, typename ST>
RR run_policy(const POL& policy, const Q& q, const KC& K, const VC& V, const ST& state) {
    auto ps = ::fier::cuda::select_for_policy<types::PolicySelection>(policy, q, K, state);
    RR r;
    r.selection.indices = std::move(ps.selection.indices);
    r.selection.budget = ps.selection.budget;
    r.est_scores.values = std::move(ps.est_scores.values);
    r.bytes_loaded_for_estimation = ps.bytes_loaded;
    r.output = ::fier::cuda::gather_attention<decltype(r.output)>(q, K, V, r.selection);
    return r;
}

}  // namespace cuda
}  // namespace fier

#endif  // FIER_CUDA_HPP_
