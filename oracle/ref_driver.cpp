// oracle/ref_driver.cpp -- extern "C" entry points over the REFERENCE's own
// headers (compiled in place from /root/reference/proj/include by
// oracle/Makefile; nothing is copied).  Output: oracle/_ref/libfier_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (parity, golden-vector
// generation) and by bench.py's cpu_baseline / --impl reference legs as the
// reference CPU implementation.  The product path never loads it.
//
// Each wrapper calls exactly one reference function; errors thrown by the
// reference (std::invalid_argument from require(), fier::DataError) are
// mapped to status 1 / 2 with the message kept in a thread-local buffer.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fier/baselines.hpp"
#include "fier/core.hpp"
#ifdef FIER_REF_HARNESS
#include "fier/evalharness.hpp"
#endif
#include "fier/half.hpp"
#include "fier/io.hpp"
#include "fier/quant1bit.hpp"
#include "fier/retrieval.hpp"
#include "fier/workload.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const fier::DataError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

fier::KeyCache key_cache(const double* K, size_t l, size_t d) {
    fier::KeyCache kc;
    kc.data = fier::Matrix(l, d);
    std::memcpy(kc.data.data().data(), K, l * d * sizeof(double));
    return kc;
}
fier::ValueCache value_cache(const double* V, size_t l, size_t d) {
    fier::ValueCache vc;
    vc.data = fier::Matrix(l, d);
    std::memcpy(vc.data.data().data(), V, l * d * sizeof(double));
    return vc;
}
fier::Selection selection(const int64_t* idx, size_t n, size_t budget) {
    fier::Selection s;
    s.budget = budget;
    s.indices.assign(idx, idx + n);
    return s;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint16_t ref_double_to_half(double x) { return fier::double_to_half(x); }   // half.hpp:30
// load_ratio_fier (quant1bit.hpp:176-184): the unreduced bit counts, the reduced ratio
// (Rational, quant1bit.hpp:143-160) and the formula flag
int ref_load_ratio_fier(size_t l, size_t g, long long* bits, long long* ratio, int* formula) {
    return guard([&] {
        const fier::LoadRatio r = fier::load_ratio_fier(l, g);
        bits[0] = r.numerator_bits;
        bits[1] = r.denominator_bits;
        const fier::Rational q = r.ratio();
        ratio[0] = q.num;
        ratio[1] = q.den;
        *formula = r.formula ? 1 : 0;
    });
}
double ref_half_to_double(uint16_t h) { return fier::half_to_double(h); }   // half.hpp:13

// quantize (quant1bit.hpp:65) -> serialize_packed_keys (io.hpp:197).
// out may be null to query the length.
int ref_quantize_fier(const double* K, size_t l, size_t d, size_t g, unsigned char* out, size_t cap,
                      size_t* len) {
    return guard([&] {
        const fier::PackedKeys pk = fier::quantize(key_cache(K, l, d), fier::GroupSpec{g});
        const std::string bytes = fier::serialize_packed_keys(pk);
        *len = bytes.size();
        if (out) {
            if (cap < bytes.size()) throw std::invalid_argument("ref_quantize_fier: buffer too small");
            std::memcpy(out, bytes.data(), bytes.size());
        }
    });
}

// quantize (quant1bit.hpp:65), in-memory fp64 parameters, raw.
int ref_quantize_inmem(const double* K, size_t l, size_t d, size_t g, uint64_t* code_words,
                       double* scales, double* zeros) {
    return guard([&] {
        const fier::PackedKeys pk = fier::quantize(key_cache(K, l, d), fier::GroupSpec{g});
        std::memcpy(code_words, pk.code_words.data(), pk.code_words.size() * sizeof(uint64_t));
        std::memcpy(scales, pk.scales.data(), pk.scales.size() * sizeof(double));
        std::memcpy(zeros, pk.zeros.data(), pk.zeros.size() * sizeof(double));
    });
}

// approx_scores (quant1bit.hpp:121) over parse_packed_keys (io.hpp:227): the
// half-round-tripped index the GPU stores.
int ref_approx_scores_fier(const double* q, const unsigned char* fier_bytes, size_t len,
                           double* out) {
    return guard([&] {
        const fier::PackedKeys pk =
            fier::parse_packed_keys(std::string(reinterpret_cast<const char*>(fier_bytes), len));
        const fier::QueryVector qv(q, q + pk.dim);
        const fier::ScoreVector s = fier::approx_scores(qv, pk);
        std::memcpy(out, s.values.data(), s.values.size() * sizeof(double));
    });
}

// topk_oracle (core.hpp:134)
int ref_topk(const double* scores, size_t l, size_t k, int64_t* out) {
    return guard([&] {
        fier::ScoreVector s;
        s.values.assign(scores, scores + l);
        const fier::Selection sel = fier::topk_oracle(s, k);
        for (size_t i = 0; i < sel.indices.size(); ++i) out[i] = static_cast<int64_t>(sel.indices[i]);
    });
}

// gather_attention (core.hpp:152)
int ref_gather_attention(const double* q, const double* K, const double* V, size_t l, size_t d,
                         const int64_t* idx, size_t n, int scaled, double* out) {
    return guard([&] {
        const fier::QueryVector qv(q, q + d);
        const fier::AttentionOutput o = fier::gather_attention(
            qv, key_cache(K, l, d), value_cache(V, l, d), selection(idx, n, n), scaled != 0);
        std::memcpy(out, o.data(), d * sizeof(double));
    });
}

// exact_scores (core.hpp:98)
int ref_exact_scores(const double* q, const double* K, size_t l, size_t d, int scaled, double* out) {
    return guard([&] {
        const fier::QueryVector qv(q, q + d);
        const fier::ScoreVector s = fier::exact_scores(qv, key_cache(K, l, d), scaled != 0);
        std::memcpy(out, s.values.data(), l * sizeof(double));
    });
}

// fier_attend (retrieval.hpp:136) on a FIER-serialized index; returns the
// selection, output, estimated scores and bytes_loaded_for_estimation.
int ref_fier_attend_fier(const double* q, const double* K, const double* V, size_t l, size_t d,
                         const unsigned char* fier_bytes, size_t len, size_t n, int64_t* sel_out,
                         double* out, double* est_out, uint64_t* bytes_loaded) {
    return guard([&] {
        const fier::PackedKeys pk =
            fier::parse_packed_keys(std::string(reinterpret_cast<const char*>(fier_bytes), len));
        const fier::QueryVector qv(q, q + d);
        const fier::RetrievalResult r =
            fier::fier_attend(qv, key_cache(K, l, d), value_cache(V, l, d), pk, n);
        for (size_t i = 0; i < r.selection.indices.size(); ++i)
            sel_out[i] = static_cast<int64_t>(r.selection.indices[i]);
        std::memcpy(out, r.output.data(), d * sizeof(double));
        if (est_out) std::memcpy(est_out, r.est_scores.values.data(), l * sizeof(double));
        *bytes_loaded = r.bytes_loaded_for_estimation;
    });
}

// generate (workload.hpp:128) with the planted_spikes / gaussian generators.
int ref_generate(size_t l, size_t d, int planted, size_t spike_count, double spike_gain,
                 uint64_t seed, size_t query_count, double* K, double* V, double* Q) {
    return guard([&] {
        fier::WorkloadSpec spec;
        spec.tokens = l;
        spec.dim = d;
        spec.generator = planted ? fier::Generator::planted_spikes : fier::Generator::gaussian;
        spec.spike_count = spike_count;
        spec.spike_gain = spike_gain;
        spec.seed = seed;
        spec.query_count = query_count;
        const fier::WorkloadInstance w = fier::generate(spec);
        std::memcpy(K, w.keys.data.data().data(), l * d * sizeof(double));
        std::memcpy(V, w.values.data.data().data(), l * d * sizeof(double));
        for (size_t i = 0; i < query_count; ++i)
            std::memcpy(Q + i * d, w.queries[i].data(), d * sizeof(double));
    });
}

// ---- multi-head CPU decode step (the reference arm / cpu_baseline) -------------
//
// One layer: Hkv key/value caches of l x d, Hq query heads (GQA: head h reads
// kv head h / (Hq/Hkv)).  The index is built once per kv head with quantize,
// round-tripped through the FIER format (the fp16 (s, z) the GPU stores), and
// hoisted out of the step (retrieval.hpp:5-6).  A step runs
// fier_attend (retrieval.hpp:136) for every q head, split across std::thread
// workers (the FIER_THREADS model, evalharness.hpp:155-162, 279-297).

struct RefLayer {
    size_t hq = 0, hkv = 0, l = 0, d = 0, g = 32;
    std::vector<fier::KeyCache> K;
    std::vector<fier::ValueCache> V;
    std::vector<fier::PackedKeys> pk;
};

void* ref_layer_build(const float* K, const float* V, size_t hkv, size_t l, size_t d, size_t g,
                      size_t threads) {
    RefLayer* L = new RefLayer;
    L->hkv = hkv; L->l = l; L->d = d; L->g = g;
    L->K.resize(hkv); L->V.resize(hkv); L->pk.resize(hkv);
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t h; (h = next.fetch_add(1)) < hkv;) {
            fier::KeyCache kc; kc.data = fier::Matrix(l, d);
            fier::ValueCache vc; vc.data = fier::Matrix(l, d);
            const float* ks = K + h * l * d;
            const float* vs = V + h * l * d;
            for (size_t i = 0; i < l * d; ++i) {
                kc.data.data()[i] = ks[i];
                vc.data.data()[i] = vs[i];
            }
            L->pk[h] = fier::parse_packed_keys(
                fier::serialize_packed_keys(fier::quantize(kc, fier::GroupSpec{g})));
            L->K[h] = std::move(kc);
            L->V[h] = std::move(vc);
        }
    };
    std::vector<std::thread> pool;
    for (size_t t = 0; t < std::max<size_t>(1, threads); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    return L;
}

void ref_layer_free(void* p) { delete static_cast<RefLayer*>(p); }

// Runs one decode step for q heads [h0, h1) of Q (hq x d floats); writes the
// per-head selections (hq x n int32) and outputs (hq x d) for those heads.
// Returns wall seconds.
double ref_layer_step(void* p, const float* Q, size_t hq, size_t h0, size_t h1, size_t n,
                      size_t threads, int32_t* sel_out, double* out) {
    RefLayer* L = static_cast<RefLayer*>(p);
    const size_t group = hq / L->hkv;
    std::atomic<size_t> next{h0};
    std::atomic<int> failed{0};
    auto t0 = std::chrono::steady_clock::now();
    auto work = [&] {
        for (size_t h; (h = next.fetch_add(1)) < h1;) {
            try {
                const size_t kv = h / group;
                fier::QueryVector q(Q + h * L->d, Q + (h + 1) * L->d);
                const fier::RetrievalResult r = fier::fier_attend(q, L->K[kv], L->V[kv], L->pk[kv], n);
                if (sel_out)
                    for (size_t i = 0; i < n; ++i) sel_out[h * n + i] = static_cast<int32_t>(r.selection.indices[i]);
                if (out) std::memcpy(out + h * L->d, r.output.data(), L->d * sizeof(double));
            } catch (const std::exception& e) {
                g_err = e.what();
                failed = 1;
            }
        }
    };
    std::vector<std::thread> pool;
    for (size_t t = 0; t < std::max<size_t>(1, threads); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    auto t1 = std::chrono::steady_clock::now();
    if (failed) return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
}

// ---- Quest page retrieval (baselines.hpp), SURVEY 8(f) row 2 ----

// build_page_summaries (baselines.hpp:34)
int ref_page_summaries(const double* K, size_t l, size_t d, size_t L, double* kmax, double* kmin) {
    return guard([&] {
        const fier::PageSummaries ps = fier::build_page_summaries(key_cache(K, l, d), L);
        std::memcpy(kmax, ps.max_vecs.data().data(), ps.page_count() * d * sizeof(double));
        std::memcpy(kmin, ps.min_vecs.data().data(), ps.page_count() * d * sizeof(double));
    });
}

// quest_page_scores (baselines.hpp:60) over build_page_summaries; variant 1 = sum, 0 = max
int ref_quest_page_scores(const double* q, const double* K, size_t l, size_t d, size_t L, int variant,
                          double* out) {
    return guard([&] {
        const fier::PageSummaries ps = fier::build_page_summaries(key_cache(K, l, d), L);
        const std::vector<double> s = fier::quest_page_scores(
            fier::QueryVector(q, q + d), ps,
            variant ? fier::QuestVariant::sum_over_channels : fier::QuestVariant::max_over_channels);
        std::memcpy(out, s.data(), s.size() * sizeof(double));
    });
}

// quest_select (baselines.hpp:113)
int ref_quest_select(const double* q, const double* K, size_t l, size_t d, size_t L, size_t n, int variant,
                     int64_t* out) {
    return guard([&] {
        const fier::KeyCache kc = key_cache(K, l, d);
        const fier::PageSummaries ps = fier::build_page_summaries(kc, L);
        const fier::Selection sel = fier::quest_select(
            fier::QueryVector(q, q + d), kc, ps, n,
            variant ? fier::QuestVariant::sum_over_channels : fier::QuestVariant::max_over_channels);
        for (size_t i = 0; i < sel.indices.size(); ++i) out[i] = static_cast<int64_t>(sel.indices[i]);
    });
}

// quest_select_quantized (baselines.hpp:120) over parse_packed_keys (io.hpp:227)
int ref_quest_select_quantized(const double* q, const unsigned char* fier_bytes, size_t len, size_t L, size_t n,
                               int64_t* out) {
    return guard([&] {
        const fier::PackedKeys pk =
            fier::parse_packed_keys(std::string(reinterpret_cast<const char*>(fier_bytes), len));
        const fier::Selection sel = fier::quest_select_quantized(fier::QueryVector(q, q + pk.dim), pk, L, n);
        for (size_t i = 0; i < sel.indices.size(); ++i) out[i] = static_cast<int64_t>(sel.indices[i]);
    });
}

// detail::select_by_page_scores (baselines.hpp:85) on given page scores (geometry only)
int ref_select_by_page_scores(const double* page_scores, size_t l, size_t L, size_t n, int64_t* out) {
    return guard([&] {
        fier::PageSummaries layout;
        layout.page_size = L;
        layout.tokens = l;
        const size_t pages = (l + L - 1) / L;
        layout.max_vecs = fier::Matrix(pages, 0);
        layout.min_vecs = fier::Matrix(pages, 0);
        const fier::Selection sel =
            fier::detail::select_by_page_scores(std::vector<double>(page_scores, page_scores + pages), layout, n);
        for (size_t i = 0; i < sel.indices.size(); ++i) out[i] = static_cast<int64_t>(sel.indices[i]);
    });
}

// ---- evaluation harness (evalharness.hpp), SURVEY 8(f) row 4 ----
#ifdef FIER_REF_HARNESS

// margin_and_errors (evalharness.hpp:63) over parse_packed_keys (io.hpp:227); out =
// (margin, max_err, l2_loss, hinge_loss, hinge_loss_symmetric)
int ref_margin_and_errors(const double* q, const double* K, size_t l, size_t d, const unsigned char* fier_bytes,
                          size_t len, size_t k, double* out) {
    return guard([&] {
        const fier::PackedKeys pk =
            fier::parse_packed_keys(std::string(reinterpret_cast<const char*>(fier_bytes), len));
        const fier::MarginReport r = fier::margin_and_errors(fier::QueryVector(q, q + d), key_cache(K, l, d), pk, k);
        out[0] = r.margin;
        out[1] = r.max_err;
        out[2] = r.l2_loss;
        out[3] = r.hinge_loss;
        out[4] = r.hinge_loss_symmetric;
    });
}

// run_trial (evalharness.hpp:184) on a fixed workload with the policies fier(g),
// quest(L, variant), quest_quant(g, L), oracle, full (in that order); cells[p][b] =
// (recall, out_err, max_err), margins[b].
int ref_run_trial(const double* K, const double* V, size_t l, size_t d, const double* Q, size_t nq, size_t g,
                  size_t L, int variant, const size_t* budgets, size_t nb, double* cells, double* margins) {
    return guard([&] {
        fier::WorkloadInstance w;
        w.keys = key_cache(K, l, d);
        w.values = value_cache(V, l, d);
        for (size_t i = 0; i < nq; ++i) w.queries.emplace_back(Q + i * d, Q + (i + 1) * d);
        std::vector<fier::BudgetPolicy> pol(5);
        const fier::PolicyKind kinds[5] = {fier::PolicyKind::fier, fier::PolicyKind::quest,
                                           fier::PolicyKind::quest_quant, fier::PolicyKind::oracle,
                                           fier::PolicyKind::full};
        for (int i = 0; i < 5; ++i) {
            pol[i].kind = kinds[i];
            pol[i].group_size = g;
            pol[i].page_size = L;
            pol[i].variant = variant ? fier::QuestVariant::sum_over_channels : fier::QuestVariant::max_over_channels;
        }
        const fier::detail::TrialData t =
            fier::detail::run_trial(fier::WorkloadSpec{}, 0, pol, std::vector<size_t>(budgets, budgets + nb), &w);
        for (size_t i = 0; i < t.cells.size(); ++i) {
            cells[3 * i] = t.cells[i].recall;
            cells[3 * i + 1] = t.cells[i].out_err;
            cells[3 * i + 2] = t.cells[i].has_max_err ? t.cells[i].max_err : -1.0;
        }
        for (size_t b = 0; b < nb; ++b) margins[b] = t.margins[b];
    });
}

#endif  // FIER_REF_HARNESS

}  // extern "C"
