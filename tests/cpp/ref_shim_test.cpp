// ref_shim_test.cpp -- the C++ drop-in (include/fier_cuda.hpp) compiled NEXT TO the
// reference's own headers and called with the reference's own types, checked against
// the reference's CPU functions on the same fp64 inputs.  Test infrastructure: built by
// paper_2508_08256_b200/build.py::build_ref_shim_test only where /root/reference exists
// (this container); the binary travels to the GPU box, where
// tests/test_capi.py::test_ref_shim_against_reference runs it.  Prints PASS/FAIL lines,
// exit code 0 iff every check passes.
//
// Checks (reference file:line of what is compared):
//   quantize       serialize_packed_keys(fier::cuda::quantize<fier::PackedKeys>(K)) ==
//                  serialize_packed_keys(fier::quantize(K))   quant1bit.hpp:65-103, io.hpp:197-225
//                  on Gaussian fp64 keys (not fp32-representable), short groups, g = 1,
//                  signed zeros, constant groups at the half-narrowing KAT values
//                  (test_io.cpp:41-86: >= 65520 -> inf, subnormals, ties)
//   topk_oracle    fp64 scores incl. doubles that tie after fp32 rounding   core.hpp:134-148
//   exact_scores   bit-identical                                           core.hpp:98-112
//   select_for_policy / run_policy: full, oracle (bit-identical), fier and quest_quant on
//                  planted keys (same selection), bytes_loaded, error texts  retrieval.hpp:155-233
//   load_ratio_fier                                                         quant1bit.hpp:176-184
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "fier/core.hpp"
#include "fier/io.hpp"
#include "fier/quant1bit.hpp"
#include "fier/retrieval.hpp"
#include "fier_cuda.hpp"

static int g_fail = 0;

static void report(bool ok, const std::string& name, const std::string& detail = "") {
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.empty() ? "" : ": ", detail.c_str());
    if (!ok) ++g_fail;
}

static fier::KeyCache gaussian(std::size_t l, std::size_t d, uint64_t seed, double scale = 1.0) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> nd(0.0, scale);
    fier::KeyCache K;
    K.data = fier::Matrix(l, d);
    for (auto& x : K.data.data()) x = nd(rng);
    return K;
}

static void check_quantize(const fier::KeyCache& K, std::size_t g, const std::string& name) {
    const std::string want = fier::serialize_packed_keys(fier::quantize(K, fier::GroupSpec{g}));
    const std::string got =
        fier::serialize_packed_keys(fier::cuda::quantize<fier::PackedKeys>(K, fier::GroupSpec{g}));
    std::size_t diff = 0;
    for (std::size_t i = 0; i < std::min(want.size(), got.size()); ++i) diff += want[i] != got[i];
    report(want == got, "quantize " + name,
           want == got ? "" : std::to_string(diff) + " bytes differ of " + std::to_string(want.size()));
}

template <typename A, typename B>
static bool same_indices(const A& a, const B& b) {
    if (a.indices.size() != b.indices.size()) return false;
    for (std::size_t i = 0; i < a.indices.size(); ++i)
        if (a.indices[i] != b.indices[i]) return false;
    return true;
}

template <typename F>
static std::string error_of(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument& e) {
        return e.what();
    }
    return "";
}

int main() {
    // ---- quantize on the reference's fp64 keys ----
    check_quantize(gaussian(4096, 128, 1), 32, "gaussian 4096x128 g=32");
    for (uint64_t s = 2; s < 12; ++s) check_quantize(gaussian(1000 + 37 * s, 64, s, 3.0), 32, "gaussian seed " + std::to_string(s));
    check_quantize(gaussian(333, 24, 13), 128, "short final group 333x24 g=128");
    check_quantize(gaussian(100, 11, 14), 1, "g=1 100x11");
    check_quantize(gaussian(257, 96, 15, 1e-3), 7, "small scale 257x96 g=7");
    check_quantize(gaussian(300, 40, 16, 5e4), 5, "large scale (half overflow) 300x40 g=5");
    {  // signed zeros: {-0,+0} -> z 0x8000, {+0,-0} -> z 0x0000
        fier::KeyCache K;
        K.data = fier::Matrix(4, 2);
        K.data(0, 0) = -0.0, K.data(1, 0) = 0.0, K.data(2, 0) = 0.0, K.data(3, 0) = -0.0;
        K.data(0, 1) = 0.0, K.data(1, 1) = -0.0, K.data(2, 1) = 1.0, K.data(3, 1) = -1.0;
        check_quantize(K, 2, "signed zeros");
    }
    {  // constant groups at the narrowing KATs (test_io.cpp:41-86): z = v, s = 0
        const double kats[] = {0.0, -0.0, 1.0, -2.0, 65504.0, 65519.999, 65520.0, 1e9, -65520.0,
                               5.960464477539063e-08, 2.9802322387695312e-08, 2.980232536792755e-08,
                               1.4901161193847656e-08, 0.1, 0.2, 0.3, 1.0009765625, 1.00048828125, 1.00146484375,
                               2047.5, 2048.5, 0.333251953125, 3.141592653589793, -0.0001, 1e-08,
                               6.097555160522461e-05, -1.4238250364546312, 12.637284581291103, -87.06617379590857,
                               -259.1732349343976, -0.0007534330701052097, -7.408846520856091e-05,
                               -13677.927017829434, 0.6488928021930399};
        const std::size_t d = sizeof(kats) / sizeof(kats[0]);
        fier::KeyCache K;
        K.data = fier::Matrix(6, d);
        for (std::size_t j = 0; j < d; ++j) {
            K.data(0, j) = K.data(1, j) = kats[j];            // constant group: z = v
            K.data(2, j) = kats[j], K.data(3, j) = -kats[j];  // symmetric group: s = |v|, z = 0
            K.data(4, j) = 2.0 * kats[j], K.data(5, j) = 0.0; // z = v, s = |v| via (mx+mn)/2
        }
        check_quantize(K, 2, "narrowing KAT groups");
    }
    // ---- topk_oracle on fp64 scores ----
    {
        fier::ScoreVector sv;
        std::mt19937_64 rng(21);
        std::normal_distribution<double> nd(0.0, 1.0);
        sv.values.resize(50000);
        for (auto& x : sv.values) x = nd(rng);
        for (std::size_t i = 0; i < sv.values.size(); i += 3)  // distinct doubles, equal as floats
            sv.values[i] = 1.0 + (double)(i % 7) * 1e-12;
        for (std::size_t i = 5; i < sv.values.size(); i += 11) sv.values[i] = 1.0;  // exact ties
        bool ok = true;
        for (std::size_t k : {1u, 100u, 9000u, 16667u, 20000u, 50000u}) {
            ok &= same_indices(fier::topk_oracle(sv, k), fier::cuda::topk_oracle<fier::Selection>(sv, k));
        }
        report(ok, "topk_oracle fp64 (ties after fp32 rounding, exact ties)");
        report(error_of([&] { fier::cuda::topk_oracle<fier::Selection>(sv, 0); }) == "topk_oracle: k out of range",
               "topk_oracle error text");
    }
    // ---- exact_scores ----
    const std::size_t l = 6000, d = 128, g = 32, n = 300;
    fier::KeyCache K = gaussian(l, d, 31);
    fier::ValueCache V;
    V.data = gaussian(l, d, 32).data;
    fier::QueryVector q(d);
    {
        std::mt19937_64 rng(33);
        std::normal_distribution<double> nd(0.0, 1.0);
        for (auto& x : q) x = nd(rng);
    }
    {
        const auto want = fier::exact_scores(q, K, false), want_s = fier::exact_scores(q, K, true);
        const auto got = fier::cuda::exact_scores<fier::ScoreVector>(q, K, false);
        const auto got_s = fier::cuda::exact_scores<fier::ScoreVector>(q, K, true);
        report(want.values == got.values && want_s.values == got_s.values, "exact_scores bit-identical");
    }
    // planted keys: n contiguous tokens aligned with q by a wide margin, so every policy's
    // estimate ranks them first (the selection is unambiguous under fp16 (s, z) and fp32
    // scores; quest_quant takes their 18 whole pages and the first 12 tokens of the 19th)
    fier::KeyCache KP = K;
    for (std::size_t i = 0; i < n; ++i) {
        const std::size_t t = 1600 + i;
        for (std::size_t j = 0; j < d; ++j) KP.data(t, j) = 0.25 * KP.data(t, j) + 2.0 * q[j];
    }
    // ---- select_for_policy / run_policy with the reference's own types ----
    std::vector<fier::BudgetPolicy> pols(4);
    pols[0].kind = fier::PolicyKind::full;
    pols[1].kind = fier::PolicyKind::oracle;
    pols[1].budget = n;
    pols[2].kind = fier::PolicyKind::fier;
    pols[2].budget = n;
    pols[2].group_size = g;
    pols[3].kind = fier::PolicyKind::quest_quant;
    pols[3].budget = n;
    pols[3].group_size = g;
    pols[3].page_size = 16;
    const fier::SideState st = fier::build_side_state(pols, KP);
    for (const auto& pol : pols) {
        const fier::PolicySelection want = fier::select_for_policy(pol, q, KP, st);
        const fier::PolicySelection got = fier::cuda::select_for_policy<fier::PolicySelection>(pol, q, KP, st);
        bool ok = same_indices(want.selection, got.selection) && want.selection.budget == got.selection.budget &&
                  want.bytes_loaded == got.bytes_loaded && want.est_scores.values.size() == got.est_scores.values.size();
        if (pol.kind == fier::PolicyKind::full || pol.kind == fier::PolicyKind::oracle)
            ok &= want.est_scores.values == got.est_scores.values;  // fp64 on the device, same term order
        report(ok, std::string("select_for_policy ") + fier::policy_name(pol.kind));
        if (pol.kind != fier::PolicyKind::full) {
            const fier::RetrievalResult rw = fier::run_policy(pol, q, KP, V, st);
            const fier::RetrievalResult rg = fier::cuda::run_policy<fier::RetrievalResult>(pol, q, KP, V, st);
            const double err = fier::relative_l2_error(rg.output, rw.output);
            report(same_indices(rw.selection, rg.selection) && err < 1e-2 &&
                       rw.bytes_loaded_for_estimation == rg.bytes_loaded_for_estimation,
                   std::string("run_policy ") + fier::policy_name(pol.kind), "rel l2 " + std::to_string(err));
        }
    }
    {  // the fier branch's side-state lookup and budget check (retrieval.hpp:93-97, :171)
        fier::BudgetPolicy p = pols[2];
        p.group_size = 64;
        report(error_of([&] { fier::cuda::select_for_policy<fier::PolicySelection>(p, q, KP, st); }) ==
                   "run_policy: missing packed keys in side state",
               "select_for_policy missing side state");
        p = pols[2];
        p.budget = l + 1;
        report(error_of([&] { fier::cuda::select_for_policy<fier::PolicySelection>(p, q, KP, st); }) ==
                   "run_policy: budget out of range for cache",
               "select_for_policy budget range");
    }
    // fier_attend on the reference's PackedKeys (fp64 in-memory (s, z)) and types
    {
        const fier::PackedKeys pk = fier::quantize(KP, fier::GroupSpec{g});
        const fier::RetrievalResult rw = fier::fier_attend(q, KP, V, pk, n);
        const fier::RetrievalResult rg = fier::cuda::fier_attend<fier::RetrievalResult>(q, KP, V, pk, n);
        const double err = fier::relative_l2_error(rg.output, rw.output);
        report(same_indices(rw.selection, rg.selection) && err < 1e-2 &&
                   rw.bytes_loaded_for_estimation == rg.bytes_loaded_for_estimation,
               "fier_attend", "rel l2 " + std::to_string(err));
    }
    // ---- load_ratio_fier ----
    {
        bool ok = true;
        for (std::size_t ll : {1u, 33u, 4096u, 100000u})
            for (std::size_t gg : {1u, 7u, 32u, 128u, 256u}) {
                const fier::LoadRatio a = fier::load_ratio_fier(ll, gg);
                const fier::LoadRatio b = fier::cuda::load_ratio_fier<fier::LoadRatio>(ll, gg);
                ok &= a.numerator_bits == b.numerator_bits && a.denominator_bits == b.denominator_bits &&
                      a.formula == b.formula && a.ratio() == b.ratio();
            }
        report(ok, "load_ratio_fier");
    }
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASS", g_fail);
    return g_fail ? 1 : 0;
}
