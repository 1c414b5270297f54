// shim_test.cpp -- host C++ through include/fier_cuda.hpp (the drop-in for the reference's
// C++ API) on the sm_100a kernels.  Writes its inputs and outputs to argv[1]; the GPU test
// tests/test_capi.py::test_cpp_shim_matches_oracle checks them against the oracle.
#include <cstdio>
#include <fstream>

#include "fier_cuda.hpp"

namespace fc = fier::cuda;

static uint64_t g_state = 0x9E3779B97F4A7C15ull;
static double next_gauss() {  // deterministic, SplitMix64-driven Box-Muller (test data only)
    auto u = [] {
        uint64_t z = (g_state += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        return ((z >> 11) + 0.5) / 9007199254740992.0;
    };
    const double a = u(), b = u();
    return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
}

template <typename T>
static void put(std::ofstream& f, const std::vector<T>& v) {
    const uint64_t n = v.size();
    f.write(reinterpret_cast<const char*>(&n), 8);
    f.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(n * sizeof(T)));
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::size_t l = 1000, d = 128, g = 32, n = 77;
    fc::types::KeyCache K, V;
    K.data = fc::types::Matrix(l, d);
    V.data = fc::types::Matrix(l, d);
    std::vector<double> q(d);
    // fp32-representable inputs so the device copies are exact
    for (auto& x : K.data.v) x = (double)(float)next_gauss();
    for (auto& x : V.data.v) x = (double)(float)next_gauss();
    for (auto& x : q) x = (double)(float)next_gauss();
    const auto pk = fc::quantize(K, fc::types::GroupSpec{g});
    const auto est = fc::approx_scores(q, pk);
    const auto sel = fc::topk_oracle(est, n);
    const auto out = fc::gather_attention(q, K, V, sel);
    const auto rr = fc::fier_attend(q, K, V, pk, n);
    // error behaviour: the reference's require() messages
    std::string e1, e2;
    try {
        fc::topk_oracle(est, 0);
    } catch (const std::invalid_argument& e) {
        e1 = e.what();
    }
    try {
        fc::fier_select(q, pk, l + 1);
    } catch (const std::invalid_argument& e) {
        e2 = e.what();
    }
    // Quest (baselines.hpp): planted pages well above the rest, so the fp32 page scores rank
    // exactly like the reference's fp64 ones
    fc::types::KeyCache KQ;
    KQ.data = fc::types::Matrix(4096, d);
    for (auto& x : KQ.data.v) x = (double)(float)next_gauss();
    for (std::size_t p = 0; p < 4096 / 16; p += 7)
        for (std::size_t j = 0; j < d; ++j) {  // keep the entries fp32-representable
            double& x = KQ.data.row(p * 16 + 3)[j];
            x = (double)(float)(x + 4.0 * (q[j] > 0 ? 1 : -1));
        }
    const auto ps = fc::build_page_summaries(KQ, 16);
    const auto qs = fc::quest_select(q, KQ, ps, 300, fc::types::QuestVariant::sum_over_channels);
    const auto pkq = fc::quantize(KQ, fc::types::GroupSpec{g});
    const auto qq = fc::quest_select_quantized(q, pkq, 16, 300);
    std::ofstream f(argv[1], std::ios::binary);
    put(f, K.data.v);
    put(f, V.data.v);
    put(f, q);
    put(f, pk.code_words);
    put(f, pk.scales);
    put(f, pk.zeros);
    put(f, est.values);
    std::vector<int64_t> s(sel.indices.begin(), sel.indices.end());
    put(f, s);
    put(f, out);
    std::vector<int64_t> s2(rr.selection.indices.begin(), rr.selection.indices.end());
    put(f, s2);
    put(f, rr.output);
    put(f, std::vector<char>(e1.begin(), e1.end()));
    put(f, std::vector<char>(e2.begin(), e2.end()));
    put(f, KQ.data.v);
    put(f, ps.max_vecs.v);
    put(f, ps.min_vecs.v);
    put(f, std::vector<int64_t>(qs.indices.begin(), qs.indices.end()));
    put(f, std::vector<int64_t>(qq.indices.begin(), qq.indices.end()));
    std::printf("shim ok: payload %zu bytes\n", (size_t)rr.bytes_loaded_for_estimation);
    return 0;
}
