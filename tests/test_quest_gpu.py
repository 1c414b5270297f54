"""Quest page retrieval on the GPU (csrc/quest.cu) against the oracle
(oracle/fier_oracle.c, pinned to the reference in tests/test_quest_oracle.py) and the
compiled reference itself.

Bars: page summaries bit-exact (extrema of the stored keys); page scores within 1e-6
relative (fp64 evaluation stored as fp32); the selection bit-exact against
select_by_page_scores on the GPU's own page scores, and against the reference's
quest_select / quest_select_quantized end to end where page scores are well separated.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TDT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


def fier():
    import paper_2508_08256_b200 as F
    return F


def rel_err(gpu, ref):
    return float(np.max(np.abs(gpu - ref) / np.maximum(1.0, np.abs(ref))))


@pytest.mark.parametrize("B, Hq, Hkv, l, d, L, dtype", [
    (1, 4, 4, 1000, 128, 16, "bf16"), (2, 8, 2, 777, 64, 16, "f16"), (1, 2, 1, 77, 11, 8, "f32"),
    (1, 1, 1, 64, 8, 64, "f32"), (1, 2, 2, 300, 32, 1, "bf16"), (1, 1, 1, 10, 16, 32, "f32"),
])
@pytest.mark.parametrize("variant", ["sum", "max"])
def test_quest_select_matches_oracle(cuda, port, B, Hq, Hkv, l, d, L, dtype, variant):
    F = fier()
    torch.manual_seed(l + d + L)
    cap = l + 5
    K = torch.randn(B, Hkv, cap, d, device=cuda).to(TDT[dtype])
    q = torch.randn(B, Hq, d, device=cuda).to(TDT[dtype])
    ps = F.build_page_summaries(K, L, tokens=l)
    pscore = F.quest_page_scores(q, ps, variant).cpu().numpy()
    Kc, qc = K.double().cpu().numpy(), q.double().cpu().numpy()
    kmax, kmin = ps.max_vecs.double().cpu().numpy(), ps.min_vecs.double().cpu().numpy()
    for n in sorted({1, max(1, l // 9), l // 2 + 3, l}):
        sel = F.quest_select(q, K, ps, n, variant).cpu().numpy()
        for b in range(B):
            for h in range(Hq):
                kv = h // (Hq // Hkv)
                rmax, rmin = port.page_summaries(Kc[b, kv, :l], L)
                np.testing.assert_array_equal(kmax[b, kv], rmax)
                np.testing.assert_array_equal(kmin[b, kv], rmin)
                want = port.quest_page_scores(qc[b, h], rmax, rmin, variant)
                assert rel_err(pscore[b, h], want) <= 1e-6
                np.testing.assert_array_equal(
                    sel[b, h], port.select_by_page_scores(pscore[b, h].astype(np.float64), l, L, n))


def test_quest_select_reference_end_to_end(cuda, ref):
    """Planted pages (well separated scores): the GPU selection equals the reference's."""
    F = fier()
    rng = np.random.default_rng(3)
    l, d, L = 4096, 128, 16
    K = rng.standard_normal((l, d)).astype(np.float32)
    q = rng.standard_normal(d).astype(np.float32)
    for p in rng.choice(l // L, 40, replace=False):
        K[p * L + 3] += 4.0 * np.sign(q)  # these pages score far above the rest
    Kt, qt = torch.from_numpy(K).to(cuda), torch.from_numpy(q).to(cuda)
    ps = F.build_page_summaries(Kt, L)
    for variant in ("sum", "max"):
        for n in (16, 300, 640, 641, 1000):
            got = F.quest_select(qt, Kt, ps, n, variant).cpu().numpy()
            np.testing.assert_array_equal(got, ref.quest_select(q.astype(np.float64), K.astype(np.float64), L, n,
                                                                variant))


def test_page_selection_ties_short_page(cuda, ref):
    F = fier()
    l, L = 70, 16  # pages of 16, 16, 16, 16, 6
    ps = torch.tensor([1.0, 3.0, 3.0, 0.5, 3.0], device=cuda)
    for n in (1, 6, 16, 22, 38, 48, 54, 70):
        got = F.select_by_page_scores(ps, l, L, n).cpu().numpy()
        np.testing.assert_array_equal(got, ref.select_by_page_scores(ps.double().cpu().numpy(), l, L, n))


def test_page_selection_many_pages(cuda, port):
    """1M tokens, 16-token pages, 11% budget: 7209 ranked pages per row in one CTA."""
    F = fier()
    l, L, n = 1 << 20, 16, 115343
    torch.manual_seed(0)
    ps = torch.randn(2, (l + L - 1) // L, device=cuda)
    ps[0, 100:200] = ps[0, 100]  # exact ties
    sel = F.select_by_page_scores(ps, l, L, n).cpu().numpy()
    for r in range(2):
        np.testing.assert_array_equal(sel[r], port.select_by_page_scores(ps[r].double().cpu().numpy(), l, L, n))


@pytest.mark.parametrize("B, Hq, Hkv, l, d, g, L, n, dtype", [
    (1, 4, 4, 1000, 128, 32, 16, 110, "bf16"), (1, 8, 2, 2048, 128, 32, 16, 225, "f16"),
    (1, 1, 1, 77, 11, 3, 8, 20, "f32"),
])
def test_quest_select_quantized(cuda, port, ref, B, Hq, Hkv, l, d, g, L, n, dtype):
    F = fier()
    torch.manual_seed(l)
    K = torch.randn(B, Hkv, l, d, device=cuda).to(TDT[dtype])
    q = torch.randn(B, Hq, d, device=cuda).to(TDT[dtype])
    pk = F.quantize(K, g)
    sel = F.quest_select_quantized(q, pk, L, n).cpu().numpy()
    est = F.approx_scores(q, pk).cpu().numpy()
    qc = q.double().cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            kv = h // (Hq // Hkv)
            buf = pk.to_fier(b, kv)
            ref_means = port.page_mean(ref.approx_scores_fier(qc[b, h], buf), L)
            gpu_means = port.page_mean(est[b, h].astype(np.float64), L).astype(np.float32)
            assert rel_err(gpu_means, ref_means) <= 1e-3
            np.testing.assert_array_equal(sel[b, h], port.select_by_page_scores(gpu_means.astype(np.float64), l,
                                                                               L, n))


def test_quest_rejects_bad_parameters(cuda):
    F = fier()
    K = torch.randn(64, 16, device=cuda)
    with pytest.raises(ValueError, match="page size must be >= 1"):
        F.build_page_summaries(K, 0)
    ps = F.build_page_summaries(K, 16)
    with pytest.raises(ValueError, match="budget out of range"):
        F.quest_select(torch.randn(16, device=cuda), K, ps, 65)
