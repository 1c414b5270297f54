"""Recall / margin sweep on the GPU (csrc/harness.cu, harness.py)
against the reference's own evaluation harness (evalharness.hpp, compiled in oracle/_ref).

Bars: exact_scores within 1e-12 relative (fp64 dot products; summation order differs);
margin_and_errors within 1e-9 relative of the reference's; run_trial recall within the
boundary swaps fp32 estimates allow (2 tokens, or one page, per budget), out_err within 2e-3
(5% for the policies that select on fp32 estimates, whose boundary swaps need not show in recall) and max_err within 1e-3 of the reference's
fp64 numbers.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def H():
    from paper_2508_08256_b200 import harness
    return harness


@pytest.mark.parametrize("B, Hq, Hkv, l, d, dtype", [(1, 4, 4, 1000, 128, torch.float32),
                                                    (2, 8, 2, 333, 64, torch.bfloat16)])
def test_exact_scores(cuda, port, B, Hq, Hkv, l, d, dtype):
    torch.manual_seed(l)
    K = torch.randn(B, Hkv, l, d, device=cuda).to(dtype)
    q = torch.randn(B, Hq, d, device=cuda).to(dtype)
    s64, s32 = H().exact_scores(q, K)
    Kc, qc = K.double().cpu().numpy(), q.double().cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            want = port.exact_scores(qc[b, h], Kc[b, h // (Hq // Hkv)])
            got = s64[b, h].cpu().numpy()
            assert np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) <= 1e-12
            np.testing.assert_array_equal(s32[b, h].cpu().numpy(), got.astype(np.float32))


@pytest.mark.parametrize("l, d, g, k", [(1000, 128, 32, 110), (4096, 64, 32, 455), (77, 11, 3, 5)])
def test_margin_and_errors(cuda, ref, l, d, g, k):
    import paper_2508_08256_b200 as F
    rng = np.random.default_rng(l + k)
    K = rng.standard_normal((l, d)).astype(np.float32)
    q = rng.standard_normal(d).astype(np.float32)
    Kt, qt = torch.from_numpy(K).to(cuda), torch.from_numpy(q).to(cuda)
    pk = F.quantize(Kt, g)
    s64, s32 = H().exact_scores(qt, Kt)
    est = F.approx_scores(qt, pk)
    got = H().margin_and_errors(s64, s32, est, k).cpu().numpy()
    want = ref.margin_and_errors(q.astype(np.float64), K.astype(np.float64), pk.to_fier(), k)
    # est is the GPU's fp32 estimate (<= 1e-3 of the reference's): the error sums follow it
    np.testing.assert_allclose(got[0], want[0], rtol=1e-9, atol=1e-12)  # margin: exact scores only
    np.testing.assert_allclose(got[1:], want[1:], rtol=2e-3, atol=1e-3)


def test_overlap_fraction(cuda, port):
    torch.manual_seed(1)
    a = torch.randperm(1000, device=cuda)[:300].sort().values.int().view(1, -1)
    b = torch.randperm(1000, device=cuda)[:200].sort().values.int().view(1, -1)
    got = H().overlap_fraction(a, b).item()
    want = len(set(a.cpu().numpy().ravel()) & set(b.cpu().numpy().ravel())) / 200
    assert got == want


@pytest.mark.parametrize("l, d, nq, g, L, budgets", [(1000, 128, 3, 32, 16, [32, 110, 500, 1000]),
                                                     (513, 64, 2, 32, 16, [17, 100, 513])])
def test_run_trial_matches_reference(cuda, ref, l, d, nq, g, L, budgets):
    rng = np.random.default_rng(l * nq)
    K = rng.standard_normal((l, d)).astype(np.float32)
    V = rng.standard_normal((l, d)).astype(np.float32)
    Q = rng.standard_normal((nq, d)).astype(np.float32)
    Q[0] = K[rng.integers(0, l, 6)].sum(0)  # a query with planted matches
    t = H().run_trial(torch.from_numpy(K).to(cuda), torch.from_numpy(V).to(cuda), torch.from_numpy(Q).to(cuda),
                      budgets, group=g, page_size=L)
    cells, margins = ref.run_trial(K.astype(np.float64), V.astype(np.float64), Q.astype(np.float64), g, L, budgets)
    for pi, p in enumerate(("fier", "quest", "quest_quant", "oracle", "full")):
        for bi, n in enumerate(budgets):
            slack = (2.0 if p in ("fier", "oracle") else float(L)) / n
            dr = abs(t.cells[p]["recall"][bi] - cells[pi, bi, 0])
            assert dr <= slack + 1e-12, (p, n)
            # fier / quest_quant select on fp32 estimates: a swap at the estimate's own boundary
            # (invisible to recall when neither token is in the exact top-n) moves the sparse
            # output by a few percent of its (large, random-data) error
            tol = 0.05 * max(1.0, cells[pi, bi, 1]) if p in ("fier", "quest_quant") or dr > 1e-12 else 2e-3
            assert abs(t.cells[p]["out_err"][bi] - cells[pi, bi, 1]) <= tol, (p, n)
            assert abs(t.cells[p]["max_err"][bi] - cells[pi, bi, 2]) <= 1e-3 * max(1.0, cells[pi, bi, 2]), (p, n)
    for bi, n in enumerate(budgets):
        if n == l:
            assert np.isnan(t.margins[bi]) and np.isnan(margins[bi])
        else:
            np.testing.assert_allclose(t.margins[bi], margins[bi], rtol=1e-6, atol=1e-9)
