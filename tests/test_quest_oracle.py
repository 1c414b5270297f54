"""Quest page retrieval (baselines.hpp): the C restatement in
oracle/fier_oracle.c pinned against the reference itself (oracle/_ref), on CPU."""
import numpy as np
import pytest


@pytest.mark.parametrize("l, d, L, n", [(1000, 128, 16, 110), (77, 11, 8, 20), (64, 8, 64, 64), (513, 32, 16, 17),
                                        (300, 64, 1, 31), (4096, 128, 16, 455)])
@pytest.mark.parametrize("variant", ["sum", "max"])
def test_quest_port_matches_reference(port, ref, l, d, L, n, variant):
    rng = np.random.default_rng(l + d + L)
    K = rng.standard_normal((l, d))
    K[rng.integers(0, l, 8)] *= 6.0  # some pages stand out
    q = rng.standard_normal(d)
    kmax, kmin = port.page_summaries(K, L)
    rmax, rmin = ref.page_summaries(K, L)
    np.testing.assert_array_equal(kmax, rmax)
    np.testing.assert_array_equal(kmin, rmin)
    ps = port.quest_page_scores(q, kmax, kmin, variant)
    np.testing.assert_array_equal(ps, ref.quest_page_scores(q, K, L, variant))
    np.testing.assert_array_equal(port.select_by_page_scores(ps, l, L, n), ref.select_by_page_scores(ps, l, L, n))
    np.testing.assert_array_equal(port.quest_select(q, K, L, n, variant), ref.quest_select(q, K, L, n, variant))


def test_page_selection_ties_and_short_page(port, ref):
    """Equal page scores rank by page index; the short last page can be taken whole."""
    l, L = 70, 16  # pages of 16, 16, 16, 16, 6
    ps = np.array([1.0, 3.0, 3.0, 0.5, 3.0])
    for n in (1, 6, 16, 22, 38, 48, 54, 70):
        np.testing.assert_array_equal(port.select_by_page_scores(ps, l, L, n), ref.select_by_page_scores(ps, l, L, n))


@pytest.mark.parametrize("l, d, g, L, n", [(1000, 128, 32, 16, 110), (77, 11, 3, 8, 20), (640, 64, 128, 32, 100)])
def test_quest_quantized_port_matches_reference(port, ref, l, d, g, L, n):
    rng = np.random.default_rng(l * d)
    K = rng.standard_normal((l, d))
    q = rng.standard_normal(d)
    buf = ref.quantize_fier(K, g)
    est = ref.approx_scores_fier(q, buf)
    sel = port.select_by_page_scores(port.page_mean(est, L), l, L, n)
    np.testing.assert_array_equal(sel, ref.quest_select_quantized(q, buf, L, n))
