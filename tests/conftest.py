"""Shared test fixtures.  `-m gpu` tests need a B200 and the in-tree CUDA library;
everything else runs on CPU (oracle vs golden vectors, host logic, C-ABI surface)."""
import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfier_cuda.so")


def golden_cases():
    return sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    c = {k: z[k] for k in z.files}
    for k in ("hq", "hkv", "l", "d", "g", "n", "fier_len"):
        c[k] = int(c[k])
    c["dtype"] = str(c["dtype"])
    fl = c["fier_len"]
    c["fier_list"] = [c["fier"][i * fl:(i + 1) * fl].tobytes() for i in range(c["hkv"])]
    return c


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference headers absent)")
    return Ref()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_08256_b200 import _lib
    _lib.load()  # raises if the library is missing: no fallback
    return torch.device("cuda:0")


SCORE_TOL = 1e-3  # |gpu - ref| <= 1e-3 * max(1, |ref|)  (BASELINE.json north star)


def check_selection(gpu_sel, ref_scores, n, port, min_recall=0.999):
    """The north-star selection bar against topk_oracle of the REFERENCE's scores: every
    index the two selections disagree on lies within score tolerance of the reference's
    threshold (a tie within 1e-3), and recall >= min_recall (evalharness.hpp:25-34)."""
    ref_sel = port.topk(ref_scores, n)
    T = ref_scores[ref_sel].min()
    diff = np.setxor1d(np.asarray(gpu_sel, np.int64), ref_sel)
    tol = 2 * SCORE_TOL * np.maximum(1.0, np.abs(ref_scores[diff]))
    far = diff[np.abs(ref_scores[diff] - T) > tol]
    assert far.size == 0, f"selection differs beyond score tolerance at {far[:8]} (T={T})"
    rec = port.recall(np.asarray(gpu_sel, np.int64), ref_sel)
    assert rec >= min_recall or diff.size <= 2, f"recall {rec} < {min_recall}"
    return rec
