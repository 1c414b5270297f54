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
