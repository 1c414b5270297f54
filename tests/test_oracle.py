"""Pin the oracle (oracle/fier_oracle.c) before trusting it.

Checks the C restatement against
  * the reference's own known-answer tests (tests/golden/kats.json, restated
    from test_io.cpp, test_quant1bit.cpp, test_kvcore.cpp, acceptance_main.cpp),
  * golden fixtures produced by the reference itself (tests/golden/*.npz,
    tests/golden/make_golden.py over oracle/_ref/libfier_ref.so),
  * the reference library directly on fresh random inputs (where built).
CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_golden

KATS = json.load(open(os.path.join(GOLDEN, "kats.json")))


def test_half_narrowing_kats(port):
    for value, pattern in KATS["half_narrow"]:
        assert port.double_to_half(value) == pattern, value
    special = {"nan": math.nan, "inf": math.inf, "-inf": -math.inf}
    for name, pattern in KATS["half_narrow_special"]:
        assert port.double_to_half(special[name]) == pattern


def test_half_widening_kats(port):
    for pattern, value in KATS["half_widen"]:
        assert port.half_to_double(pattern) == value
    assert math.isinf(port.half_to_double(0x7C00)) and port.half_to_double(0xFC00) < 0
    assert math.isnan(port.half_to_double(0x7E00))
    assert math.copysign(1.0, port.half_to_double(0x8000)) < 0


def test_every_half_pattern_round_trips(port):
    # test_io.cpp:88-98
    for h in range(0x10000):
        x = port.half_to_double(h)
        if math.isnan(x):
            assert math.isnan(port.half_to_double(port.double_to_half(x)))
        else:
            assert port.double_to_half(x) == h


def test_quantizer_kats(port):
    for case in KATS["quantize_columns"]:
        K = np.array(case["col"], float).reshape(-1, 1)
        cw, s, z = port.quantize(K, case["g"])
        assert s[0] == case["s"] and z[0] == case["z"], case["what"]
        bits = [int((cw[t] >> 0) & 1) for t in range(K.shape[0])]
        assert bits == case["bits"], case["what"]


def test_single_token_score_kat(port):
    c = KATS["single_token_score"]
    K = np.array(c["K"], float)
    buf = port.quantize_fier(K, c["g"])
    (l, d, g), cw, s, z = port.parse(buf)
    assert port.approx_scores_packed(c["q"], l, d, g, cw, s, z)[0] == c["score"]


def test_topk_kats(port):
    for c in KATS["topk"]:
        assert list(port.topk(c["scores"], c["k"])) == c["sel"], c["what"]
    with pytest.raises(ValueError):
        port.topk([1.0, 2.0], 0)
    with pytest.raises(ValueError):
        port.topk([1.0, 2.0], 3)


def test_payload_kats(port):
    from fractions import Fraction
    for c in KATS["payload"]:
        p = port.lib.fo_payload_bytes(c["l"], c["d"], c["g"])
        assert p == c["payload"]
        assert Fraction(p, c["l"] * c["d"] * 2) == Fraction(*c["ratio"])


@pytest.mark.parametrize("name", golden_cases())
def test_port_matches_reference_golden(port, name):
    c = load_golden(name)
    group = c["hq"] // c["hkv"]
    for h in range(c["hkv"]):
        assert port.quantize_fier(c["K"][h].astype(np.float64), c["g"]) == c["fier_list"][h]
    for h in range(c["hq"]):
        kv = h // group
        q = c["Q"][h].astype(np.float64)
        est = port.approx_scores_fier(q, c["fier_list"][kv])
        np.testing.assert_array_equal(est, c["scores"][h])  # bit-exact fp64
        sel = port.topk(est, c["n"])
        np.testing.assert_array_equal(sel, c["sel"][h])
        out = port.gather_attention(q, c["K"][kv], c["V"][kv], sel)
        np.testing.assert_array_equal(out, c["out"][h])
        full = port.gather_attention(q, c["K"][kv], c["V"][kv], np.arange(c["l"]))
        np.testing.assert_array_equal(full, c["full"][h])
        assert port.lib.fo_payload_bytes(c["l"], c["d"], c["g"]) == c["bytes_loaded"][h]


def test_port_matches_reference_library_random(port, ref):
    rng = np.random.default_rng(123)
    for rep in range(25):
        l = int(rng.integers(1, 300))
        d = int(rng.integers(1, 70))
        g = int(rng.choice([1, 2, 3, 8, 32, 64, 100]))
        K = rng.standard_normal((l, d)) * rng.choice([1e-3, 1.0, 50.0])
        V = rng.standard_normal((l, d))
        q = rng.standard_normal(d)
        buf = ref.quantize_fier(K, g)
        assert port.quantize_fier(K, g) == buf
        cw_r, s_r, z_r = ref.quantize_inmem(K, g)
        cw_p, s_p, z_p = port.quantize(K, g)
        np.testing.assert_array_equal(cw_p, cw_r)
        np.testing.assert_array_equal(s_p, s_r)
        np.testing.assert_array_equal(z_p, z_r)
        est = ref.approx_scores_fier(q, buf)
        np.testing.assert_array_equal(port.approx_scores_fier(q, buf), est)
        n = int(rng.integers(1, l + 1))
        np.testing.assert_array_equal(port.topk(est, n), ref.topk(est, n))
        sel = ref.topk(est, n)
        np.testing.assert_array_equal(port.gather_attention(q, K, V, sel), ref.gather_attention(q, K, V, sel))


def test_oracle_rejects_like_reference(port, ref):
    K = np.ones((4, 3))
    K[1, 1] = np.nan
    with pytest.raises(ValueError):
        port.quantize(K, 2)
    with pytest.raises(ValueError, match="non-finite"):
        ref.quantize_fier(K, 2)
    with pytest.raises(ValueError, match="empty selection"):
        ref.gather_attention(np.ones(3), np.ones((4, 3)), np.ones((4, 3)), np.array([], np.int64))
    with pytest.raises(ValueError):
        port.gather_attention(np.ones(3), np.ones((4, 3)), np.ones((4, 3)), np.array([2, 1]))
