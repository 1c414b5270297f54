"""The drop-in boundary on the GPU: fp64 keys (the reference's own KeyCache type) through
the device packer, the reference's half-narrowing KATs and the exhaustive binary16 round
trip through the device packer (half.hpp:13-61, test_io.cpp:41-98), the decode step's
non-finite rejection (quant1bit.hpp:68, core.hpp:122), the exact fp64 Top-k, and the C++
drop-in compiled next to the reference's own headers (tests/cpp/ref_shim_test.cpp).
"""
import json
import os
import subprocess

import numpy as np
import pytest
import torch

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu


def fier():
    import paper_2508_08256_b200 as F
    return F


def kats():
    return json.load(open(os.path.join(GOLDEN, "kats.json")))


def z_half_bits(pk, g_count):
    """(s, z) binary16 bit patterns [B, H, G, d, 2] of a device index."""
    return pk.params[:, :, :g_count].contiguous().cpu().numpy().view(np.uint16)


def test_fp64_keys_pack_bit_exact_vs_reference(cuda, port, ref):
    """quantize of fp64 keys that fp32 cannot represent: FIER bytes identical to the
    reference's quantize (the narrowing the round-1 drop-in did changed ~21 bytes)."""
    F = fier()
    rng = np.random.default_rng(5)
    for l, d, g, scale in [(4096, 128, 32, 1.0), (1000, 64, 7, 3.0), (333, 24, 128, 1e-3), (200, 11, 1, 5e4)]:
        K = rng.standard_normal((l, d)) * scale
        pk = F.quantize(torch.from_numpy(K).to(cuda), g)
        assert pk.to_fier() == ref.quantize_fier(K, g), (l, d, g, scale)


def test_half_narrowing_kats_through_device_packer(cuda):
    """The reference's 34 narrowing KATs (test_io.cpp:41-86) as constant fp64 groups: the
    device packer's z (and s of the symmetric groups) carry exactly the KAT patterns,
    including >= 65520 -> inf, subnormals and ties to even."""
    F = fier()
    cases = kats()["half_narrow"]
    vals = np.array([v for v, _ in cases], np.float64)
    pats = np.array([p for _, p in cases], np.uint16)
    d = len(vals)
    K = np.zeros((4, d))
    K[0] = K[1] = vals                 # constant group: z = v, s = 0
    K[2], K[3] = vals, -vals           # symmetric group: z = 0 (sign per first-seen), s = |v|
    pk = F.quantize(torch.from_numpy(K).to(cuda), 2)
    P = z_half_bits(pk, 2)[0, 0]       # [G=2, d, (s, z)]
    np.testing.assert_array_equal(P[0, :, 1], pats)
    assert np.all(P[0, :, 0] == 0)
    np.testing.assert_array_equal(P[1, :, 0], pats & 0x7FFF)
    bits = pk.bits[0, 0, :4].cpu().numpy().view(np.uint32)
    W = (d + 31) // 32
    for t in range(2):  # s == 0: every code bit is +1 (quant1bit.hpp:95-96)
        for j in range(d):
            assert (bits[t, j // 32] >> (j % 32)) & 1


def test_half_round_trip_exhaustive_through_device_packer(cuda):
    """Every finite binary16 pattern h, widened exactly (half_to_double) and packed as a
    constant fp64 group, comes back as z == h (test_io.cpp:88-98 through the device)."""
    F = fier()
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    fin = h[(h & 0x7C00) != 0x7C00]
    vals = fin.view(np.float16).astype(np.float64)
    H = -(-fin.size // 1024)
    K = np.zeros((1, H, 2, 1024))
    flat = np.zeros(H * 1024)
    flat[:fin.size] = vals
    K[0, :, 0, :] = K[0, :, 1, :] = flat.reshape(H, 1024)
    pk = F.quantize(torch.from_numpy(K).to(cuda), 2)
    z = pk.params[0, :, 0, :, 1].contiguous().cpu().numpy().view(np.uint16).reshape(-1)[:fin.size]
    np.testing.assert_array_equal(z, fin)


def test_fp64_append_matches_one_shot(cuda, ref):
    """fier_append on an fp64 cache re-packs the open group bit-exactly."""
    F = fier()
    rng = np.random.default_rng(8)
    l, d, g, cap = 300, 64, 32, 320
    K = torch.from_numpy(rng.standard_normal((cap, d))).to(cuda)
    V = torch.zeros_like(K)
    pk = F.quantize(K, g, tokens=270)
    for pos in range(270, l):
        kn = torch.from_numpy(rng.standard_normal(d)).to(cuda)
        F.append_token(K, V, kn, kn, pos, pk)
    pk.tokens = l
    assert pk.to_fier() == ref.quantize_fier(K[:l].cpu().numpy(), g)


def test_f64_rejected_outside_the_packer(cuda):
    F = fier()
    q = torch.zeros(128, dtype=torch.float64, device=cuda)
    pk = F.quantize(torch.zeros(64, 128, dtype=torch.float64, device=cuda))
    with pytest.raises(ValueError, match="unsupported dtype"):
        F.approx_scores(q, pk)


@pytest.mark.parametrize("hq,hkv,dtype,separate", [(4, 4, torch.bfloat16, False), (4, 4, torch.bfloat16, True),
                                                   (8, 2, torch.bfloat16, False), (4, 4, torch.float32, False),
                                                   (4, 2, torch.float16, False)])
def test_decode_step_flags_nonfinite_inputs(cuda, hq, hkv, dtype, separate):
    """A non-finite appended key sets FIER_NONFINITE_KEY ("quantize: non-finite key entry",
    quant1bit.hpp:68); a non-finite query FIER_NONFINITE_QUERY ("softmax: non-finite logit",
    core.hpp:122); finite inputs leave the word 0.  One-launch and separate-kernel paths."""
    F = fier()
    B, d, cap, pos, n = 1, 128 if hq != 4 or hkv != 2 else 40, 1024, 700, 64
    layer = F.DecodeLayer(B, hq, hkv, cap, d, 32, dtype=dtype, device=cuda)
    layer.K.copy_(torch.randn(B, hkv, cap, d, device=cuda).to(dtype))
    layer.V.copy_(torch.randn(B, hkv, cap, d, device=cuda).to(dtype))
    layer.prefill(pos)
    q = torch.randn(B, hq, d, device=cuda).to(dtype)
    kn = torch.randn(B, hkv, d, device=cuda).to(dtype)
    for bad_q, bad_k, want, msg in [(False, False, 0, None),
                                    (False, True, 1, "quantize: non-finite key entry"),
                                    (True, False, 2, "softmax: non-finite logit"),
                                    (True, True, 3, "quantize: non-finite key entry")]:
        qq, kk = q.clone(), kn.clone()
        if bad_q:
            qq[0, hq - 1, 5] = float("nan")
        if bad_k:
            kk[0, hkv - 1, 7] = float("inf")
        flag = torch.zeros(1, dtype=torch.int32, device=cuda)
        layer.step(qq, kk, kk, pos, n, nonfinite=flag, separate=separate)
        torch.cuda.synchronize()
        assert int(flag.item()) == want
        if msg:
            with pytest.raises(ValueError, match=msg):
                F.raise_nonfinite(flag)
        else:
            F.raise_nonfinite(flag)
    layer.K[:, :, pos].copy_(kn)  # leave the cache finite


def test_topk_f64_exact_on_doubles(cuda, port):
    """topk_oracle on float64 scores (fier_topk_f64): exact where fp32 rounding would merge
    distinct doubles, with exact ties and +-0 (core.hpp:134-148)."""
    F = fier()
    rng = np.random.default_rng(3)
    s = rng.standard_normal((3, 20000))
    s[0, ::3] = 1.0 + (np.arange(0, 20000, 3) % 7) * 1e-12
    s[1, ::5] = 0.0
    s[1, 1::5] = -0.0
    s[2, ::2] = 2.5
    for k in (1, 17, 4000, 6667, 19999, 20000):
        got = F.topk_oracle(torch.from_numpy(s).to(cuda), k).cpu().numpy()
        for r in range(3):
            np.testing.assert_array_equal(got[r], port.topk(s[r], k))


def test_ref_shim_against_reference(cuda):
    """include/fier_cuda.hpp compiled next to the reference's headers with the reference's own
    types (tests/cpp/ref_shim_test.cpp): quantize byte-identical on fp64 keys, topk_oracle /
    exact_scores exact, select_for_policy / run_policy / fier_attend / load_ratio_fier."""
    from paper_2508_08256_b200 import build as b
    exe = b.REF_SHIM_BIN
    if not os.path.exists(exe):
        exe = b.build_ref_shim_test()
    if not exe:
        pytest.skip("reference headers were never available to build tests/cpp/ref_shim_test")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout + r.stderr
