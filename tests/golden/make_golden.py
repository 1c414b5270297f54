"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every expected value here comes from the reference's own functions, compiled
from /root/reference/proj/include into oracle/_ref/libfier_ref.so:
  quantize + serialize_packed_keys   (quant1bit.hpp:65, io.hpp:197)
  approx_scores over parse_packed_keys (quant1bit.hpp:121, io.hpp:227)
  topk_oracle                         (core.hpp:134)
  gather_attention (scaled)           (core.hpp:152)
  fier_attend                         (retrieval.hpp:136)
  generate (planted_spikes)           (workload.hpp:128-191)

Inputs are stored as float32 arrays whose values are exactly representable in
the case's GPU dtype (bf16 / fp16 / fp32), so the GPU sees the same numbers the
reference saw after exact widening to fp64.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref  # noqa: E402


def to_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round to the named dtype (RNE) and return float32 holding those values."""
    x = np.asarray(x, np.float64)
    if dtype == "f32":
        return x.astype(np.float32)
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        f = x.astype(np.float32)
        u = f.view(np.uint32).astype(np.uint64)
        u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        return u.astype(np.uint32).view(np.float32)
    raise ValueError(dtype)


def make_case(ref: Ref, name, *, hq, hkv, l, d, g, n, dtype, seed, planted=False, scale=1.0,
              tweak=None):
    rng = np.random.default_rng(seed)
    K = np.zeros((hkv, l, d), np.float32)
    V = np.zeros((hkv, l, d), np.float32)
    Q = np.zeros((hq, d), np.float32)
    group = hq // hkv
    for h in range(hkv):
        if planted:
            # reference workload generator: spike keys whose exact logit is the gain
            k, v, qs = ref.generate(l, d, planted=True, spike_count=4, spike_gain=50.0,
                                    seed=seed * 131 + h, query_count=group)
            K[h], V[h] = to_dtype(k, dtype), to_dtype(v, dtype)
            Q[h * group:(h + 1) * group] = to_dtype(qs, dtype)
        else:
            K[h] = to_dtype(rng.standard_normal((l, d)) * scale, dtype)
            V[h] = to_dtype(rng.standard_normal((l, d)), dtype)
    if not planted:
        Q[:] = to_dtype(rng.standard_normal((hq, d)), dtype)
    if tweak:
        tweak(K, V, Q)

    fier = [ref.quantize_fier(K[h].astype(np.float64), g) for h in range(hkv)]
    scores = np.zeros((hq, l))
    sel = np.zeros((hq, n), np.int64)
    out = np.zeros((hq, d))
    full = np.zeros((hq, d))
    bytes_loaded = np.zeros(hq, np.int64)
    for h in range(hq):
        kv = h // group
        Kd, Vd, q = K[kv].astype(np.float64), V[kv].astype(np.float64), Q[h].astype(np.float64)
        s_, o_, est, nb = ref.fier_attend_fier(q, Kd, Vd, fier[kv], n)
        sel[h], out[h], scores[h], bytes_loaded[h] = s_, o_, est, nb
        assert np.array_equal(est, ref.approx_scores_fier(q, fier[kv]))
        assert np.array_equal(s_, ref.topk(est, n))
        full[h] = ref.gather_attention(q, Kd, Vd, np.arange(l), True)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        hq=hq, hkv=hkv, l=l, d=d, g=g, n=n, dtype=dtype, K=K, V=V, Q=Q,
        fier=np.concatenate([np.frombuffer(f, np.uint8) for f in fier]),
        fier_len=len(fier[0]), scores=scores, sel=sel, out=out, full=full,
        bytes_loaded=bytes_loaded)
    print(f"{name}: hq={hq} hkv={hkv} l={l} d={d} g={g} n={n} {dtype}")


def signed_zero_tweak(K, V, Q):
    # quant1bit.hpp:85-89 first-seen ties: {-0,+0} -> z = -0 (0x8000), {+0,-0} -> +0
    K[0, 0:2, 0] = [-0.0, 0.0]
    K[0, 0:2, 1] = [0.0, -0.0]
    K[0, 2:32, 0:2] = 0.0
    K[0, 32:64, 2] = 7.0          # constant group -> s == 0, all bits 1 (:96)
    K[0, 64:66, 3] = [1.0, 1.0]   # duplicate extremes


def tie_tweak(K, V, Q):
    # duplicate key rows -> equal estimated scores -> lower index wins (core.hpp:139-142)
    for h in range(K.shape[0]):
        K[h, 40] = K[h, 7]
        K[h, 41] = K[h, 7]
        K[h, 90] = K[h, 3]


def main():
    ref = Ref()
    make_case(ref, "odd_d11_g3", hq=1, hkv=1, l=21, d=11, g=3, n=5, dtype="f32", seed=1)
    make_case(ref, "short_group_d24", hq=2, hkv=2, l=100, d=24, g=32, n=17, dtype="f16", seed=2)
    make_case(ref, "g1_lossless", hq=1, hkv=1, l=64, d=8, g=1, n=8, dtype="bf16", seed=3)
    make_case(ref, "gqa_d64", hq=4, hkv=2, l=257, d=64, g=32, n=40, dtype="bf16", seed=4)
    make_case(ref, "mha_d128", hq=2, hkv=2, l=1000, d=128, g=32, n=110, dtype="bf16", seed=5)
    make_case(ref, "c1_head_f32", hq=1, hkv=1, l=4096, d=128, g=32, n=512, dtype="f32", seed=6)
    make_case(ref, "g128_fp16", hq=1, hkv=1, l=700, d=128, g=128, n=64, dtype="f16", seed=7,
              scale=20.0)
    make_case(ref, "g256_short", hq=1, hkv=1, l=300, d=128, g=256, n=33, dtype="bf16", seed=8)
    make_case(ref, "planted_spikes", hq=4, hkv=1, l=2048, d=128, g=32, n=16, dtype="bf16",
              seed=9, planted=True)
    make_case(ref, "signed_zero", hq=1, hkv=1, l=96, d=32, g=32, n=9, dtype="f32", seed=10,
              tweak=signed_zero_tweak)
    make_case(ref, "score_ties", hq=2, hkv=1, l=128, d=64, g=32, n=20, dtype="bf16", seed=11,
              tweak=tie_tweak)
    make_case(ref, "single_token", hq=1, hkv=1, l=1, d=128, g=32, n=1, dtype="bf16", seed=12)
    make_case(ref, "full_budget", hq=1, hkv=1, l=77, d=128, g=32, n=77, dtype="bf16", seed=13)


if __name__ == "__main__":
    main()
