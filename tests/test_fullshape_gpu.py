"""Full-shape parity of the decode step (fier_decode_step through DecodeLayer.step) at the
BASELINE.json configurations, against the oracle on the same inputs:

  C1  32 MHA heads, d=128, l=4096, fp32, n=512          every head
  C3  Llama-3-8B GQA 32 q / 8 kv, l=131072, n=4096, bf16  sampled q heads (all 8 kv heads' index)
  C4  batch 32, GQA 32/8, l=32768, n=3604, bf16          sampled (sequence, q head) pairs

Bars (BASELINE.json north star): the appended index bit-exact (FIER bytes of quantize of the
grown cache, quant1bit.hpp:65-103, io.hpp:197-225); scores within 1e-3 of approx_scores over
the FIER round trip (quant1bit.hpp:121-140); the selection exactly topk_oracle of the GPU's
own scores (core.hpp:134-148) and, against topk_oracle of the reference's scores, recall
>= 0.999 with every disagreement a tie within score tolerance; the output within 1e-2 of
gather_attention on the GPU's selection (core.hpp:152-179).  C2 is
tests/test_kernels_gpu.py::test_c2_shape_step_properties.
"""
import numpy as np
import pytest
import torch

from conftest import SCORE_TOL, check_selection

pytestmark = pytest.mark.gpu
OUT_TOL = 1e-2


def score_err(gpu, ref):
    return np.max(np.abs(gpu - ref) / np.maximum(1.0, np.abs(ref)))


def run(cuda, B, Hq, Hkv, L, n, dtype, seed):
    import paper_2508_08256_b200 as F
    torch.manual_seed(seed)
    d, g, pos = 128, 32, L - 1
    layer = F.DecodeLayer(B, Hq, Hkv, L, d, g, dtype=dtype, device=cuda)
    layer.K.copy_(torch.randn(B, Hkv, L, d, device=cuda).to(dtype))
    layer.V.copy_(torch.randn(B, Hkv, L, d, device=cuda).to(dtype))
    layer.prefill(pos)
    q = torch.randn(B, Hq, d, device=cuda).to(dtype)
    kn = torch.randn(B, Hkv, d, device=cuda).to(dtype)
    vn = torch.randn(B, Hkv, d, device=cuda).to(dtype)
    scores = torch.empty(B, Hq, L + (-L) % 32, device=cuda)
    flag = torch.zeros(1, dtype=torch.int32, device=cuda)
    out, sel = layer.step(q, kn, vn, pos, n, scores_out=scores, nonfinite=flag)
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    assert torch.equal(layer.K[:, :, pos], kn) and torch.equal(layer.V[:, :, pos], vn)
    return layer, q, out, sel, scores


def check_pairs(port, layer, q, out, sel, scores, pairs, n):
    Hq, Hkv = q.shape[1], layer.Hkv
    L = layer.cap
    fier_of = {}
    for b, h in pairs:
        kv = h // (Hq // Hkv)
        K = layer.K[b, kv].double().cpu().numpy()
        V = layer.V[b, kv].double().cpu().numpy()
        if (b, kv) not in fier_of:
            buf = port.quantize_fier(K, layer.g)
            assert layer.pk.to_fier(b, kv) == buf, f"appended index not bit-exact (b={b}, kv={kv})"
            fier_of[(b, kv)] = buf
        qd = q[b, h].double().cpu().numpy()
        ref = port.approx_scores_fier(qd, fier_of[(b, kv)])
        got = scores[b, h, :L].cpu().numpy().astype(np.float64)
        assert score_err(got, ref) <= SCORE_TOL
        s = sel[b, h].cpu().numpy()
        np.testing.assert_array_equal(s, port.topk(got, n))
        check_selection(s, ref, n, port)
        want = port.gather_attention(qd, K, V, s.astype(np.int64))
        assert port.relative_l2_error(out[b, h].cpu().numpy().astype(np.float64), want) < OUT_TOL


def test_c1_full_shape_every_head(cuda, port):
    layer, q, out, sel, scores = run(cuda, 1, 32, 32, 4096, 512, torch.float32, seed=101)
    check_pairs(port, layer, q, out, sel, scores, [(0, h) for h in range(32)], 512)


def test_c3_full_shape_sampled_heads(cuda, port):
    layer, q, out, sel, scores = run(cuda, 1, 32, 8, 131072, 4096, torch.bfloat16, seed=103)
    check_pairs(port, layer, q, out, sel, scores, [(0, 0), (0, 5), (0, 14), (0, 23), (0, 31)], 4096)
    for kv in range(8):  # every kv head's grown index stays bit-exact (bits of the open group)
        K = layer.K[0, kv, 131072 - 64:].double().cpu().numpy()
        W = layer.pk.bits[0, kv, 131072 - 64:].cpu().numpy().view(np.uint32)
        ref = np.frombuffer(port.quantize_fier(K, 32), np.uint8)[18 + 64 * 128 // 32 * 4:]
        got = np.zeros(64 * 16, np.uint8)
        for t in range(64):
            got[16 * t:16 * t + 16] = W[t].view(np.uint8)
        assert np.array_equal(got, ref)


def test_c4_full_shape_sampled_pairs(cuda, port):
    layer, q, out, sel, scores = run(cuda, 32, 32, 8, 32768, 3604, torch.bfloat16, seed=104)
    check_pairs(port, layer, q, out, sel, scores, [(0, 0), (7, 3), (13, 17), (22, 30), (31, 31)], 3604)
