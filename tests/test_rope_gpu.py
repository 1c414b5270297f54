"""RoPE fused into the decode step (fier_decode_step_ex) against a
float64 restatement of the rotation followed by the reference's own pipeline.

Rotation: frequency i < rd/2 turns by pos * base^(-2i/rd); rotate_half pairs (i, i + rd/2)
(NeoX / Llama) or interleaved pairs (2i, 2i + 1) (GPT-J); channels >= rd pass through.
The rotation is evaluated in fp32 and rounded to the cache dtype (include/fier_cuda.h).
Checks: the stored k row is within two ulps of the float64 rotation and bit-exact with the
fp32 evaluation (rope32); the index is bit-exact for the stored cache; scores of the rotated
q within 1e-3 of approx_scores; exact Top-n on the GPU's scores; attention within 1e-2 of
gather_attention -- on the one-launch (MHA) and the separate-kernel (GQA, fp32) paths.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TDT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}
ULP = {"f32": 2.0 ** -23, "f16": 2.0 ** -10, "bf16": 2.0 ** -7}


def rope32(x, pos, base, rd, interleaved, dtype):
    """The kernels' arithmetic: cos/sin of the float64 angle rounded to fp32, one fp32
    product and one fused multiply-add per channel, rounded to the cache dtype."""
    x = x.astype(np.float32)
    i = np.arange(rd // 2, dtype=np.float64)
    ang = pos * base ** (-2.0 * i / rd)
    c, s = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)

    def fma(a, b, t):  # fmaf(a, b, t): exact in float64 for fp32 inputs, one rounding
        return (a.astype(np.float64) * b.astype(np.float64) + t.astype(np.float64)).astype(np.float32)

    y = x.copy()
    if interleaved:
        a, b = x[..., 0:rd:2], x[..., 1:rd:2]
        y[..., 0:rd:2] = fma(a, c, -(b * s))
        y[..., 1:rd:2] = fma(b, c, a * s)
    else:
        h = rd // 2
        a, b = x[..., :h], x[..., h:rd]
        y[..., :h] = fma(a, c, -(b * s))
        y[..., h:rd] = fma(b, c, a * s)
    return torch.from_numpy(y).to(TDT[dtype]).double().numpy()


def rope64(x, pos, base, rd, interleaved):
    """x: [..., d] float64."""
    y = x.copy()
    i = np.arange(rd // 2, dtype=np.float64)
    ang = pos * base ** (-2.0 * i / rd)
    c, s = np.cos(ang), np.sin(ang)
    if interleaved:
        a, b = x[..., 0:rd:2], x[..., 1:rd:2]
        y[..., 0:rd:2] = a * c - b * s
        y[..., 1:rd:2] = b * c + a * s
    else:
        h = rd // 2
        a, b = x[..., :h], x[..., h:rd]
        y[..., :h] = a * c - b * s
        y[..., h:rd] = b * c + a * s
    return y


def score_err(gpu, ref):
    return np.max(np.abs(gpu - ref) / np.maximum(1.0, np.abs(ref)))


@pytest.mark.parametrize("B,Hq,Hkv,d,dtype,rd,inter,pos", [
    (1, 4, 4, 128, "bf16", 128, False, 2500),    # fused step, full rotation (Llama)
    (2, 3, 3, 128, "f16", 64, True, 3999),      # fused step, partial interleaved (GPT-J)
    (1, 4, 4, 128, "bf16", 128, False, 65600),  # fused, large angles (fp64 on the host)
    (1, 8, 2, 128, "bf16", 128, False, 1800),   # GQA: rope kernel + separate kernels
    (2, 2, 2, 64, "f32", 32, False, 700),       # fp32: separate kernels
])
def test_rope_step_matches_reference(cuda, port, B, Hq, Hkv, d, dtype, rd, inter, pos):
    import paper_2508_08256_b200 as F
    torch.manual_seed(pos)
    dt, g, base, n = TDT[dtype], 32, 10000.0, 97
    cap = pos + 50
    layer = F.DecodeLayer(B, Hq, Hkv, cap, d, g, dtype=dt, device=cuda)
    layer.K.copy_(torch.randn(B, Hkv, cap, d, device=cuda).to(dt))
    layer.V.copy_(torch.randn(B, Hkv, cap, d, device=cuda).to(dt))
    layer.prefill(pos)
    q = torch.randn(B, Hq, d, device=cuda).to(dt)
    kn = torch.randn(B, Hkv, d, device=cuda).to(dt)
    vn = torch.randn(B, Hkv, d, device=cuda).to(dt)
    ld = pos + 1 + (-(pos + 1)) % 32
    scores = torch.empty(B, Hq, ld, device=cuda)
    out, sel = layer.step(q, kn, vn, pos, n, scores_out=scores, rope=(base, rd, inter))
    torch.cuda.synchronize()
    Kc, Vc = layer.K.double().cpu().numpy(), layer.V.double().cpu().numpy()
    k64 = rope64(kn.double().cpu().numpy(), pos, base, rd, inter)
    np.testing.assert_allclose(Kc[:, :, pos], k64, rtol=2 * ULP[dtype], atol=1e-6)  # the rotation itself
    np.testing.assert_array_equal(Kc[:, :, pos], rope32(kn.cpu().float().numpy(), pos, base, rd, inter, dtype))
    np.testing.assert_array_equal(Vc[:, :, pos], vn.double().cpu().numpy())  # v is not rotated
    q_rot = rope32(q.cpu().float().numpy(), pos, base, rd, inter, dtype)  # what the step scores with
    sel_np, out_np, sc = sel.cpu().numpy(), out.cpu().numpy(), scores.cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            kv = h // (Hq // Hkv)
            buf = port.quantize_fier(Kc[b, kv, :pos + 1], g)
            assert layer.pk.to_fier(b, kv) == buf
            ref_scores = port.approx_scores_fier(q_rot[b, h], buf)
            assert score_err(sc[b, h, :pos + 1], ref_scores) <= 1e-3
            np.testing.assert_array_equal(sel_np[b, h], port.topk(sc[b, h, :pos + 1].astype(np.float64), n))
            ref_out = port.gather_attention(q_rot[b, h], Kc[b, kv, :pos + 1], Vc[b, kv, :pos + 1],
                                            sel_np[b, h].astype(np.int64))
            assert port.relative_l2_error(out_np[b, h], ref_out) < 1e-2


def test_rope_rejects_bad_parameters(cuda):
    import paper_2508_08256_b200 as F
    layer = F.DecodeLayer(1, 2, 2, 64, 128, 32, dtype=torch.bfloat16, device=cuda)
    layer.prefill(10)
    q = torch.zeros(1, 2, 128, device=cuda, dtype=torch.bfloat16)
    for bad in [(10000.0, 3, False), (10000.0, 256, False), (0.0, 64, False)]:
        with pytest.raises(ValueError):
            layer.step(q, q, q, 10, 4, rope=bad)
