"""GPU parity of the one-launch decode step (csrc/step_fused.cu: append -> score ->
Top-n -> sparse attention in one cluster per (sequence, head)) against the oracle.

The fused path serves MHA layers with d = 128, 32 | g and 16-bit caches; the bars are
the same as for the separate kernels (tests/test_kernels_gpu.py): the appended index
bit-exact, scores within 1e-3 of approx_scores over the FIER round trip, the selection
exactly topk_oracle of the GPU's own scores, the output within 1e-2 of
gather_attention on that selection.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TDT = {"f16": torch.float16, "bf16": torch.bfloat16}
SCORE_TOL = 1e-3
OUT_TOL = 1e-2
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def score_err(gpu, ref):
    return np.max(np.abs(gpu - ref) / np.maximum(1.0, np.abs(ref)))


def run_step(cuda, B, H, cap, pos, n, g, dtype, seed=5, K=None, separate=False):
    import paper_2508_08256_b200 as F
    torch.manual_seed(seed)
    dt, d = TDT[dtype], 128
    layer = F.DecodeLayer(B, H, H, cap, d, g, dtype=dt, device=cuda)
    layer.K.copy_((torch.randn(B, H, cap, d, device=cuda) if K is None else K).to(dt))
    layer.V.copy_(torch.randn(B, H, cap, d, device=cuda).to(dt))
    layer.prefill(pos)
    q = torch.randn(B, H, d, device=cuda).to(dt)
    kn = torch.randn(B, H, d, device=cuda).to(dt) if K is None else layer.K[:, :, 0].clone()
    vn = torch.randn(B, H, d, device=cuda).to(dt)
    ld = pos + 1 + (-(pos + 1)) % 32
    scores = torch.empty(B, H, ld, device=cuda)
    out, sel = layer.step(q, kn, vn, pos, n, scores_out=scores, separate=separate)
    torch.cuda.synchronize()
    return layer, q, kn, vn, out, sel, scores


def check(port, layer, q, kn, out, sel, scores, pos, n, g, heads=None):
    B, H = q.shape[0], q.shape[1]
    Kc, Vc = layer.K.double().cpu().numpy(), layer.V.double().cpu().numpy()
    assert np.array_equal(Kc[:, :, pos], kn.double().cpu().numpy())
    sel_np, out_np, sc = sel.cpu().numpy(), out.cpu().numpy(), scores.cpu().numpy()
    for b in range(B):
        for h in (range(H) if heads is None else heads):
            buf = port.quantize_fier(Kc[b, h, :pos + 1], g)
            assert layer.pk.to_fier(b, h) == buf, "appended index not bit-exact"
            qd = q[b, h].double().cpu().numpy()
            ref_scores = port.approx_scores_fier(qd, buf)
            assert score_err(sc[b, h, :pos + 1], ref_scores) <= SCORE_TOL
            np.testing.assert_array_equal(sel_np[b, h], port.topk(sc[b, h, :pos + 1].astype(np.float64), n))
            ref_out = port.gather_attention(qd, Kc[b, h, :pos + 1], Vc[b, h, :pos + 1],
                                            sel_np[b, h].astype(np.int64))
            assert port.relative_l2_error(out_np[b, h], ref_out) < OUT_TOL


@pytest.mark.parametrize("B,H,cap,pos,n,g,dtype", [
    (1, 4, 64, 5, 3, 32, "bf16"),            # one CTA, one slab, short open group
    (2, 3, 9000, 8191, 900, 32, "bf16"),     # 8192 tokens over an 8-CTA cluster
    (1, 2, 40000, 33000, 3630, 64, "f16"),   # 9-CTA cluster (non-portable size), g = 64
    (1, 1, 1000, 999, 1000, 128, "bf16"),    # n = tokens: everything selected
    (1, 2, 300, 200, 1, 32, "bf16"),         # n = 1
    (4, 8, 5000, 4500, 495, 32, "f16"),      # batch, several clusters per wave
    (1, 2, 131072, 131008, 4096, 32, "bf16"),  # 16-CTA clusters, append into a fresh group
])
def test_fused_step_matches_oracle(cuda, port, B, H, cap, pos, n, g, dtype):
    layer, q, kn, vn, out, sel, scores = run_step(cuda, B, H, cap, pos, n, g, dtype)
    heads = None if B * H <= 8 else [0, H - 1]
    check(port, layer, q, kn, out, sel, scores, pos, n, g, heads)


def test_fused_step_all_ties(cuda, port):
    """Constant keys: every score is equal, so the reference keeps the n lowest indices
    (core.hpp:139-142) -- the tie path of the cluster select inside the fused step."""
    B, H, cap, pos, n = 1, 2, 3000, 2500, 700
    K = torch.full((B, H, cap, 128), 0.5, device=cuda)
    layer, q, kn, vn, out, sel, scores = run_step(cuda, B, H, cap, pos, n, 32, "bf16", K=K)
    np.testing.assert_array_equal(sel.cpu().numpy(), np.broadcast_to(np.arange(n), (B, H, n)))
    check(port, layer, q, kn, out, sel, scores, pos, n, 32)


@pytest.mark.parametrize("tokens,n", [(1000, 300), (700, 699), (40, 7)])
def test_fused_step_tie_groups(cuda, port, tokens, n):
    """Constant keys with fewer ties than the radix candidate buffer: the threshold is
    one tie group resolved by the digit refinement on the indices (lowest indices kept)."""
    B, H, cap = 1, 3, tokens + 64
    K = torch.full((B, H, cap, 128), -0.25, device=cuda)
    layer, q, kn, vn, out, sel, scores = run_step(cuda, B, H, cap, tokens - 1, n, 32, "bf16", K=K)
    np.testing.assert_array_equal(sel.cpu().numpy(), np.broadcast_to(np.arange(n), (B, H, n)))
    check(port, layer, q, kn, out, sel, scores, tokens - 1, n, 32)


def test_fused_step_narrow_scores(cuda, port):
    """Scores squeezed into one radix bin (keys = 8 + tiny noise, q > 0): candidate
    overflow takes the exact MSD radix fallback."""
    torch.manual_seed(21)
    B, H, cap, pos, n = 1, 2, 6000, 5000, 551
    K = 8.0 + 1e-3 * torch.randn(B, H, cap, 128, device=cuda)
    layer, q, kn, vn, out, sel, scores = run_step(cuda, B, H, cap, pos, n, 32, "bf16", K=K)
    check(port, layer, q, kn, out, sel, scores, pos, n, 32)


def test_fused_step_repeated_decode(cuda, port):
    """Several consecutive steps through the same layer (appends crossing a group boundary)
    leave the index equal to a one-shot quantize of the grown cache."""
    import paper_2508_08256_b200 as F
    torch.manual_seed(9)
    B, H, cap, d, g, n = 1, 4, 2048, 128, 32, 150
    layer = F.DecodeLayer(B, H, H, cap, d, g, dtype=torch.bfloat16, device=cuda)
    layer.K.copy_(torch.randn(B, H, cap, d, device=cuda).to(torch.bfloat16))
    layer.V.copy_(torch.randn(B, H, cap, d, device=cuda).to(torch.bfloat16))
    pos0 = 1500
    layer.prefill(pos0)
    for pos in range(pos0, pos0 + 40):
        q = torch.randn(B, H, d, device=cuda).to(torch.bfloat16)
        kn = torch.randn(B, H, d, device=cuda).to(torch.bfloat16)
        out, sel = layer.step(q, kn, kn, pos, n)
    torch.cuda.synchronize()
    Kc = layer.K.double().cpu().numpy()
    for h in range(H):
        assert layer.pk.to_fier(0, h) == port.quantize_fier(Kc[0, h, :pos + 1], g)


def test_separate_step_path_still_matches(cuda, port):
    """FIER_STEP_SEPARATE forces the separate-kernel path (score -> top-k -> attention) for
    the same MHA shape: it must stay correct since it serves A/B measurements."""
    r = run_step(cuda, 1, 4, 9000, 8500, 935, 32, "bf16", separate=True)
    assert r[0].launches(8501, 935, separate=True) == 3 and r[0].launches(8501, 935) == 1
    check(port, r[0], r[1], r[2], r[4], r[5], r[6], 8500, 935, 32)
