"""GPU parity of the four kernels against the oracle and the reference's golden vectors.

Bars (BASELINE.json north_star):
  packed bits + (s, z)          bit-exact (FIER bytes compared byte for byte)
  scores                        |gpu - ref| <= 1e-3 * max(1, |ref|)  (test_quant1bit.cpp:149 denominator)
  selection                     bit-exact vs topk_oracle on the GPU's own scores; recall >= 0.999
                                vs the reference's selection, mismatches only at score-tolerance ties
  attention output              relative L2 < 1e-2 vs gather_attention on the same selection
"""
import numpy as np
import pytest
import torch

from conftest import check_selection, golden_cases, load_golden

pytestmark = pytest.mark.gpu

TDT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}
SCORE_TOL = 1e-3
OUT_TOL = 1e-2


def fier():
    import paper_2508_08256_b200 as F
    return F


def case_tensors(c, dev):
    dt = TDT[c["dtype"]]
    K = torch.from_numpy(c["K"]).to(dev, dt).unsqueeze(0)  # [1, Hkv, l, d]
    V = torch.from_numpy(c["V"]).to(dev, dt).unsqueeze(0)
    Q = torch.from_numpy(c["Q"]).to(dev, dt).unsqueeze(0)  # [1, Hq, d]
    return K, V, Q


def score_err(gpu, ref):
    return np.max(np.abs(gpu - ref) / np.maximum(1.0, np.abs(ref)))


@pytest.mark.parametrize("name", golden_cases())
def test_pack_bit_exact(cuda, name):
    c = load_golden(name)
    K, V, Q = case_tensors(c, cuda)
    pk = fier().quantize(K, c["g"])
    for h in range(c["hkv"]):
        assert pk.to_fier(0, h) == c["fier_list"][h], f"kv head {h}"


@pytest.mark.parametrize("name", golden_cases())
def test_scores_within_tolerance(cuda, name):
    c = load_golden(name)
    K, V, Q = case_tensors(c, cuda)
    pk = fier().quantize(K, c["g"])
    s = fier().approx_scores(Q, pk)[0].cpu().numpy().astype(np.float64)
    assert score_err(s, c["scores"]) <= SCORE_TOL


@pytest.mark.parametrize("name", golden_cases())
def test_selection_and_output(cuda, port, name):
    c = load_golden(name)
    K, V, Q = case_tensors(c, cuda)
    F = fier()
    pk = F.quantize(K, c["g"])
    est = F.approx_scores(Q, pk)
    sel = F.topk_oracle(est, c["n"])
    out = F.gather_attention(Q, K, V, sel)
    est_np, sel_np, out_np = est[0].cpu().numpy(), sel[0].cpu().numpy(), out[0].cpu().numpy()
    group = c["hq"] // c["hkv"]
    for h in range(c["hq"]):
        kv = h // group
        # K3 is exact on the scores it was given
        np.testing.assert_array_equal(sel_np[h], port.topk(est_np[h].astype(np.float64), c["n"]))
        # against the reference's selection on its fp64 scores
        want = c["sel"][h]
        rec = port.recall(sel_np[h], want)
        assert rec >= 0.999 or _only_tolerance_ties(sel_np[h], want, c["scores"][h]), (h, rec)
        q = c["Q"][h].astype(np.float64)
        ref_out = port.gather_attention(q, c["K"][kv], c["V"][kv], sel_np[h].astype(np.int64))
        assert port.relative_l2_error(out_np[h], ref_out) < OUT_TOL
        if np.array_equal(sel_np[h], want):
            assert port.relative_l2_error(out_np[h], c["out"][h]) < OUT_TOL


def _only_tolerance_ties(got, want, ref_scores):
    """Every index in the symmetric difference scores within tolerance of the threshold."""
    diff = np.setxor1d(got, want)
    thr = np.sort(ref_scores)[::-1][len(want) - 1]
    return all(abs(ref_scores[i] - thr) <= 2 * SCORE_TOL * max(1.0, abs(thr)) for i in diff)


@pytest.mark.parametrize("name", golden_cases())
def test_full_attention_matches_reference(cuda, name):
    c = load_golden(name)
    K, V, Q = case_tensors(c, cuda)
    out = fier().full_attention(Q, K, V)[0].cpu().numpy()
    group = c["hq"] // c["hkv"]
    for h in range(c["hq"]):
        num = np.linalg.norm(out[h] - c["full"][h])
        assert num / np.linalg.norm(c["full"][h]) < OUT_TOL


@pytest.mark.parametrize("name", ["mha_d128", "gqa_d64", "planted_spikes", "score_ties"])
def test_fier_attend_composition(cuda, name):
    """fier_attend == topk_oracle(approx_scores) -> gather_attention (test_retrieval.cpp:108-120)."""
    c = load_golden(name)
    K, V, Q = case_tensors(c, cuda)
    F = fier()
    pk = F.quantize(K, c["g"])
    r = F.fier_attend(Q, K, V, pk, c["n"])
    sel = F.fier_select(Q, pk, c["n"])
    assert torch.equal(r.selection, sel)
    assert torch.equal(r.output, F.gather_attention(Q, K, V, sel))
    assert r.bytes_loaded_for_estimation == int(c["bytes_loaded"][0])
    with pytest.raises(ValueError, match="fier_select: budget out of range"):
        F.fier_select(Q, pk, c["l"] + 1)


def test_planted_spikes_selected(cuda):
    """Planted keys (workload.hpp:169-191) own the top logits and are always selected."""
    c = load_golden("planted_spikes")
    K, V, Q = case_tensors(c, cuda)
    F = fier()
    sel = F.fier_select(Q, F.quantize(K, c["g"]), c["n"])[0].cpu().numpy()
    np.testing.assert_array_equal(sel, c["sel"])


@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("g", [32, 8, 128])
def test_append_equals_one_shot(cuda, port, dtype, g):
    """Incremental decode-time packing == quantize(K[0:l]) bit for bit, across group boundaries."""
    F = fier()
    torch.manual_seed(7)
    B, H, cap, d = 2, 3, 200, 128
    dt = TDT[dtype]
    Kfull = (torch.randn(B, H, cap, d, device=cuda) * 3).to(dt)
    Vfull = torch.randn(B, H, cap, d, device=cuda).to(dt)
    t0 = 37
    K = torch.zeros_like(Kfull)
    V = torch.zeros_like(Vfull)
    K[:, :, :t0] = Kfull[:, :, :t0]
    V[:, :, :t0] = Vfull[:, :, :t0]
    pk = F.quantize(K, g, tokens=t0)
    for pos in range(t0, 141):
        F.append_token(K, V, Kfull[:, :, pos].contiguous(), Vfull[:, :, pos].contiguous(), pos, pk,
                       check_finite=(pos % 50 == 0))
        if pos in (t0, 63, 64, 95, 127, 128, 140):
            for b in range(B):
                for h in range(H):
                    want = port.quantize_fier(Kfull[b, h, :pos + 1].double().cpu().numpy(), g)
                    assert pk.to_fier(b, h) == want, (pos, b, h)
    assert torch.equal(V[:, :, :141], Vfull[:, :, :141])


def test_nonfinite_keys_rejected(cuda):
    F = fier()
    K = torch.randn(40, 16, device=cuda)
    K[17, 3] = float("inf")
    with pytest.raises(ValueError, match="quantize: non-finite key entry"):
        F.quantize(K, 32)


def test_gather_attention_rejects_like_reference(cuda):
    F = fier()
    K = torch.randn(10, 128, device=cuda, dtype=torch.bfloat16)
    q = torch.randn(128, device=cuda, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="selection invalid for cache"):
        F.gather_attention(q, K, K, torch.tensor([3, 2], device=cuda))
    with pytest.raises(ValueError, match="selection invalid for cache"):
        F.gather_attention(q, K, K, torch.tensor([3, 10], device=cuda))
    with pytest.raises(ValueError, match="topk_oracle: k out of range"):
        F.topk_oracle(torch.randn(5, device=cuda), 6)


def test_single_token_returns_value_row(cuda):
    """test_kvcore.cpp:156-166 / test_retrieval.cpp:100-106."""
    F = fier()
    K = torch.randn(8, 128, device=cuda)
    V = torch.randn(8, 128, device=cuda)
    q = torch.randn(128, device=cuda)
    out = F.gather_attention(q, K, V, torch.tensor([5], device=cuda, dtype=torch.int32))
    torch.testing.assert_close(out, V[5], rtol=0, atol=0)


@pytest.mark.parametrize("l,k", [(1, 1), (31, 7), (33, 33), (1000, 1), (4097, 4096), (70000, 7700),
                                 (300000, 33000)])
def test_topk_exact_sizes(cuda, port, l, k):
    F = fier()
    g = torch.Generator(device="cpu").manual_seed(l)
    s = torch.randn(3, l, generator=g)
    s[1] = torch.round(s[1] * 4) / 4  # heavy ties
    s[2, : l // 2] = 0.0
    s[2, l // 2:] = -0.0  # signed zeros tie (core.hpp:139-142)
    sel = F.topk_oracle(s.to(cuda), k).cpu().numpy()
    for r in range(3):
        np.testing.assert_array_equal(sel[r], port.topk(s[r].double().numpy(), k))


def test_topk_extremes(cuda, port):
    F = fier()
    s = torch.tensor([0.0, float("inf"), -float("inf"), 1e38, -1e38, 3.0, 3.0, -0.0, 1e-45, -1e-45])
    for k in range(1, s.numel() + 1):
        got = F.topk_oracle(s.to(cuda), k).cpu().numpy()
        np.testing.assert_array_equal(got, port.topk(s.double().numpy(), k))


@pytest.mark.parametrize("B,Hq,Hkv,d,dtype", [(2, 4, 2, 128, "bf16"), (1, 8, 8, 64, "f16"),
                                              (3, 2, 1, 24, "f32"), (1, 32, 8, 128, "bf16")])
def test_decode_step_matches_oracle(cuda, port, B, Hq, Hkv, d, dtype):
    F = fier()
    torch.manual_seed(11)
    dt, cap, g = TDT[dtype], 700, 32
    layer = F.DecodeLayer(B, Hq, Hkv, cap, d, g, dtype=dt, device=cuda)
    layer.K.copy_(torch.randn(B, Hkv, cap, d, device=cuda).to(dt))
    layer.V.copy_(torch.randn(B, Hkv, cap, d, device=cuda).to(dt))
    pos = 613
    layer.prefill(pos)
    q = torch.randn(B, Hq, d, device=cuda).to(dt)
    kn = torch.randn(B, Hkv, d, device=cuda).to(dt)
    vn = torch.randn(B, Hkv, d, device=cuda).to(dt)
    n = 77
    ld = pos + 1 + (-(pos + 1)) % 32
    scores = torch.empty(B, Hq, ld, device=cuda)
    out, sel = layer.step(q, kn, vn, pos, n, scores_out=scores)
    torch.cuda.synchronize()
    Kc, Vc = layer.K.double().cpu().numpy(), layer.V.double().cpu().numpy()
    assert np.array_equal(Kc[:, :, pos], kn.double().cpu().numpy())
    sel_np, out_np, sc = sel.cpu().numpy(), out.cpu().numpy(), scores.cpu().numpy()
    group = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            kv = h // group
            buf = port.quantize_fier(Kc[b, kv, :pos + 1], g)
            assert layer.pk.to_fier(b, kv) == buf
            qd = q[b, h].double().cpu().numpy()
            ref_scores = port.approx_scores_fier(qd, buf)
            assert score_err(sc[b, h, :pos + 1], ref_scores) <= SCORE_TOL
            np.testing.assert_array_equal(sel_np[b, h], port.topk(sc[b, h, :pos + 1].astype(np.float64), n))
            check_selection(sel_np[b, h], ref_scores, n, port)
            ref_out = port.gather_attention(qd, Kc[b, kv, :pos + 1], Vc[b, kv, :pos + 1],
                                            sel_np[b, h].astype(np.int64))
            assert port.relative_l2_error(out_np[b, h], ref_out) < OUT_TOL
    # K0 on the same cache
    full = layer.full_step(q, pos + 1).cpu().numpy()
    for b in range(B):
        for h in range(0, Hq, max(1, Hq // 4)):
            kv = h // group
            qd = q[b, h].double().cpu().numpy()
            ref = port.gather_attention(qd, Kc[b, kv, :pos + 1], Vc[b, kv, :pos + 1], np.arange(pos + 1))
            assert port.relative_l2_error(full[b, h], ref) < OUT_TOL


def test_c2_shape_step_properties(cuda, port):
    """Full C2 shape (32 MHA heads, d=128, l=32768, n=3604, bf16): exact selection on the
    GPU scores, score tolerance and output tolerance on sampled heads, FIER round trip."""
    F = fier()
    torch.manual_seed(3)
    B, H, L, d, n = 1, 32, 32768, 128, 3604
    layer = F.DecodeLayer(B, H, H, L, d, 32, dtype=torch.bfloat16, device=cuda)
    layer.K.copy_(torch.randn(B, H, L, d, device=cuda).to(torch.bfloat16))
    layer.V.copy_(torch.randn(B, H, L, d, device=cuda).to(torch.bfloat16))
    layer.prefill(L - 1)
    q = torch.randn(B, H, d, device=cuda).to(torch.bfloat16)
    kn = torch.randn(B, H, d, device=cuda).to(torch.bfloat16)
    scores = torch.empty(B, H, L, device=cuda)
    out, sel = layer.step(q, kn, kn, L - 1, n, scores_out=scores)
    sel_np = sel[0].cpu().numpy()
    assert (np.diff(sel_np, axis=1) > 0).all() and sel_np.min() >= 0 and sel_np.max() < L
    sc = scores[0].cpu().numpy().astype(np.float64)
    for h in (0, 13, 31):
        np.testing.assert_array_equal(sel_np[h], port.topk(sc[h], n))
        Kh = layer.K[0, h].double().cpu().numpy()
        Vh = layer.V[0, h].double().cpu().numpy()
        buf = layer.pk.to_fier(0, h)
        assert buf == port.quantize_fier(Kh, 32)
        qd = q[0, h].double().cpu().numpy()
        ref_scores = port.approx_scores_fier(qd, buf)
        assert score_err(sc[h], ref_scores) <= SCORE_TOL
        assert port.recall(sel_np[h], port.topk(ref_scores, n)) >= 0.999
        ref_out = port.gather_attention(qd, Kh, Vh, sel_np[h].astype(np.int64))
        assert port.relative_l2_error(out[0, h].cpu().numpy(), ref_out) < OUT_TOL


@pytest.mark.parametrize("hpg", [1, 2, 4, 8])
@pytest.mark.parametrize("g,L,dtype", [(32, 1000, "bf16"), (64, 777, "f16"), (128, 2085, "f32"),
                                       (32, 31, "bf16"), (32, 8193, "bf16")])
def test_score_tensor_core_shapes(cuda, port, hpg, g, L, dtype):
    """K2 (tensor-core sign-select scorer, d = 128): every GQA ratio, g in {32, 64, 128},
    ragged token counts, against approx_scores over the FIER round trip."""
    F = fier()
    torch.manual_seed(hpg * 1000 + L)
    dt, Hkv, B, d = TDT[dtype], 2, 2, 128
    K = (torch.randn(B, Hkv, L, d, device=cuda) * 3).to(dt)
    q = torch.randn(B, Hkv * hpg, d, device=cuda).to(dt)
    pk = F.quantize(K, g)
    s = F.approx_scores(q, pk).cpu().numpy().astype(np.float64)
    for b in range(B):
        for h in range(Hkv * hpg):
            kv = h // hpg
            buf = pk.to_fier(b, kv)
            ref = port.approx_scores_fier(q[b, h].double().cpu().numpy(), buf)
            assert score_err(s[b, h], ref) <= SCORE_TOL, (b, h)


@pytest.mark.parametrize("g", [32, 64, 128])
def test_score_tensor_core_multi_slab_stages(cuda, port, g):
    """K2's ring stages of up to 4 slabs: enough slabs per warp that stages hold 1..4 slabs, cross
    sequence boundaries (a stage never does: it is cut there) and, for g > 32, cover 1..3 groups."""
    F = fier()
    torch.manual_seed(g)
    B, Hkv, hpg, L, d = 1, 8, 4, 40013, 128
    K = (torch.randn(B, Hkv, L, d, device=cuda) * 3).to(torch.bfloat16)
    q = torch.randn(B, Hkv * hpg, d, device=cuda).to(torch.bfloat16)
    pk = F.quantize(K, g)
    s = F.approx_scores(q, pk).cpu().numpy().astype(np.float64)
    for kv in range(Hkv):
        buf = pk.to_fier(0, kv)
        for h in range(kv * hpg, (kv + 1) * hpg):
            ref = port.approx_scores_fier(q[0, h].double().cpu().numpy(), buf)
            assert score_err(s[0, h], ref) <= SCORE_TOL, (g, h)


@pytest.mark.parametrize("hpg,g,pos", [(1, 32, 4100), (4, 32, 4127), (4, 64, 4097), (8, 128, 4000),
                                       (2, 32, 31), (1, 32, 0)])
def test_fused_append_score_tensor_core(cuda, port, hpg, g, pos):
    """The decode step's fused append + score: open group re-packed, then scored by the same CTA."""
    F = fier()
    torch.manual_seed(pos + hpg)
    B, Hkv, d, cap, n = 1, 4, 128, 4200, 1
    dt = torch.bfloat16
    layer = F.DecodeLayer(B, Hkv * hpg, Hkv, cap, d, g, dtype=dt, device=cuda)
    layer.K.copy_(torch.randn(B, Hkv, cap, d, device=cuda).to(dt))
    layer.V.copy_(torch.randn(B, Hkv, cap, d, device=cuda).to(dt))
    if pos > 0:
        layer.prefill(pos)
    q = torch.randn(B, Hkv * hpg, d, device=cuda).to(dt)
    kn = torch.randn(B, Hkv, d, device=cuda).to(dt)
    ld = pos + 1 + (-(pos + 1)) % 32
    scores = torch.empty(B, Hkv * hpg, ld, device=cuda)
    layer.step(q, kn, kn, pos, n, scores_out=scores)
    torch.cuda.synchronize()
    sc = scores.cpu().numpy().astype(np.float64)
    for h in range(Hkv * hpg):
        kv = h // hpg
        buf = layer.pk.to_fier(0, kv)
        assert buf == port.quantize_fier(layer.K[0, kv, :pos + 1].double().cpu().numpy(), g)
        ref = port.approx_scores_fier(q[0, h].double().cpu().numpy(), buf)
        assert score_err(sc[0, h, :pos + 1], ref) <= SCORE_TOL, h


@pytest.mark.parametrize("rows,l,k", [(32, 32768, 3604), (32, 131072, 4096), (200, 32768, 3604), (8, 8192, 1),
                                      (4, 262144, 28835), (16, 32768, 32768)])
def test_topk_register_path_shapes(cuda, port, rows, l, k):
    """K3 at the bench shapes (cluster sizes 1..8) plus value distributions that stress
    each branch: clustered candidates (refinement), exact-tie plateaus at the threshold,
    outliers stretching the range, and -inf padding (the shard merge)."""
    F = fier()
    g = torch.Generator(device="cpu").manual_seed(rows * 7 + l)
    s = torch.randn(rows, l, generator=g) * 20
    s[1] = torch.round(s[1])                             # ties everywhere
    s[2, :] = 1.0
    s[2, ::97] = 2.0                                     # a plateau straddling the k-th value
    if rows > 3:
        s[3, 5] = 3e38
        s[3, 6] = -3e38                                  # range blow-up -> candidates cluster
    if rows > 4:
        s[4, l // 3:] = -float("inf")                    # padding
        s[4, : l // 3] = torch.round(s[4, : l // 3] * 8) / 8
    if rows > 5:
        s[5] = 1e-3 * torch.randn(l, generator=g) + 5.0  # narrow band
    sel = F.topk_oracle(s.to(cuda), k).cpu().numpy()
    for r in range(min(rows, 8)):
        np.testing.assert_array_equal(sel[r], port.topk(s[r].double().numpy(), k), err_msg=f"row {r}")
    if rows > 8:  # remaining rows: cheap structural checks + a sample against the oracle
        assert (np.diff(sel, axis=1) > 0).all()
        for r in range(8, rows, max(1, rows // 16)):
            np.testing.assert_array_equal(sel[r], port.topk(s[r].double().numpy(), k))


@pytest.mark.parametrize("l,k", [(1048576, 4096), (600001, 66000)])
def test_topk_long_rows(cuda, port, l, k):
    """K3 for rows beyond the on-chip paths (topk_long.cu, C5's 1M tokens): random scores,
    heavy ties, and a constant row (candidate overflow -> the streaming radix fallback)."""
    F = fier()
    g = torch.Generator(device="cpu").manual_seed(l + k)
    s = torch.randn(3, l, generator=g) * 8
    s[1] = torch.round(s[1] * 2) / 2                      # ties at the threshold
    s[2] = 0.75
    s[2, ::1000] = 1.5
    sel = F.topk_oracle(s.to(cuda), k).cpu().numpy()
    for r in range(3):
        np.testing.assert_array_equal(sel[r], port.topk(s[r].double().numpy(), k))


@pytest.mark.parametrize("hq,hkv,dtype,g,pos", [
    (8, 8, torch.bfloat16, 32, 4127),   # MHA: one-launch step (the appending CTA re-packs, then stores)
    (8, 8, torch.float32, 32, 4096),    # fp32 MHA: append fused into score128
    (8, 2, torch.bfloat16, 32, 4131),   # GQA: append fused into the tensor-core scorer
    (8, 2, torch.bfloat16, 64, 0),      # first token of an empty cache
])
def test_step_writes_kv_rows_and_open_group(cuda, port, hq, hkv, dtype, g, pos):
    """Every step path stores the new k / v rows exactly (the re-pack reads token pos from
    k_new and the row stores come after it) and leaves the index == quantize(K[0:pos+1])."""
    F = fier()
    torch.manual_seed(pos + hq + hkv)
    B, d, cap, n = 1, 128, 4200, 1
    layer = F.DecodeLayer(B, hq, hkv, cap, d, g, dtype=dtype, device=cuda)
    layer.K.copy_(torch.randn(B, hkv, cap, d, device=cuda).to(dtype))
    layer.V.copy_(torch.randn(B, hkv, cap, d, device=cuda).to(dtype))
    if pos > 0:
        layer.prefill(pos)
    q = torch.randn(B, hq, d, device=cuda).to(dtype)
    kn = (torch.randn(B, hkv, d, device=cuda) * 4).to(dtype)  # likely a new group min/max
    vn = torch.randn(B, hkv, d, device=cuda).to(dtype)
    layer.step(q, kn, vn, pos, n)
    torch.cuda.synchronize()
    assert torch.equal(layer.K[:, :, pos], kn)
    assert torch.equal(layer.V[:, :, pos], vn)
    for kv in range(hkv):
        assert layer.pk.to_fier(0, kv) == port.quantize_fier(layer.K[0, kv, :pos + 1].double().cpu().numpy(), g)


@pytest.mark.parametrize("hq,hkv,dtype,rope,d", [
    (8, 2, torch.bfloat16, None, 128),                 # GQA: inputs staged from host memory, then 3 launches
    (8, 8, torch.float32, None, 128),                  # fp32 MHA
    (8, 2, torch.bfloat16, (10000.0, 128, False), 128),  # RoPE: the rope kernel reads host q / k_new, v_new direct
    (4, 2, torch.float16, None, 11),                   # odd d: generic scorer, byte-wise staging copy
    (4, 4, torch.bfloat16, None, 128),                 # MHA one-launch kernel reading host memory directly
])
def test_step_with_host_resident_inputs(cuda, hq, hkv, dtype, rope, d):
    """fier_decode_step on pinned host q / k_new / v_new / out (the zero-copy public-API path,
    FIER_STEP_HOST_INPUTS) gives bit-identical results to the same step on device buffers."""
    F = fier()
    B, cap, pos, n = 2, 3000, 2500, 300
    torch.manual_seed(11)
    K0 = torch.randn(B, hkv, cap, d, device=cuda).to(dtype)
    V0 = torch.randn(B, hkv, cap, d, device=cuda).to(dtype)
    q = torch.randn(B, hq, d, device=cuda).to(dtype)
    kn = torch.randn(B, hkv, d, device=cuda).to(dtype)
    vn = torch.randn(B, hkv, d, device=cuda).to(dtype)
    outs = []
    for host in (False, True):
        layer = F.DecodeLayer(B, hq, hkv, cap, d, 32, dtype=dtype, device=cuda)
        layer.K.copy_(K0)
        layer.V.copy_(V0)
        layer.prefill(pos)
        if host:
            qa, ka, va = (x.cpu().pin_memory() for x in (q, kn, vn))
            out = torch.empty(B, hq, d, dtype=torch.float32).pin_memory()
        else:
            qa, ka, va, out = q, kn, vn, None
        o, sel = layer.step(qa, ka, va, pos, n, out=out, rope=rope, host_inputs=host)
        torch.cuda.synchronize()
        outs.append((o.cpu().clone(), sel.cpu().clone(), layer.K[:, :, pos].cpu(), layer.V[:, :, pos].cpu()))
    (o0, s0, k0, v0), (o1, s1, k1, v1) = outs
    assert torch.equal(s0, s1) and torch.equal(k0, k1) and torch.equal(v0, v1)
    if layer.launches(pos + 1, n) == 1:
        # the one-launch kernel merges its gather warps' partials in completion order:
        # equal up to fp32 summation order
        assert torch.allclose(o0, o1, rtol=1e-5, atol=1e-6)
    else:
        assert torch.equal(o0, o1)


@pytest.mark.parametrize("l,k", [(5000, 550), (70000, 4096), (300000, 9000), (1048576, 4096)])
def test_topk_nan_scores_rank_lowest(cuda, l, k):
    """NaN scores (a non-finite query) rank below every number, ties to the lower index:
    every path (cluster select, long rows) still writes k valid ascending indices."""
    F = fier()
    g = torch.Generator().manual_seed(l)
    s = torch.randn(3, l, generator=g)
    s[0, ::3] = float("nan")
    s[1] = float("nan")
    s[2, ::2] = float("nan")
    s[2, 1::2] = float("-inf")
    got = F.topk_oracle(s.to(cuda), k).cpu().numpy()
    for r in range(3):
        v = s[r].double().numpy()
        nan = np.isnan(v)
        order = np.lexsort((np.arange(l), -np.where(nan, 0.0, v), nan))  # numbers desc, then NaN; index asc
        np.testing.assert_array_equal(got[r], np.sort(order[:k]))


@pytest.mark.parametrize("rows,l,k", [(128, 131072, 4096), (1024, 32768, 3604), (17, 1048576, 4096),
                                      (36, 500001, 8192), (256, 65537, 1), (160, 131072, 8192),
                                      (700, 4096, 4096), (800, 5001, 1), (640, 65536, 60000), (600, 1030, 515)])
def test_topk_wide_grid(cuda, port, rows, l, k):
    """The wide-grid radix selects (topk_global.cu): the CTA-per-row kernel for launches of
    many short rows (C4) and the global-state kernels for millions of keys in few rows (C5):
    exact vs the oracle on random rows, tie plateaus at the threshold, range outliers,
    -inf padding, NaN rows, a constant row (candidate overflow -> the in-kernel exact
    path); identical to the cluster select on every row."""
    F = fier()
    g = torch.Generator(device="cpu").manual_seed(rows + l + k)
    s = torch.randn(rows, l, generator=g) * 20
    s[1] = torch.round(s[1])                              # ties everywhere
    s[2, :] = 1.0
    s[2, ::97] = 2.0                                      # plateau straddling the k-th value
    s[3, 5], s[3, 6] = 3e38, -3e38                        # range outliers
    s[4, l // 3:] = -float("inf")                         # padding
    if rows > 5:
        s[5, ::3] = float("nan")
        s[5, 1::3] = 1e-3 * torch.randn(len(range(1, l, 3)), generator=g) + 5.0  # narrow band + NaN
    if rows > 6:
        s[6] = 0.5                                        # constant: one bin holds every key
    sd = s.to(cuda)
    wide = F.topk_oracle(sd, k).cpu().numpy()
    clus = F.topk_oracle(sd, k, wide=False).cpu().numpy()
    np.testing.assert_array_equal(wide, clus)
    for r in list(range(min(rows, 7))) + list(range(7, rows, max(1, rows // 8))):
        v = s[r].double().numpy()
        nan = np.isnan(v)
        if nan.any():
            order = np.lexsort((np.arange(l), -np.where(nan, 0.0, v), nan))
            want = np.sort(order[:k])
        else:
            want = port.topk(v, k)
        np.testing.assert_array_equal(wide[r], want, err_msg=f"row {r}")


@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32"])
def test_score_tensor_core_extremes(cuda, port, dtype):
    """The sign-select scorer's operand ranges: per-head query scales 2^-20 .. 2^20 (2^-10 .. 2^10
    for fp16 queries; the fp16 q pieces are scaled by 2^-e per head), channels spanning 2^-10 ..
    2^10 inside one head, zero
    heads, constant key groups (s = 0), groups with a large spread (s near the fp16 range), and
    negative / positive offsets z -- all within the 1e-3 score tolerance of approx_scores."""
    F = fier()
    g_ = torch.Generator().manual_seed(7)
    dt, B, Hkv, hpg, L, d, g = TDT[dtype], 1, 2, 4, 160, 128, 32
    K = torch.randn(B, Hkv, L, d, generator=g_) * 2
    K[0, 0, 0:32] = 3.25                                   # constant group: s = 0
    K[0, 0, 32:64] *= 1500.0                               # large spread: s ~ 1e3..1e4
    K[0, 1, 64:96] += 200.0                                # positive offsets
    K[0, 1, 96:128] -= 300.0                               # negative offsets
    q = torch.randn(B, Hkv * hpg, d, generator=g_)
    big = 10 if dtype == "f16" else 20                     # (fp16 queries overflow past 2^16)
    q[0, 0] *= 2.0 ** big
    q[0, 1] *= 2.0 ** -big
    q[0, 2] = 0.0
    q[0, 3] *= torch.logspace(-big // 2, big // 2, d, base=2.0)  # dynamic range inside one head
    q[0, 5] *= 2.0 ** (big // 2)
    pk = F.quantize(K.to(dt).to(cuda), g)
    qd = q.to(dt).to(cuda)
    s = F.approx_scores(qd, pk).cpu().numpy().astype(np.float64)
    for h in range(Hkv * hpg):
        kv = h // hpg
        ref = port.approx_scores_fier(qd[0, h].double().cpu().numpy(), pk.to_fier(0, kv))
        assert score_err(s[0, h], ref) <= SCORE_TOL, h
