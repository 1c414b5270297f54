"""Recall / margin sweep on the GPU: the reference's evaluation
harness (evalharness.hpp) for one fixed workload, with every selection, score and
attention output computed by this package's kernels.

  margin_and_errors (evalharness.hpp:63-83)  -> margin_and_errors()
  run_trial          (evalharness.hpp:184-259) -> run_trial()  (policies fier, quest,
                                                  quest_quant, oracle, full)
  overlap_fraction   (evalharness.hpp:40-48)  -> overlap_fraction()

Out of scope (tier framing): the workload generators beyond a fixed instance, the
streaming / H2O eviction baselines, JSON reporting and the CLI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import torch

from . import _lib
from ._lib import check
from .api import (_as3, _as4, _cuda, _dtype_code, _p, _require, _stream, approx_scores, build_page_summaries,
                  gather_attention, make_shape, quantize, quest_page_scores, quest_select_quantized,
                  select_by_page_scores, topk_oracle)

POLICIES = ("fier", "quest", "quest_quant", "oracle", "full")


def exact_scores(q: torch.Tensor, K: torch.Tensor, scaled: bool = False, tokens: int | None = None
                 ) -> Tuple[torch.Tensor, torch.Tensor]:
    """exact_scores (core.hpp:98-112): (fp64, fp32) [B, Hq, l] (or [l] for a single head)."""
    single = q.dim() == 1
    K4, q3 = _as4(_cuda(K, "exact_scores")), _as3(_cuda(q, "exact_scores"))
    B, Hkv, cap, d = K4.shape
    _require(q3.shape[-1] == d, "exact_scores: query length does not match key dim")
    l = cap if tokens is None else tokens
    Hq = q3.shape[1]
    s64 = torch.empty((B, Hq, l), dtype=torch.float64, device=K4.device)
    s32 = torch.empty((B, Hq, l), dtype=torch.float32, device=K4.device)
    shape = make_shape(B, Hq, Hkv, cap, d, 1, _dtype_code(K4))
    _require(_dtype_code(q3) == shape.dtype, "exact_scores: q and K dtypes differ")
    check(_lib.load().fier_exact_scores(C.byref(shape), _p(q3), _p(K4), l, int(scaled), _p(s64), _p(s32), l,
                                        _stream()))
    return (s64.view(-1), s32.view(-1)) if single else (s64, s32)


def margin_and_errors(exact64: torch.Tensor, exact32: torch.Tensor, est: torch.Tensor, k: int) -> torch.Tensor:
    """margin_and_errors (evalharness.hpp:63-83) per row: fp64 [..., 5] = (margin, max_err,
    l2_loss, hinge_loss, hinge_loss_symmetric)."""
    l = exact64.shape[-1]
    _require(1 <= k < l, "margin_and_errors: need 1 <= k < l")
    rows = exact64.numel() // l
    lib = _lib.load()
    ws = torch.empty(lib.fier_margin_errors_workspace(rows, k), dtype=torch.uint8, device=exact64.device)
    rep = torch.empty(exact64.shape[:-1] + (5,), dtype=torch.float64, device=exact64.device)
    check(lib.fier_margin_errors(_p(exact64.contiguous()), _p(exact32.contiguous()), _p(est.contiguous()), rows, l, l,
                                 k, _p(rep), _p(ws), ws.numel(), _stream()))
    return rep


def overlap_fraction(sel: torch.Tensor, oracle: torch.Tensor) -> torch.Tensor:
    """overlap_fraction (evalharness.hpp:40-48) per row: fp64 [...]."""
    n, no = sel.shape[-1], oracle.shape[-1]
    rows = sel.numel() // n
    out = torch.empty(sel.shape[:-1], dtype=torch.float64, device=sel.device)
    check(_lib.load().fier_overlap(_p(sel.to(torch.int32).contiguous()), n, _p(oracle.to(torch.int32).contiguous()),
                                   no, rows, _p(out), _stream()))
    return out


def _rel_l2(got: torch.Tensor, want: torch.Tensor) -> torch.Tensor:
    """relative_l2_error (core.hpp:181-190) per row (fp64 reduction of the fp32 outputs)."""
    g, w = got.double(), want.double()
    num, den = ((g - w) ** 2).sum(-1), (w * w).sum(-1)
    return torch.where(den == 0, torch.where(num == 0, torch.zeros_like(num), torch.full_like(num, float("inf"))),
                       (num / den).sqrt())


@dataclass
class Trial:
    budgets: List[int]
    cells: Dict[str, Dict[str, List[float]]] = field(default_factory=dict)  # policy -> metric -> per budget
    margins: List[float] = field(default_factory=list)


def run_trial(K: torch.Tensor, V: torch.Tensor, queries: torch.Tensor, budgets: Sequence[int], group: int = 32,
              page_size: int = 16, variant: str = "sum") -> Trial:
    """run_trial (evalharness.hpp:184-259) on one fixed workload: K, V [l, d], queries [nq, d]
    (one head).  Per policy and budget, averaged over the queries: recall (overlap with the
    exact top-n), out_err (relative L2 of the attention output against full attention),
    max_err (max |exact - estimate| over tokens); margins per budget (NaN at n = l)."""
    _require(K.dim() == 2 and K.shape == V.shape, "run_trial: K and V must be [l, d] and aligned")
    l, d = K.shape
    Q = queries if queries.dim() == 2 else queries.view(1, -1)
    for b in budgets:
        _require(1 <= b <= l, "sweep: budget out of range")
    pk = quantize(K, group)
    ps = build_page_summaries(K, page_size)
    t = Trial(list(budgets))
    acc = {p: {"recall": [0.0] * len(budgets), "out_err": [0.0] * len(budgets), "max_err": [0.0] * len(budgets)}
           for p in POLICIES}
    marg = [0.0] * len(budgets)
    every = torch.arange(l, dtype=torch.int32, device=K.device)
    for qi in range(Q.shape[0]):
        q = Q[qi]
        ex64, ex32 = exact_scores(q, K)
        full = gather_attention(q, K, V, every, validate=False)
        est_f = approx_scores(q, pk)
        pscores = quest_page_scores(q, ps, variant)
        est_q = pscores.repeat_interleave(page_size)[:l]  # page scores broadcast over members
        err = {"fier": (ex64 - est_f.double()).abs().max().item(), "quest": (ex64 - est_q.double()).abs().max().item(),
               "quest_quant": (ex64 - est_f.double()).abs().max().item(), "oracle": 0.0, "full": 0.0}
        for bi, n in enumerate(budgets):
            oracle = topk_oracle(ex32, n)
            if n < l:
                marg[bi] += float(margin_and_errors(ex64, ex32, est_f, n)[0].item())
            else:
                marg[bi] = float("nan")
            sels = {"fier": topk_oracle(est_f, n),
                    "quest": select_by_page_scores(pscores, l, page_size, n),
                    "quest_quant": quest_select_quantized(q, pk, page_size, n),
                    "oracle": oracle, "full": every}
            for p in POLICIES:
                s = sels[p]
                out = full if p == "full" else gather_attention(q, K, V, s, validate=False)
                acc[p]["recall"][bi] += float(overlap_fraction(s, oracle).item())
                acc[p]["out_err"][bi] += float(_rel_l2(out, full).item())
                acc[p]["max_err"][bi] += err[p]
    nq = Q.shape[0]
    for p in POLICIES:
        t.cells[p] = {m: [v / nq for v in vals] for m, vals in acc[p].items()}
    t.margins = [m / nq for m in marg]
    return t
