"""Phase timeline of the fused decode step (csrc/step_fused.cu, -DFIER_STEP_TRACE build).

  python -m paper_2508_08256_b200.build --trace
  FIER_LIB=paper_2508_08256_b200/libfier_cuda_trace.so python tools/step_trace.py [--config c2]

Runs the step over rotated layer instances (cold L2, like bench.py) and prints, per
phase, the median / max over CTAs of the time since the kernel's earliest CTA start:
  0 start  1 append done  2 scoring done  3 threshold done  4 compaction done
  5 gather done (warp 0)  6 cluster merge barrier  7 rank 0 wrote the output
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2508_08256_b200 as F  # noqa: E402
from paper_2508_08256_b200 import _lib  # noqa: E402

NAMES = ["start", "append", "score", "resolve", "emit", "gather", "merge_sync", "out",
         "t:hist_sync", "t:find_bin", "t:partition", "t:cand_sync", "t:cand_gather", "t:rank", "t:merged", "g:above_done",
         "a:pack_start", "cta_scored", "p:keys", "p:cands", "p:sync", "a:packed", "a:published", "a:open_scored"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--pairs", type=lambda x: [tuple(map(int, p.split(":"))) for p in x.split(",")], default=[],
                    help="mark pairs i:j to print per-CTA interval percentiles for, e.g. 16:17,18:19")
    ap.add_argument("--raw", type=lambda x: [int(v) for v in x.split(",")], default=[],
                    help="slots to print raw (probe builds: cycles), e.g. 16,17,18")
    a = ap.parse_args()
    assert os.environ.get("FIER_LIB", "").endswith("_trace.so"), "set FIER_LIB to the trace build"
    cfg = bench.CONFIGS[a.config]
    dev = torch.device("cuda")
    lib = _lib.load()
    lib.fier_debug_step_trace.argtypes = [C.c_void_p, C.c_int]
    lib.fier_debug_step_trace_clear()
    lib.fier_debug_step_occupancy.argtypes = [C.c_int]
    print("max active clusters (bf16):",
          {c: lib.fier_debug_step_occupancy(c) for c in (1, 2, 4, 8, 16)})
    B, Hq, Hkv, L, d, n, g = (cfg[k] for k in ("B", "Hq", "Hkv", "L", "d", "n", "g"))
    pos = L - 1
    layers = []
    for i in range(a.layers):
        K, V, q, kn, vn = bench.make_inputs(cfg, 1234 + i, dev)
        lay = F.DecodeLayer(B, Hq, Hkv, L, d, g, dtype=K.dtype, device=dev, K=K, V=V)
        lay.prefill(pos)
        layers.append((lay, q, kn, vn))
    buf = np.zeros((4096, len(NAMES)), dtype=np.uint64)
    rows, raws = [], []
    for r in range(a.reps):
        lay, q, kn, vn = layers[r % len(layers)]
        torch.cuda.synchronize()
        lay.step(q, kn, vn, pos, n)
        torch.cuda.synchronize()
        if r < len(layers):
            continue  # warm-up
        lib.fier_debug_step_trace(buf.ctypes.data, buf.shape[0])
        lib.fier_debug_step_trace_clear()
        t = buf.astype(np.int64)
        t = t[t[:, 0] > 0]
        buf[:] = 0
        t0 = t[:, 0].min()
        rows.append(t - t0)
        raws.append(t.copy())
    nct = rows[0].shape[0] // (B * Hq)  # CTAs per cluster (grid = cluster x rows)
    if nct > 1:
        for mk, nm in ((2, "score end (warp 0)"), (17, "CTA scored (all warps)"), (5, "gather done")):
            by_rank = np.stack([r[:B * Hq * nct, mk].reshape(B * Hq, nct) for r in rows])
            print(f"{nm} by cluster rank (median / max, us):",
                  [(round(float(np.median(by_rank[..., c])) / 1e3, 2), round(float(by_rank[..., c].max()) / 1e3, 2))
                   for c in range(nct)])
            spread = by_rank.max(-1) - by_rank.min(-1)  # inside each cluster
            print(f"  {nm}: spread inside a cluster (us) percentiles 10/50/90",
                  np.round(np.percentile(spread, [10, 50, 90]) / 1e3, 2))
    t = np.concatenate(rows)
    print(f"{a.config}: {len(rows)} steps, {t.shape[0] // len(rows)} CTAs per step (us since first CTA start)")
    for i, nm in enumerate(NAMES):
        v = t[:, i]
        v = v[v >= 0]
        v = v[v < 10**7]
        if len(v):
            print(f"  {i} {nm:11s} median {np.median(v) / 1e3:8.2f}  max {v.max() / 1e3:8.2f}")
    if a.raw:  # probe slots (cycles), not timestamps
        r = np.concatenate(raws)
        for i in a.raw:
            v = r[:, i]
            v = v[(v > 0) & (v < 10**7)]
            if len(v):
                print(f"  raw slot {i}: percentiles 10/50/90 {np.percentile(v, [10, 50, 90])}")
    for i, j in a.pairs:  # per-CTA interval between two marks (timer resolution check)
        d = t[:, j] - t[:, i]  # the per-step offset cancels (also for clock64 marks)
        d = d[(d > 0) & (d < 10**8)]
        if len(d):
            print(f"  {NAMES[i]} -> {NAMES[j]}: ns percentiles 10/50/90 {np.percentile(d, [10, 50, 90])}, "
                  f"distinct values {len(np.unique(d))}, smallest {np.unique(d)[:6]}")


if __name__ == "__main__":
    main()
