"""A recall / output-error sweep at long context on the GPU (harness.run_trial, SURVEY
§8(f) row 4): Fier vs Quest vs quantized Quest vs the exact top-n, one head.

  python tools/recall_sweep.py [--l 131072] [--queries 4]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_08256_b200 import harness  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--l", type=int, default=131072)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--queries", type=int, default=4)
    a = ap.parse_args()
    dev = torch.device("cuda")
    torch.manual_seed(0)
    K = torch.randn(a.l, a.d, device=dev)
    V = torch.randn(a.l, a.d, device=dev)
    Q = torch.randn(a.queries, a.d, device=dev)
    for i in range(a.queries):  # each query has 64 planted matches
        idx = torch.randint(0, a.l, (64,), device=dev)
        K[idx] += 0.75 * Q[i] / Q[i].norm() * a.d ** 0.5
    budgets = [a.l // 64, a.l // 16, a.l // 9]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = harness.run_trial(K, V, Q, budgets)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"run_trial on the GPU: l={a.l}, d={a.d}, {a.queries} queries, budgets {budgets}: {dt:.2f} s wall")
    print(f"{'policy':12s} " + " ".join(f"{'n=' + str(n):>24s}" for n in budgets))
    for p, m in t.cells.items():
        print(f"{p:12s} " + " ".join(f"recall {r:.3f} err {e:.3f}".rjust(24) for r, e in zip(m["recall"], m["out_err"])))
    print("margins " + " ".join(f"{x:.4g}" for x in t.margins))


if __name__ == "__main__":
    main()
