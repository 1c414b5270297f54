"""Quest page retrieval on the GPU at the C2 shape (csrc/quest.cu), next to Fier's own
per-step selection, plus the recall of each selection against exact top-n attention
scores on a planted-spike workload (a page-level vs token-level comparison).

  python tools/quest_bench.py [--reps 20]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_08256_b200 as F  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def recall(sel, want):
    s, w = sel.long(), want.long()
    hit = torch.zeros(s.shape[:-1] + (int(max(s.max(), w.max())) + 1,), dtype=torch.bool, device=s.device)
    hit.scatter_(-1, w, True)
    return float(hit.gather(-1, s).float().mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda")
    H, l, d, L, n, g = 32, 32768, 128, 16, 3604, 32
    torch.manual_seed(0)
    K = torch.randn(1, H, l, d, device=dev)
    q = torch.randn(1, H, d, device=dev)
    spikes = torch.randint(0, l, (H, 64), device=dev)  # tokens aligned with q
    for h in range(H):
        K[0, h, spikes[h]] += 3.0 * q[0, h] / q[0, h].norm() * d ** 0.5 / 4
    K, q = K.to(torch.bfloat16), q.to(torch.bfloat16)
    exact = torch.einsum("bhd,bhld->bhl", q.float(), K.float())
    want = torch.topk(exact, n, dim=-1).indices.sort(-1).values
    ps = F.build_page_summaries(K, L)
    pk = F.quantize(K, g)
    t_sum = timed(lambda: F.build_page_summaries(K, L), a.reps)
    t_q = timed(lambda: F.quest_select(q, K, ps, n, "sum"), a.reps)
    t_qq = timed(lambda: F.quest_select_quantized(q, pk, L, n), a.reps)
    t_f = timed(lambda: F.topk_oracle(F.approx_scores(q, pk), n), a.reps)
    r_q = recall(F.quest_select(q, K, ps, n, "sum"), want)
    r_qm = recall(F.quest_select(q, K, ps, n, "max"), want)
    r_qq = recall(F.quest_select_quantized(q, pk, L, n), want)
    r_f = recall(F.topk_oracle(F.approx_scores(q, pk), n), want)
    print(f"C2 shape (32 heads, l={l}, d={d}, page {L}, n={n}, bf16), planted spikes:")
    print(f"  page summaries (prefill-time) {t_sum:.1f} us")
    print(f"  quest_select (sum)            {t_q:.1f} us   recall@n {r_q:.3f}  (max variant {r_qm:.3f})")
    print(f"  quest_select_quantized        {t_qq:.1f} us   recall@n {r_qq:.3f}")
    print(f"  fier select (K2 + K3)         {t_f:.1f} us   recall@n {r_f:.3f}")


if __name__ == "__main__":
    main()
