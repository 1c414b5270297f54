"""Run only the top-k kernel on C2-shaped scores (for ncu)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2508_08256_b200 as F
rows, L, k = int(sys.argv[1]) if len(sys.argv) > 1 else 32, 32768, 3604
g = torch.Generator(device="cuda").manual_seed(0)
s = torch.randn(rows, L, device="cuda", generator=g) * 16
for _ in range(3):
    sel = F.topk_oracle(s, k)
torch.cuda.synchronize()
print("ok", sel.shape)
