import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2508_08256_b200 as F
s = torch.randn(32, 1 << 20, device="cuda") * 8
for _ in range(3): F.topk_oracle(s, 4096)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): F.topk_oracle(s, 4096)
e1.record(); torch.cuda.synchronize()
print("topk 32 x 1M, k=4096:", e0.elapsed_time(e1) * 100, "us")
