"""Run one golden case through quantize -> approx_scores -> topk -> gather (debug helper)."""
import sys
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import load_golden
import paper_2508_08256_b200 as F

name = sys.argv[1] if len(sys.argv) > 1 else "full_budget"
c = load_golden(name)
dt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[c["dtype"]]
K = torch.from_numpy(c["K"]).cuda().to(dt).unsqueeze(0)
V = torch.from_numpy(c["V"]).cuda().to(dt).unsqueeze(0)
Q = torch.from_numpy(c["Q"]).cuda().to(dt).unsqueeze(0)
pk = F.quantize(K, c["g"]); torch.cuda.synchronize(); print("quantize ok")
est = F.approx_scores(Q, pk); torch.cuda.synchronize(); print("score ok")
sel = F.topk_oracle(est, c["n"]); torch.cuda.synchronize(); print("topk ok", sel[0, 0, :8].tolist())
out = F.gather_attention(Q, K, V, sel); torch.cuda.synchronize(); print("attn ok")
