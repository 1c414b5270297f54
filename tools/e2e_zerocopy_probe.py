import sys, os, torch, math
sys.path.insert(0, os.getcwd())
import bench, paper_2508_08256_b200 as F
cfg = bench.CONFIGS["c2"]; dev = torch.device("cuda")
B, Hq, Hkv, L, d, n, g = (cfg[k] for k in ("B", "Hq", "Hkv", "L", "d", "n", "g"))
pos = L - 1
layers, hin, hout = [], [], []
for i in range(4):
    K, V, q, kn, vn = bench.make_inputs(cfg, 1234 + i, dev)
    lay = F.DecodeLayer(B, Hq, Hkv, L, d, g, dtype=K.dtype, device=dev, K=K, V=V); lay.prefill(pos); lay.workspace(pos+1, n)
    layers.append(lay); hin.append(tuple(t.cpu().pin_memory() for t in (q, kn, vn)))
    hout.append(torch.empty((B, Hq, d), dtype=torch.float32).pin_memory())
sels = [torch.empty((B, Hq, n), dtype=torch.int32, device=dev) for _ in range(4)]
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
def step(li):
    q, kn, vn = hin[li]
    layers[li].step(q, kn, vn, pos, n, out=hout[li], sel=sels[li])
for li in range(4): step(li)
torch.cuda.synchronize()
g_ = torch.cuda.CUDAGraph()
with torch.cuda.graph(g_, stream=st):
    for li in range(4): step(li)
for _ in range(5): g_.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(250): g_.replay()
e1.record(st); torch.cuda.synchronize()
print("zero-copy e2e us/step", e0.elapsed_time(e1) * 1000 / 1000)
# correctness vs device-input step
qd, knd, vnd = (t.to(dev) for t in hin[0])
o2 = torch.empty((B, Hq, d), device=dev)
layers[0].step(qd, knd, vnd, pos, n, out=o2, sel=sels[0]); torch.cuda.synchronize()
print("max diff", (o2.cpu() - hout[0]).abs().max().item())
