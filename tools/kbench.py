"""Per-kernel timing probe (CUDA events): each C-ABI kernel of the decode step
timed in isolation, on one layer repeated (warm L2/TLB) vs rotated layers.

  python tools/kbench.py [--config c2] [--layers 4] [--reps 50]
"""
import argparse
import ctypes as C
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2508_08256_b200 as F  # noqa: E402
from paper_2508_08256_b200 import _lib  # noqa: E402
from paper_2508_08256_b200.api import _p, _stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    dev = torch.device("cuda")
    lib = _lib.load()
    B, Hq, Hkv, L, d, n, g = (cfg[k] for k in ("B", "Hq", "Hkv", "L", "d", "n", "g"))
    pos = L - 1
    layers, inp = [], []
    for i in range(a.layers):
        K, V, q, kn, vn = bench.make_inputs(cfg, 1234 + i, dev)
        lay = F.DecodeLayer(B, Hq, Hkv, L, d, g, dtype=K.dtype, device=dev, K=K, V=V)
        lay.prefill(pos)
        layers.append(lay)
        inp.append((q, kn, vn))
    ld = lib.fier_step_scores_ld(pos + 1)
    sc = [torch.empty((B, Hq, ld), device=dev) for _ in layers]
    sel = [torch.empty((B, Hq, n), dtype=torch.int32, device=dev) for _ in layers]
    out = [torch.empty((B, Hq, d), device=dev) for _ in layers]
    wsb = lib.fier_sparse_attention_workspace(C.byref(layers[0].shape), n)
    ws = [torch.zeros(wsb, dtype=torch.uint8, device=dev) for _ in layers]
    fwb = lib.fier_full_attention_workspace(C.byref(layers[0].shape), pos + 1)
    fws = torch.zeros(fwb, dtype=torch.uint8, device=dev)

    def k_append(i):
        lay, (q, kn, vn) = layers[i], inp[i]
        _lib.check(lib.fier_append(C.byref(lay.shape), _p(lay.K), _p(lay.V), _p(kn), _p(vn), pos,
                                   _p(lay.pk.bits), _p(lay.pk.params), None, _stream()))

    def k_score(i):
        lay, (q, _, _) = layers[i], inp[i]
        _lib.check(lib.fier_score(C.byref(lay.shape), _p(q), _p(lay.pk.bits), _p(lay.pk.params), pos + 1,
                                  _p(sc[i]), ld, _stream()))

    tws_b = lib.fier_topk_workspace(B * Hq, pos + 1, n)
    tws = torch.empty(max(tws_b, 1), dtype=torch.uint8, device=dev)

    def k_topk(i):  # with the workspace, as in the decode step
        _lib.check(lib.fier_topk(_p(sc[i]), B * Hq, pos + 1, ld, n, _p(sel[i]), _p(tws), tws_b, _stream()))

    def k_attn(i):
        lay, (q, _, _) = layers[i], inp[i]
        _lib.check(lib.fier_sparse_attention(C.byref(lay.shape), _p(q), _p(lay.K), _p(lay.V), _p(sel[i]), n,
                                             pos + 1, 1 / math.sqrt(d), _p(out[i]), _p(ws[i]), wsb, _stream()))

    def k_full(i):
        lay, (q, _, _) = layers[i], inp[i]
        _lib.check(lib.fier_full_attention(C.byref(lay.shape), _p(q), _p(lay.K), _p(lay.V), pos + 1,
                                           1 / math.sqrt(d), _p(out[i]), _p(fws), fwb, _stream()))

    def k_chain(i):  # the separate kernels back to back, no append
        k_score(i), k_topk(i), k_attn(i)

    def k_append_chain(i):  # fier_append then the chain (the step's work in four launches)
        k_append(i), k_chain(i)

    def k_step(i):  # the decode step itself (fused append in the scorer on the GQA path)
        lay, (q, kn, vn) = layers[i], inp[i]
        lay.step(q, kn, vn, pos, n, out=out[i], sel=sel[i])

    for i in range(a.layers):  # populate scores/selections
        k_append(i), k_score(i), k_topk(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    for name, fn in [("append", k_append), ("score", k_score), ("topk", k_topk), ("sparse_attn", k_attn),
                     ("full_attn", k_full), ("chain", k_chain), ("append+chain", k_append_chain), ("step", k_step)]:
        res = []
        for mode in ("same", "rotate"):
            # one CUDA graph of `reps` launches: GPU time without host launch overhead
            fn(0)
            torch.cuda.synchronize()
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, stream=stream):
                for r in range(a.reps):
                    fn(0 if mode == "same" else r % a.layers)
            gph.replay()
            torch.cuda.synchronize()
            s.record(stream)
            gph.replay()
            e.record(stream)
            torch.cuda.synchronize()
            res.append(s.elapsed_time(e) * 1000 / a.reps)
        print(f"{name:12s} same-layer {res[0]:8.2f} us   rotating {res[1]:8.2f} us")


if __name__ == "__main__":
    main()
