"""Cross-check of K0 (fier_full_attention, the full-KV decode baseline) against FlashInfer's
single-request decode kernel (library code): same inputs, output agreement and
device time per layer (CUDA events, layer instances rotated so K/V come from HBM).

  python tools/flashinfer_k0.py [--config c2] [--layers 4] [--reps 20]
"""
import argparse
import ctypes as C
import math
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2508_08256_b200 as F  # noqa: E402
from paper_2508_08256_b200 import _lib  # noqa: E402
from paper_2508_08256_b200.api import _p, _stream  # noqa: E402


def time_rotating(fn, n_layers, reps):
    for i in range(n_layers):
        fn(i)
    torch.cuda.synchronize()
    out = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in range(reps):
            fn(r % n_layers)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1000.0 / reps)
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import flashinfer
    cfg = bench.CONFIGS[a.config]
    assert cfg["B"] == 1, "single-request decode only"
    dev = torch.device("cuda")
    lib = _lib.load()
    Hq, Hkv, L, d, g = cfg["Hq"], cfg["Hkv"], cfg["L"], cfg["d"], cfg["g"]
    layers, qs = [], []
    for i in range(a.layers):
        K, V, q, _, _ = bench.make_inputs(cfg, 1234 + i, dev)
        layers.append(F.DecodeLayer(1, Hq, Hkv, L, d, g, dtype=K.dtype, device=dev, K=K, V=V))
        qs.append(q)
    scale = 1.0 / math.sqrt(d)
    outs = [torch.empty((1, Hq, d), device=dev) for _ in layers]
    ws = torch.zeros(lib.fier_full_attention_workspace(C.byref(layers[0].shape), L), dtype=torch.uint8, device=dev)

    def k0(i):
        lay = layers[i]
        _lib.check(lib.fier_full_attention(C.byref(lay.shape), _p(qs[i]), _p(lay.K), _p(lay.V), L, scale,
                                           _p(outs[i]), _p(ws), ws.numel(), _stream()))

    fi_out = [None] * len(layers)

    def fi(i):  # K/V [Hkv, L, d] per request = FlashInfer's HND layout
        fi_out[i] = flashinfer.single_decode_with_kv_cache(qs[i][0], layers[i].K[0], layers[i].V[0],
                                                           kv_layout="HND", sm_scale=scale)

    k0(0)
    fi(0)
    torch.cuda.synchronize()
    ref = (torch.softmax((layers[0].K[0].float().repeat_interleave(Hq // Hkv, 0) @ qs[0][0].float()[:, :, None])
                         .squeeze(-1) * scale, -1)[:, None, :]
           @ layers[0].V[0].float().repeat_interleave(Hq // Hkv, 0)).squeeze(1)
    rel = lambda x: float((x.float() - ref).norm() / ref.norm())  # noqa: E731
    t_k0 = time_rotating(k0, a.layers, a.reps)
    t_fi = time_rotating(fi, a.layers, a.reps)
    byts = bench.full_kv_bytes(cfg)
    print(f"{a.config}: K0 {t_k0:.2f} us ({byts / t_k0 / 1e3:.0f} GB/s), FlashInfer single_decode {t_fi:.2f} us "
          f"({byts / t_fi / 1e3:.0f} GB/s), K0/FlashInfer time {t_k0 / t_fi:.3f}; rel-L2 vs fp32 torch: "
          f"K0 {rel(outs[0][0]):.2e}, FlashInfer {rel(fi_out[0]):.2e}, K0 vs FlashInfer "
          f"{float((outs[0][0] - fi_out[0].float()).norm() / fi_out[0].float().norm()):.2e}")


if __name__ == "__main__":
    main()
