"""Throughput of the device-side FIER / KVD1 stream kernels (csrc/fier_io.cu).

  python tools/io_bench.py [--tokens 1048576] [--reps 20]

Bytes counted = bytes read + bytes written by the kernels (the stream and the index /
fp32 values), timed with CUDA events on the launching stream after warm-up.
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
    return a.elapsed_time(b) * 1e3 / reps  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda")
    l, d, g = a.tokens, 128, 32
    K = torch.randn(1, 1, l, d, device=dev).to(torch.bfloat16)
    pk = F.quantize(K, g)
    stream = pk.to_fier_device()
    nb = stream.numel()
    t_exp = timed(lambda: pk.to_fier_device(), a.reps)
    t_imp = timed(lambda: F.PackedKeys.from_fier_device(stream), a.reps)
    print(f"FIER l={l} d={d} g={g}: {nb / 1e6:.1f} MB stream; export {t_exp:.1f} us "
          f"({2 * nb / t_exp / 1e3:.0f} GB/s), import {t_imp:.1f} us ({2 * nb / t_imp / 1e3:.0f} GB/s, "
          f"incl. the 18-byte header read-back)")
    Kf = torch.randn(l // 8, d, device=dev)
    raw = F.save_cache_dump(Kf, Kf, None, dtype="f16")
    vals = 2 * Kf.numel()
    t_st = timed(lambda: F.save_cache_dump(Kf, Kf, None, dtype="f16"), a.reps)
    t_ld = timed(lambda: F.load_cache_dump(raw), a.reps)
    print(f"KVD1 f16 l={l // 8} d={d}: {raw.numel() / 1e6:.1f} MB stream; store {t_st:.1f} us (incl. the fp32 "
          f"concat), load {t_ld:.1f} us ({(raw.numel() + 4 * vals) / t_ld / 1e3:.0f} GB/s)")


if __name__ == "__main__":
    main()
