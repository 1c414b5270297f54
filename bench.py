#!/usr/bin/env python
"""Fier decode-step benchmark (BASELINE.json metric: "Fier decode µs/layer & HBM GB/s at
32k ctx; speedup vs full-KV attn").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one decode step of one attention layer: append the new token
(write k/v row + re-pack its open group) -> score every token from the packed
keys -> per-head Top-n -> sparse attention over the selected rows.  Inputs
(the per-step q, k_new, v_new) are resident in HBM for `value`; `e2e` passes
pinned HOST buffers for the inputs and the output to the public step
(DecodeLayer.step -> fier_decode_step), so every step moves them across the
host link inside the timed region (`dma_variant_us`: the same with explicit
H2D/D2H copies).  The KV caches of several layer instances are rotated, one
CUDA graph per rotation, so the bytes touched between visits exceed 2x L2
(config.l2).  N > 1 (torchrun): every rank runs its own independent sequence
(weak scaling, no data-path collective); time = max over ranks.

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from the reference's headers) of the same step on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Fier decode µs/layer & HBM GB/s at 32k ctx; speedup vs full-KV attn"
UNIT = "us/step"

CONFIGS = {
    "c1": dict(B=1, Hq=32, Hkv=32, L=4096, d=128, n=512, g=32, dtype="f32",
               desc="C1: single-layer decode, 32 MHA heads, d=128, 4k ctx, fp32, Top-k 512"),
    "c2": dict(B=1, Hq=32, Hkv=32, L=32768, d=128, n=3604, g=32, dtype="bf16",
               desc="C2: LLaMA-2-7B decode layer, 32 MHA heads, d=128, 32k ctx, 11% budget "
                    "(n=3604), batch 1, bf16"),
    "c3": dict(B=1, Hq=32, Hkv=8, L=131072, d=128, n=4096, g=32, dtype="bf16",
               desc="C3: Llama-3-8B GQA layer (32 q / 8 kv), d=128, 128k ctx, n=4096, batch 1, bf16"),
    "c4": dict(B=32, Hq=32, Hkv=8, L=32768, d=128, n=3604, g=32, dtype="bf16",
               desc="C4: batched decode, batch 32, 32k ctx, Llama-3-8B GQA shape, 11% budget, bf16"),
    "c5": dict(B=1, Hq=32, Hkv=8, L=1048576, d=128, n=4096, g=32, dtype="bf16",
               desc="C5: 1M-token context, Llama-3-8B GQA layer, n=4096, sequence-sharded over the GPUs "
                    "(per-shard Top-k + candidate all-gather + LSE merge over NVLink)"),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def elem_size(dt: str) -> int:
    return 4 if dt == "f32" else 2


def algorithmic_bytes(cfg, unique_rows=None):
    """packed keys + selected K/V rows + Q/O, per step (one layer)."""
    B, Hq, Hkv, L, d, n, g = (cfg[k] for k in ("B", "Hq", "Hkv", "L", "d", "n", "g"))
    es = elem_size(cfg["dtype"])
    packed = B * Hkv * (L * ((d + 7) // 8) + ((L + g - 1) // g) * d * 4)
    rows = B * Hq * n if unique_rows is None else unique_rows
    kv = rows * d * 2 * es
    qo = B * Hq * d * (es + 4)  # q in the cache dtype, o in fp32
    return packed, kv, qo


def full_kv_bytes(cfg):
    es = elem_size(cfg["dtype"])
    return cfg["B"] * cfg["Hkv"] * cfg["L"] * cfg["d"] * 2 * es + cfg["B"] * cfg["Hq"] * cfg["d"] * (es + 4)


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
             0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
             0x2: "applications_clocks_setting", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.NAMES.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        self.sample()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()
        self.sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo", device_id=torch.device("cuda", local)
                                if args.impl == "ours" else None)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_inputs(cfg, seed, device):
    """Synthetic random-init Q/K/V of the named shape (torch Philox, fixed seed)."""
    import torch
    dt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[cfg["dtype"]]
    gen = torch.Generator(device=device).manual_seed(seed)
    B, Hq, Hkv, L, d = cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["L"], cfg["d"]
    K = torch.randn((B, Hkv, L, d), generator=gen, device=device, dtype=torch.float32).to(dt)
    V = torch.randn((B, Hkv, L, d), generator=gen, device=device, dtype=torch.float32).to(dt)
    q = torch.randn((B, Hq, d), generator=gen, device=device, dtype=torch.float32).to(dt)
    kn = torch.randn((B, Hkv, d), generator=gen, device=device, dtype=torch.float32).to(dt)
    vn = torch.randn((B, Hkv, d), generator=gen, device=device, dtype=torch.float32).to(dt)
    return K, V, q, kn, vn


# ---------------------------------------------------------------------------------------
def run_ours(args, cfg, world, rank, local):
    import torch

    import paper_2508_08256_b200 as F
    from paper_2508_08256_b200 import _lib
    from paper_2508_08256_b200.api import _p, _stream

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    lib = _lib.load()
    B, Hq, Hkv, L, d, n, g = (cfg[k] for k in ("B", "Hq", "Hkv", "L", "d", "n", "g"))
    pos = L - 1  # the step appends token L-1: a decode step at context L
    packed, kvb, qo = algorithmic_bytes(cfg)
    touched = packed + kvb + qo
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    n_layers = max(1, min(16, math.ceil(2.5 * l2 / touched)))
    if args.layers:
        n_layers = args.layers
    layers, inputs = [], []
    for i in range(n_layers):
        K, V, q, kn, vn = make_inputs(cfg, 1234 + 1000 * rank + i, dev)
        layer = F.DecodeLayer(B, Hq, Hkv, L, d, g, dtype=K.dtype, device=dev, K=K, V=V)
        layer.prefill(pos)
        layer.workspace(pos + 1, n)
        layers.append(layer)
        inputs.append((q, kn, vn))
    outs = [torch.empty((B, Hq, d), dtype=torch.float32, device=dev) for _ in range(n_layers)]
    sels = [torch.empty((B, Hq, n), dtype=torch.int32, device=dev) for _ in range(n_layers)]
    torch.cuda.synchronize()

    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    def step(i):
        li = i % n_layers
        q, kn, vn = inputs[li]
        layers[li].step(q, kn, vn, pos, n, out=outs[li], sel=sels[li])

    # CUDA graphs: one per layer instance, and one with a step of every instance back to back
    # (the layers of a decode step; no host gap between them).  K steps = K // n_layers
    # replays of the rotation graph + the remainder as single-layer graphs: exactly K steps.
    graphs = []
    for li in range(n_layers):
        step(li)  # warm the plan / attributes outside capture
    torch.cuda.synchronize()
    for li in range(n_layers):
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=stream):
            step(li)
        graphs.append(gph)
    rot = torch.cuda.CUDAGraph()
    with torch.cuda.graph(rot, stream=stream):
        for li in range(n_layers):
            step(li)
    torch.cuda.synchronize()

    def run_steps(k):
        for _ in range(k // n_layers):
            rot.replay()
        for i in range(k % n_layers):
            graphs[i].replay()

    run_steps(max(args.warmup, 1))
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record(stream)
        run_steps(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ms = max_over_ranks(ms, world)
    us_per_step = ms * 1000.0 / args.steps

    # ---- per-kernel breakdown: each C-ABI kernel alone, `reps` launches captured in one
    # CUDA graph rotating over the layer instances (no host gaps), CUDA events on `stream` ----
    import ctypes as C
    ld = lib.fier_step_scores_ld(pos + 1)
    scores = [torch.empty((B, Hq, ld), dtype=torch.float32, device=dev) for _ in range(n_layers)]
    part_bytes = lib.fier_sparse_attention_workspace(C.byref(layers[0].shape), n)
    parts = [torch.zeros(part_bytes, dtype=torch.uint8, device=dev) for _ in range(n_layers)]
    fws = torch.zeros(lib.fier_full_attention_workspace(C.byref(layers[0].shape), pos + 1),
                      dtype=torch.uint8, device=dev)

    def k_append(li):
        lay, (q, kn, vn) = layers[li], inputs[li]
        _lib.check(lib.fier_append(C.byref(lay.shape), _p(lay.K), _p(lay.V), _p(kn), _p(vn), pos,
                                   _p(lay.pk.bits), _p(lay.pk.params), None, _stream()))

    def k_score(li):
        lay, (q, _, _) = layers[li], inputs[li]
        _lib.check(lib.fier_score(C.byref(lay.shape), _p(q), _p(lay.pk.bits), _p(lay.pk.params), pos + 1,
                                  _p(scores[li]), ld, _stream()))

    tws_b = lib.fier_topk_workspace(B * Hq, pos + 1, n)
    tws = torch.empty(max(tws_b, 1), dtype=torch.uint8, device=dev)

    def k_topk(li):  # with the workspace, as in the decode step
        _lib.check(lib.fier_topk(_p(scores[li]), B * Hq, pos + 1, ld, n, _p(sels[li]), _p(tws), tws_b,
                                 _stream()))

    def k_attn(li):
        lay, (q, _, _) = layers[li], inputs[li]
        _lib.check(lib.fier_sparse_attention(C.byref(lay.shape), _p(q), _p(lay.K), _p(lay.V), _p(sels[li]), n,
                                             pos + 1, 1.0 / math.sqrt(d), _p(outs[li]), _p(parts[li]),
                                             parts[li].numel(), _stream()))

    def k_full(li):
        lay, (q, _, _) = layers[li], inputs[li]
        _lib.check(lib.fier_full_attention(C.byref(lay.shape), _p(q), _p(lay.K), _p(lay.V), pos + 1,
                                           1.0 / math.sqrt(d), _p(outs[li]), _p(fws), fws.numel(), _stream()))

    def graph_time(fn, reps):
        """Average device time of one launch: `reps` launches (rotating layers) in one graph."""
        for li in range(n_layers):
            fn(li)
        torch.cuda.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=stream):
            for r in range(reps):
                fn(r % n_layers)
        gph.replay()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = []
        for _ in range(3):
            s0.record(stream)
            gph.replay()
            s1.record(stream)
            torch.cuda.synchronize()
            best.append(s0.elapsed_time(s1) * 1000.0 / reps)
        return statistics.median(best)

    kreps = max(4 * n_layers, 40)
    launches = layers[0].launches(pos + 1, n)
    fused_us = graph_time(step, kreps) if launches == 1 else None  # the one-launch step kernel alone
    for li in range(n_layers):  # scores/selections of every layer for the isolated K3/K4 runs
        k_score(li)
        k_topk(li)
    per = {"append": graph_time(k_append, kreps), "score": graph_time(k_score, kreps),
           "topk": graph_time(k_topk, kreps), "sparse_attn": graph_time(k_attn, kreps)}
    for li in range(n_layers):  # restore every layer's selection from the step itself
        step(li)
    # ---- K0: in-house full-KV decode attention on the same caches (the speedup baseline) ----
    full_us = graph_time(k_full, max(2 * n_layers, 20))

    # ---- e2e: public API with host buffers, H2D + step + D2H inside the timed region ----
    # q, k_new, v_new of a step travel in one pinned buffer (one H2D copy), the output back in one D2H
    def pack_inputs(inp):
        return torch.cat([t.reshape(-1) for t in inp]), [t.numel() for t in inp]

    hpack = [pack_inputs(inp)[0].cpu().pin_memory() for inp in inputs]
    sizes = pack_inputs(inputs[0])[1]
    dpack = [torch.empty_like(h, device=dev) for h in hpack]
    dviews = []
    for li in range(n_layers):
        parts, off = [], 0
        for t, sz in zip(inputs[li], sizes):
            parts.append(dpack[li][off:off + sz].view(t.shape))
            off += sz
        dviews.append(parts)
    hout = [torch.empty((B, Hq, d), dtype=torch.float32).pin_memory() for _ in range(n_layers)]
    h2d = hpack[0].numel() * hpack[0].element_size()
    d2h = hout[0].numel() * 4

    def e2e_step(li):
        dpack[li].copy_(hpack[li], non_blocking=True)
        q_, kn_, vn_ = dviews[li]
        layers[li].step(q_, kn_, vn_, pos, n, out=outs[li], sel=sels[li])
        hout[li].copy_(outs[li], non_blocking=True)

    egraphs = []
    for li in range(n_layers):
        e2e_step(li)
    torch.cuda.synchronize()
    for li in range(n_layers):
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=stream):
            e2e_step(li)
        egraphs.append(gph)
    erot = torch.cuda.CUDAGraph()
    with torch.cuda.graph(erot, stream=stream):
        for li in range(n_layers):
            e2e_step(li)
    for _ in range(max(1, args.warmup // n_layers)):
        erot.replay()
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps // n_layers):
        erot.replay()
    for i in range(args.steps % n_layers):
        egraphs[i].replay()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_dma_us = max_over_ranks(e0.elapsed_time(e1), world) * 1000.0 / args.steps

    # zero-copy variant (the reported e2e): fier_decode_step gets the pinned HOST pointers of
    # q, k_new, v_new and of the output; the kernel reads the 24 KB of inputs over the host
    # link and writes the result straight to host memory -- no DMA copy nodes in the step.
    hin = [tuple(t.cpu().pin_memory() for t in inp) for inp in inputs]

    def zc_step(li):
        q_, kn_, vn_ = hin[li]
        layers[li].step(q_, kn_, vn_, pos, n, out=hout[li], sel=sels[li], host_inputs=True)

    zgraphs = []
    for li in range(n_layers):
        zc_step(li)
    torch.cuda.synchronize()
    for li in range(n_layers):
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=stream):
            zc_step(li)
        zgraphs.append(gph)
    zrot = torch.cuda.CUDAGraph()
    with torch.cuda.graph(zrot, stream=stream):
        for li in range(n_layers):
            zc_step(li)
    for _ in range(max(1, args.warmup // n_layers)):
        zrot.replay()
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps // n_layers):
        zrot.replay()
    for i in range(args.steps % n_layers):
        zgraphs[i].replay()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_us = max_over_ranks(e0.elapsed_time(e1), world) * 1000.0 / args.steps

    # unique (kv head, token) rows actually selected (GQA overlap), last step of layer 0
    s0 = sels[0].view(B, Hkv, Hq // Hkv, n).long()
    key = (torch.arange(B * Hkv, device=dev).view(B, Hkv, 1, 1) * L + s0).flatten()
    unique_rows = int(torch.unique(key).numel())

    # ---- roofline of the dominant kernel ----
    peak, peak_src = peaks()
    es = elem_size(cfg["dtype"])
    alg = {
        "score": packed + B * Hq * d * es,
        # U = unique selected (kv head, token) rows (the GQA q heads of a group share
        # rows through L2); U = B*Hq*n for MHA
        "sparse_attn": unique_rows * d * 2 * es + qo,
        "append": B * Hkv * (g * d * es + 2 * d * es + g * d // 8 + d * 4),
        # the scratch scores are read at least once (not SURVEY §8(d) algorithmic bytes of the
        # step, but what bounds a Top-k kernel from below)
        "topk": B * Hq * (pos + 1) * 4,
    }
    pk_u, kv_u, qo_u = algorithmic_bytes(cfg, unique_rows)
    dom = max(per, key=per.get)
    if fused_us is not None:  # one cluster kernel does append + score + Top-n + attention
        alg["fused_step"] = pk_u + kv_u + qo_u
        dom = "fused_step"
    gather_ceiling = None
    gpath = os.path.join(ROOT, "profiles", "gather_ceiling.json")
    if os.path.exists(gpath):
        gather_ceiling = json.load(open(gpath)).get("cold_l2_gbs")
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.config, {}).get(dom)
    roof = None
    t_dom = fused_us if dom == "fused_step" else per.get(dom)
    if alg.get(dom):
        ach = alg[dom] / (t_dom * 1e-6) / 1e9
        roof = {"bound": "hbm" if dom != "topk" else "latency (hbm bytes: one read of the scratch scores)",
                "kernel": "step_fused_kernel" if dom == "fused_step" else dom,
                "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "alg_bytes": alg[dom],
                "launch_us": round(t_dom, 3), "peak_source": peak_src}
        if dom == "sparse_attn" and gather_ceiling:
            # random 256-B row gathers at this density cap below the copy peak on B200
            # (tools/gather_probe.cu, profiles/gather_ceiling.json)
            roof["gather_ceiling_gbs"] = gather_ceiling
            roof["frac_of_gather_ceiling"] = round(ach / gather_ceiling, 4)
    step_bytes = packed + kvb + qo
    step_gbs = step_bytes / (us_per_step * 1e-6) / 1e9
    per_out = {k: round(v, 3) for k, v in per.items()}
    if fused_us is not None:  # the separate-kernel path's pieces, for comparison only
        per_out = {"fused_step": round(fused_us, 3), "unfused_components": per_out}
    res = {
        "launches_per_step": launches,
        "per_kernel_us": per_out,
        "roofline": roof,
        "step_roofline": {"alg_bytes": step_bytes, "alg_bytes_unique_rows": pk_u + kv_u + qo_u,
                          "unique_rows": unique_rows, "achieved_gbs": round(step_gbs, 1),
                          "frac_of_measured": round(step_gbs / peak, 4),
                          "frac_of_8TBs": round(step_gbs / 8000.0, 4)},
        "full_kv": {"us_per_step": round(full_us, 3),
                    "achieved_gbs": round(full_kv_bytes(cfg) / (full_us * 1e-6) / 1e9, 1),
                    "speedup_fier_vs_full": round(full_us / us_per_step, 3)},
        "e2e": {"value": round(e2e_us, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "how": "fier_decode_step_ex(FIER_STEP_HOST_INPUTS) on pinned host buffers: the one-launch step "
                       "kernel reads q/k_new/v_new from host memory itself; the separate-kernel path first stages "
                       "them into the workspace with one extra launch; the output is written to host memory "
                       "(zero-copy); one CUDA graph per layer rotation",
                "launches_per_step": layers[0].launches(pos + 1, n, host_inputs=True),
                "dma_variant_us": round(e2e_dma_us, 3)},
        "clocks": sampler.summary(),
        "n_layers": n_layers,
    }
    # data for the CPU baseline: layer 0's caches and step-0 query, exactly as the GPU saw them
    res["_cpu_inputs"] = (layers[0].K, layers[0].V, inputs[0])
    return us_per_step, ms, res


def run_sharded(args, cfg, world, rank, local):
    """C5 sequence-sharded over the N ranks (N = 1 with --sharded: the same protocol on one
    GPU): every step runs shard-local append/score/Top-k, one NCCL all-gather of the (score,
    index) candidates, the global merge, ragged K4 and a second all-gather of the (o, lse)
    partials (paper_2508_08256_b200.shard.sharded_step).  The whole step -- kernels and both
    collectives -- is captured in one CUDA graph per rank (eager if capture fails); device
    time with CUDA events, max over ranks.  e2e: the same step with q / k_new / v_new copied
    from pinned host memory and the output copied back, inside the timed region."""
    import torch
    import torch.distributed as dist

    from paper_2508_08256_b200.shard import DistExchange, NcclDeviceExchange, ShardedDecodeLayer, sharded_step

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if not dist.is_initialized():  # --sharded at N = 1: a one-rank NCCL group
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    B, Hq, Hkv, L, d, n, g = (cfg[k] for k in ("B", "Hq", "Hkv", "L", "d", "n", "g"))
    dt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[cfg["dtype"]]
    shard = ShardedDecodeLayer(B, Hq, Hkv, L, d, g, rank=rank, shards=world, dtype=dt, device=dev)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    shard.K.copy_(torch.randn(shard.K.shape, generator=gen, device=dev).to(dt))
    shard.V.copy_(torch.randn(shard.V.shape, generator=gen, device=dev).to(dt))
    gq = torch.Generator(device=dev).manual_seed(99)  # identical query / new token on every rank
    q = torch.randn((B, Hq, d), generator=gq, device=dev).to(dt)
    kn = torch.randn((B, Hkv, d), generator=gq, device=dev).to(dt)
    vn = torch.randn((B, Hkv, d), generator=gq, device=dev).to(dt)
    pos = L - 1
    shard.prefill(pos)
    if args.exchange == "device":  # the NCCL device API: LSA stores into symmetric windows + LSA barrier
        ex = NcclDeviceExchange(slot_bytes=max(2 * B * Hq * n * 4, B * Hq * (d + 1) * 4))
    else:  # host-launched ncclAllGather (torch.distributed)
        ex = DistExchange()
    stream = torch.cuda.Stream(device=dev)
    out_buf = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)

    def step():
        out_buf.copy_(sharded_step(shard, ex, q, kn, vn, pos, n))

    with torch.cuda.stream(stream):
        for _ in range(2):  # eager: buffers allocated, NCCL communicator warmed up
            step()
    torch.cuda.synchronize()
    graph = None
    try:
        g0 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g0, stream=stream):
            step()
        g0.replay()
        torch.cuda.synchronize()
        graph = g0
    except Exception as e:  # noqa: BLE001 -- fall back to eager launches, say so in the line
        print(f"[bench] graph capture of the sharded step failed ({e}); eager", file=sys.stderr)
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else step

    def timed(fn, steps):
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        return max_over_ranks(e0.elapsed_time(e1), world) * 1000.0 / steps

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            run()
    sampler = ClockSampler(local)
    with sampler:
        us = timed(run, args.steps)

    # e2e: q / k_new / v_new from pinned host memory (one H2D), the output back (one D2H)
    hin = torch.cat([q.reshape(-1), kn.reshape(-1), vn.reshape(-1)]).cpu().pin_memory()
    hout = torch.empty(out_buf.shape, dtype=torch.float32).pin_memory()
    din = torch.empty_like(hin, device=dev)
    nq, nk = q.numel(), kn.numel()

    def e2e_step():
        din.copy_(hin, non_blocking=True)
        q.copy_(din[:nq].view_as(q))
        kn.copy_(din[nq:nq + nk].view_as(kn))
        vn.copy_(din[nq + nk:].view_as(vn))
        run()
        hout.copy_(out_buf, non_blocking=True)

    with torch.cuda.stream(stream):
        for _ in range(3):
            e2e_step()
    e2e_us = timed(e2e_step, max(10, args.steps // 4))
    # per-rank algorithmic bytes: this shard's packed index + its share of the selected rows + q/o
    lt = shard.end - shard.start
    es = elem_size(cfg["dtype"])
    packed = B * Hkv * (lt * ((d + 7) // 8) + ((lt + g - 1) // g) * d * 4)
    sel = shard.sel_global
    rows = int(((sel >= shard.start) & (sel < shard.end)).sum().item()) if sel is not None else B * Hq * n // world
    alg = packed + rows * d * 2 * es + B * Hq * d * (es + 4)
    peak, src = peaks()
    ach = alg / (us * 1e-6) / 1e9
    info = {
        "graph": graph is not None,
        "exchange": args.exchange,
        "roofline": {"bound": "hbm", "kernel": "sharded step of one rank (all kernels + 2 all-gathers)",
                     "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                     "traffic": None, "alg_bytes": alg, "peak_source": src,
                     "note": "rank-local algorithmic bytes (its packed slice + its selected rows + q/o) over "
                             "the max-over-ranks step time"},
        "e2e": {"value": round(e2e_us, 3), "unit": UNIT, "h2d_bytes_per_step": hin.numel() * hin.element_size(),
                "d2h_bytes_per_step": hout.numel() * 4,
                "how": "q/k_new/v_new H2D from pinned memory + the captured sharded step + output D2H, per rank"},
        "launches_per_step": 8,
        "clocks": sampler.summary(),
    }
    return us, info


def cpu_baseline(cfg, K, V, inp, budget_s=20.0):
    """oracle/_ref (the reference compiled from its headers) on the host cores: a full
    decode step of this layer (every q head), all host threads, median of reps."""
    import numpy as np
    import torch

    from oracle.oracle import REF_SO, Port, Ref, RefLayer
    kind = "reference" if os.path.exists(REF_SO) else "port"
    threads = os.cpu_count() or 1
    q, kn, vn = inp
    b = 0
    Kc = K[b].float().cpu().numpy()
    Vc = V[b].float().cpu().numpy()
    Kc[:, -1] = kn[b].float().cpu().numpy()  # the appended token
    Vc[:, -1] = vn[b].float().cpu().numpy()
    Q = q[b].float().cpu().numpy()
    if kind != "reference":
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": "oracle/_ref missing; not timed"}
    ref = Ref()
    t0 = time.time()
    layer = RefLayer(ref, Kc, Vc, g=cfg["g"], threads=threads)
    build_s = time.time() - t0
    n = cfg["n"]
    Hq = cfg["Hq"]
    # first rep on all heads sizes the sample
    secs, _, _ = layer.step(Q, n)
    reps = [secs]
    while sum(reps) < budget_s / 4 and len(reps) < 5:
        reps.append(layer.step(Q, n)[0])
    layer.close()
    med = statistics.median(reps)
    scale = cfg["B"]  # the sample is one sequence of the batch
    return {"value": round(med * scale * 1e6, 1), "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"one full decode step of sequence 0 ({Hq} q heads, l={cfg['L']}, n={n}, fp64) x "
                      f"{scale} sequences, median of {len(reps)} reps; index built once ({build_s:.1f}s, "
                      f"hoisted)", "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------------------------------
def run_reference(args, cfg, world, rank):
    """The reference's own CPU path (oracle/_ref) on this host, same config/metric."""
    import numpy as np
    import torch

    from oracle.oracle import REF_SO, Ref, RefLayer
    if rank != 0:
        return None
    if not os.path.exists(REF_SO):
        return {"impl": "reference", "unavailable": "oracle/_ref/libfier_ref.so not built"}
    threads = os.cpu_count() or 1
    K, V, q, kn, vn = make_inputs(cfg, 1234, "cpu")
    Kc = K[0].float().numpy()
    Vc = V[0].float().numpy()
    Kc[:, -1] = kn[0].float().numpy()
    Vc[:, -1] = vn[0].float().numpy()
    Q = q[0].float().numpy()
    ref = Ref()
    layer = RefLayer(ref, Kc, Vc, g=cfg["g"], threads=threads)
    Hq, n = cfg["Hq"], cfg["n"]
    # size each timed step so the whole run stays within ~2 minutes
    t_full = layer.step(Q, n)[0]
    budget = 120.0
    heads = max(1, min(Hq, int(Hq * budget / max(1e-9, (args.steps + args.warmup) * t_full))))
    heads = max(heads, min(Hq, threads))
    times = []
    for i in range(args.warmup + args.steps):
        h0 = (i * heads) % Hq
        h1 = min(Hq, h0 + heads)
        secs = layer.step(Q, n, heads=(h0, h1))[0] * Hq / (h1 - h0)
        if i >= args.warmup:
            times.append(secs)
    layer.close()
    us = statistics.mean(times) * 1e6 * cfg["B"]
    sample = (f"each step: fier_attend (approx_scores -> topk_oracle -> gather_attention, fp64) over "
              f"{heads} of {Hq} q heads of sequence 0, scaled x{Hq}/{heads} heads and x{cfg['B']} "
              f"sequences; {threads} std::threads; index hoisted (quantize once)")
    return {
        "impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(us / 1000.0, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (torch Philox seed 1234, bf16-rounded, widened to fp64)",
        "config": config_block(args, cfg, world),
        "cpu_baseline": {"value": round(us, 1), "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample, "cpu": _cpu_model()},
        "e2e": {"value": round(us, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def config_block(args, cfg, world, n_layers=None, touched=None):
    c = {"workload": cfg["desc"], "batch": cfg["B"], "q_heads": cfg["Hq"], "kv_heads": cfg["Hkv"],
         "context": cfg["L"], "head_dim": cfg["d"], "budget_n": cfg["n"], "group_g": cfg["g"],
         "parallelism": f"replicas x{world} (independent sequences, no collective)" if world > 1 else "1 GPU",
         "config_id": args.config}
    if n_layers:
        c["l2"] = (f"inputs larger than L2: {n_layers} layer instances rotated, "
                   f"{n_layers * touched / 1e6:.0f} MB touched per rotation")
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 at N = 1 (the headline), c5 sequence-sharded at N > 1")
    ap.add_argument("--sharded", action="store_true", help="c5: run the sharded protocol even at N = 1")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "device"],
                    help="sharded step: host-launched NCCL all-gathers, or the NCCL device-API kernel")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=0, help="override the layer-rotation count")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup(args)
    if args.config is None:  # N > 1 exercises the sequence-sharded exchange
        args.config = "c5" if world > 1 and args.impl == "ours" else "c2"
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        out = run_reference(args, cfg, world, rank)
        if rank == 0 and out is not None:
            print(json.dumps(out))
        return

    if args.config == "c5" and (world > 1 or args.sharded):
        us, info = run_sharded(args, cfg, world, rank, local)
        if rank == 0:
            packed, kvb, qo = algorithmic_bytes(cfg)
            print(json.dumps({
                "metric": METRIC, "value": round(us, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(us / 1000.0, 6), "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"],
                "data": "synthetic random-init Q/K/V (torch Philox), prefix index pre-packed",
                "config": dict(config_block(args, cfg, world),
                               parallelism=f"sequence-sharded x{world} ({'NCCL device-API exchange' if info['exchange'] == 'device' else 'NCCL all-gathers'}, CUDA graph: "
                                           f"{info['graph']})",
                               l2="inputs larger than L2: each rank streams its whole slice (>= 134 MB of "
                                  "K/V + index per rank at N <= 8) every step"),
                "roofline": info["roofline"], "cpu_baseline": None, "e2e": info["e2e"],
                "gpu_launches": args.steps * info["launches_per_step"], "clocks": info["clocks"],
                "alg_bytes_per_step": packed + kvb + qo}))
        import torch.distributed as dist
        dist.destroy_process_group()
        return
    us, ms, res = run_ours(args, cfg, world, rank, local)
    K, V, inp = res.pop("_cpu_inputs")
    if rank == 0:
        packed, kvb, qo = algorithmic_bytes(cfg)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, K, V, inp)
        line = {
            "metric": METRIC, "value": round(us, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(us / 1000.0, 6),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic random-init Q/K/V (torch Philox), prefix index pre-packed",
            "config": config_block(args, cfg, world, res["n_layers"], packed + kvb + qo),
            "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"],
            "gpu_launches": args.steps * res["launches_per_step"], "clocks": res["clocks"],
            "per_kernel_us": res["per_kernel_us"], "step_roofline": res["step_roofline"],
            "full_kv": res["full_kv"],
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
