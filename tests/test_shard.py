"""Sequence-sharded decode step (X1, BASELINE config C5).

CPU (gloo, world_size 2 and 3): the exchange protocol of
``paper_2508_08256_b200.shard.sharded_step`` -- candidate all-gather, global
merge with the reference tie rule, ragged partials, LSE merge -- driven by an
oracle-backed shard (test infrastructure), checked against the unsharded
reference path (fier_attend, retrieval.hpp:136-146).

GPU: the same protocol over the CUDA kernels with P shards in one process
(``virtual_sharded_step``), against the oracle and against the unsharded GPU
path, up to the 1M-token C5 context.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch

from conftest import ROOT  # noqa: F401


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_whole_groups():
    from paper_2508_08256_b200.shard import shard_bounds
    for L, P, g in [(1 << 20, 8, 32), (4096, 3, 32), (1000, 4, 7), (33, 8, 32), (5, 2, 1)]:
        b = shard_bounds(L, P, g)
        assert b[0][0] == 0 and b[-1][1] == L
        for (s0, e0), (s1, _) in zip(b, b[1:]):
            assert e0 == s1
        for s, e in b[:-1]:
            assert (s % g == 0 or s == L) and (e % g == 0 or e == L) and e >= s
        sizes = [e - s for s, e in b]
        assert max(sizes) - min(sizes) < 2 * g or L < P * g


def test_shard_index_is_slice_of_global_index(port):
    """quantize on a g-aligned shard == the matching slice of the global index (quant1bit.hpp:5-9)."""
    rng = np.random.default_rng(3)
    L, d, g = 300, 24, 7
    K = rng.standard_normal((L, d))
    cw, s, z = port.quantize(K, g)
    W = (d + 63) // 64
    from paper_2508_08256_b200.shard import shard_bounds
    for a, b in shard_bounds(L, 3, g):
        cw_r, s_r, z_r = port.quantize(K[a:b], g)
        assert np.array_equal(cw_r, cw[a * W:b * W])
        assert np.array_equal(s_r, s[(a // g) * d:((b + g - 1) // g) * d])
        assert np.array_equal(z_r, z[(a // g) * d:((b + g - 1) // g) * d])


class OracleShard:
    """A CPU shard computing with the oracle (test infrastructure), same
    interface as ShardedDecodeLayer.  lse in the log2 domain, like K4."""

    def __init__(self, port, K, V, g, start, end):
        self.port, self.g, self.start, self.end = port, g, start, end
        self.K, self.V = K[:, start:end], V[:, start:end]   # [Hkv, l_r, d] fp64
        self.Hkv, _, self.d = K.shape

    def select_local(self, q, k_new, v_new, pos, n):
        Q = q.numpy()  # [Hq, d]
        Hq = Q.shape[0]
        lt = min(max(pos + 1 - self.start, 0), self.end - self.start)
        cs = np.full((Hq, n), -np.inf, np.float32)
        ci = np.full((Hq, n), -1, np.int32)
        self.lt = lt
        if lt > 0:
            for h in range(Hq):
                kv = h // (Hq // self.Hkv)
                buf = self.port.quantize_fier(self.K[kv, :lt], self.g)
                sc = self.port.approx_scores_fier(Q[h], buf).astype(np.float32)
                k = min(n, lt)
                sel = self.port.topk(sc.astype(np.float64), k)
                cs[h, :k] = sc[sel]
                ci[h, :k] = sel + self.start
        return torch.from_numpy(cs), torch.from_numpy(ci)

    def attend_local(self, q, CS, CI, n):
        Q = q.numpy()
        P, Hq, nc = CS.shape
        out = np.zeros((Hq, self.d), np.float32)
        lse = np.full(Hq, -np.inf, np.float32)
        self.sel_global = np.zeros((Hq, n), np.int64)
        for h in range(Hq):
            flat_s = CS[:, h].reshape(-1).numpy().astype(np.float64)
            flat_i = CI[:, h].reshape(-1).numpy()
            flat_s[flat_i < 0] = -np.inf
            pos = self.port.topk(flat_s, n)  # ties -> lower position == lower global index
            gsel = flat_i[pos]
            self.sel_global[h] = gsel
            mine = gsel[(gsel >= self.start) & (gsel < self.end)] - self.start
            if mine.size:
                kv = h // (Hq // self.Hkv)
                Kh, Vh = self.K[kv, :self.lt], self.V[kv, :self.lt]
                out[h] = self.port.gather_attention(Q[h], Kh, Vh, mine)
                logits = (Kh[mine] @ Q[h]) / math.sqrt(self.d) * math.log2(math.e)
                m = logits.max()
                lse[h] = m + math.log2(np.exp2(logits - m).sum())
        return torch.from_numpy(out), torch.from_numpy(lse)

    def combine(self, O, LSE):
        O, LSE = O.numpy().astype(np.float64), LSE.numpy().astype(np.float64)
        M = LSE.max(axis=0)
        w = np.where(np.isinf(LSE), 0.0, np.exp2(LSE - M))
        return torch.from_numpy((w[..., None] * O).sum(0) / w.sum(0)[..., None])


def _gloo_worker(rank, world, port_no, L, Hq, Hkv, d, g, n, pos, q_seed, result_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    from paper_2508_08256_b200.shard import DistExchange, shard_bounds, sharded_step
    rng = np.random.default_rng(q_seed)
    K = rng.standard_normal((Hkv, L, d))
    V = rng.standard_normal((Hkv, L, d))
    q = torch.from_numpy(rng.standard_normal((Hq, d)))
    a, b = shard_bounds(L, world, g)[rank]
    shard = OracleShard(Port(), K, V, g, a, b)
    out = sharded_step(shard, DistExchange(), q, None, None, pos, n)
    np.savez(result_path + f".{rank}.npz", out=out.numpy(), sel=shard.sel_global)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,L,pos,n,Hq,Hkv", [(2, 640, 639, 96, 4, 2), (3, 500, 430, 200, 2, 1),
                                                  (3, 500, 200, 100, 2, 2)])
def test_gloo_sharded_step_matches_unsharded(tmp_path, port, world, L, pos, n, Hq, Hkv):
    import torch.multiprocessing as mp
    d, g, seed = 16, 32, 11
    res = str(tmp_path / "res")
    mp.spawn(_gloo_worker, args=(world, _free_port(), L, Hq, Hkv, d, g, n, pos, seed, res), nprocs=world,
             join=True)
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((Hkv, L, d))
    V = rng.standard_normal((Hkv, L, d))
    Q = rng.standard_normal((Hq, d))
    outs = [np.load(res + f".{r}.npz") for r in range(world)]
    for r in range(1, world):  # identical on every rank
        assert np.array_equal(outs[r]["sel"], outs[0]["sel"])
        assert np.allclose(outs[r]["out"], outs[0]["out"], rtol=0, atol=1e-6)
    for h in range(Hq):
        kv = h // (Hq // Hkv)
        buf = port.quantize_fier(K[kv, :pos + 1], g)
        sc = port.approx_scores_fier(Q[h], buf).astype(np.float32).astype(np.float64)
        want_sel = port.topk(sc, n)
        assert np.array_equal(outs[0]["sel"][h], want_sel)
        want = port.gather_attention(Q[h], K[kv, :pos + 1], V[kv, :pos + 1], want_sel)
        assert port.relative_l2_error(outs[0]["out"][h], want) < 1e-5


# ---------------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("P,L,Hq,Hkv,n,dt", [(2, 2048, 4, 4, 256, torch.bfloat16),
                                             (4, 4000, 8, 2, 300, torch.float16),
                                             (3, 1000, 4, 1, 900, torch.float32)])
def test_virtual_sharded_step_vs_oracle(cuda, port, P, L, Hq, Hkv, n, dt):
    import paper_2508_08256_b200 as F
    from paper_2508_08256_b200.shard import ShardedDecodeLayer, virtual_sharded_step
    d, g = 128, 32
    gen = torch.Generator(device=cuda).manual_seed(5)
    K = torch.randn((1, Hkv, L, d), generator=gen, device=cuda).to(dt)
    V = torch.randn((1, Hkv, L, d), generator=gen, device=cuda).to(dt)
    q = torch.randn((1, Hq, d), generator=gen, device=cuda).to(dt)
    kn = torch.randn((1, Hkv, d), generator=gen, device=cuda).to(dt)
    vn = torch.randn((1, Hkv, d), generator=gen, device=cuda).to(dt)
    pos = L - 1
    shards = []
    for r in range(P):
        s = ShardedDecodeLayer(1, Hq, Hkv, L, d, g, rank=r, shards=P, dtype=dt, device=cuda)
        s.K[:, :, : s.end - s.start].copy_(K[:, :, s.start:s.end])
        s.V[:, :, : s.end - s.start].copy_(V[:, :, s.start:s.end])
        s.prefill(pos)
        shards.append(s)
    out = virtual_sharded_step(shards, q, kn, vn, pos, n)
    torch.cuda.synchronize()
    K[:, :, pos] = kn
    V[:, :, pos] = vn
    # unsharded GPU path on the same inputs: identical selection, close output
    layer = F.DecodeLayer(1, Hq, Hkv, L, d, g, dtype=dt, device=cuda, K=K.clone(), V=V.clone())
    layer.prefill(pos)
    o1, s1 = layer.step(q, kn, vn, pos, n)
    for s in shards:
        assert torch.equal(s.sel_global, s1), "sharded selection differs from unsharded"
    assert torch.allclose(out, o1, rtol=1e-4, atol=1e-5)
    Kd, Vd = K[0].double().cpu().numpy(), V[0].double().cpu().numpy()
    for h in range(Hq):
        kv = h // (Hq // Hkv)
        buf = port.quantize_fier(Kd[kv], g)
        sc = port.approx_scores_fier(q[0, h].double().cpu().numpy(), buf)
        want = port.topk(sc, n)
        got = shards[0].sel_global[0, h].cpu().numpy()
        assert port.recall(got, want) >= 0.999
        o = port.gather_attention(q[0, h].double().cpu().numpy(), Kd[kv], Vd[kv], got.astype(np.int64))
        assert port.relative_l2_error(out[0, h].cpu().numpy(), o) < 1e-2


@pytest.mark.gpu
def test_virtual_sharded_1m_context(cuda, port):
    """C5: a 1M-token GQA layer sharded 8 ways on one GPU == the unsharded GPU step."""
    import paper_2508_08256_b200 as F
    from paper_2508_08256_b200.shard import ShardedDecodeLayer, virtual_sharded_step
    P, L, Hq, Hkv, d, g, n = 8, 1 << 20, 32, 8, 128, 32, 4096
    dt = torch.bfloat16
    gen = torch.Generator(device=cuda).manual_seed(9)
    layer = F.DecodeLayer(1, Hq, Hkv, L, d, g, dtype=dt, device=cuda)
    layer.K.copy_(torch.randn(layer.K.shape, generator=gen, device=cuda).to(dt))
    layer.V.copy_(torch.randn(layer.V.shape, generator=gen, device=cuda).to(dt))
    q = torch.randn((1, Hq, d), generator=gen, device=cuda).to(dt)
    kn = torch.randn((1, Hkv, d), generator=gen, device=cuda).to(dt)
    vn = torch.randn((1, Hkv, d), generator=gen, device=cuda).to(dt)
    pos = L - 1
    shards = []
    for r in range(P):
        s = ShardedDecodeLayer(1, Hq, Hkv, L, d, g, rank=r, shards=P, dtype=dt, device=cuda)
        s.K.copy_(layer.K[:, :, s.start:s.end])
        s.V.copy_(layer.V[:, :, s.start:s.end])
        s.prefill(pos)
        shards.append(s)
    out = virtual_sharded_step(shards, q, kn, vn, pos, n)
    layer.prefill(pos)
    o1, s1 = layer.step(q, kn, vn, pos, n)
    torch.cuda.synchronize()
    assert torch.equal(shards[-1].sel_global, s1)
    assert torch.allclose(out, o1, rtol=1e-4, atol=1e-5)
    # the oracle on two heads (fp64 over 1M tokens)
    for h in (0, 31):
        kv = h // 4
        Kd = layer.K[0, kv].double().cpu().numpy()
        Vd = layer.V[0, kv].double().cpu().numpy()
        o = port.gather_attention(q[0, h].double().cpu().numpy(), Kd, Vd,
                                  s1[0, h].cpu().numpy().astype(np.int64))
        assert port.relative_l2_error(out[0, h].cpu().numpy(), o) < 1e-2


def _cuda_shard_worker(rank, world, port_no, L, Hq, Hkv, n, dt_name, seed, result_path):
    """One process per shard, all on cuda:0: the CUDA ShardedDecodeLayer of `rank`, the
    exchange over gloo through host copies (HostStagedExchange)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_08256_b200.shard import HostStagedExchange, ShardedDecodeLayer, sharded_step
    dev = torch.device("cuda", 0)
    dt = getattr(torch, dt_name)
    d, g = 128, 32
    gen = torch.Generator(device="cpu").manual_seed(seed)  # identical full inputs on every rank
    K = torch.randn((1, Hkv, L, d), generator=gen).to(dt)
    V = torch.randn((1, Hkv, L, d), generator=gen).to(dt)
    q = torch.randn((1, Hq, d), generator=gen).to(dt).to(dev)
    kn = torch.randn((1, Hkv, d), generator=gen).to(dt).to(dev)
    vn = torch.randn((1, Hkv, d), generator=gen).to(dt).to(dev)
    pos = L - 1
    s = ShardedDecodeLayer(1, Hq, Hkv, L, d, g, rank=rank, shards=world, dtype=dt, device=dev)
    s.K[:, :, : s.end - s.start].copy_(K[:, :, s.start:s.end])
    s.V[:, :, : s.end - s.start].copy_(V[:, :, s.start:s.end])
    s.prefill(pos)
    ex = HostStagedExchange()
    outs = []
    for _ in range(2):  # two steps: the second re-appends the same token (idempotent)
        outs.append(sharded_step(s, ex, q, kn, vn, pos, n).cpu())
    torch.cuda.synchronize()
    np.savez(result_path + f".{rank}.npz", out=outs[-1].numpy(), out0=outs[0].numpy(),
             sel=s.sel_global.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,L,Hq,Hkv,n,dt", [(2, 4096, 8, 2, 400, "bfloat16"), (3, 3000, 4, 4, 350, "float16")])
def test_two_process_cuda_sharded_step(cuda, tmp_path, world, L, Hq, Hkv, n, dt):
    """SURVEY §8(e) on real processes: `world` ranks, each a CUDA ShardedDecodeLayer on cuda:0,
    exchanging candidates and partials over gloo -- the same selection as the unsharded GPU
    step and the same output within fp32 merge rounding, identical on every rank."""
    import torch.multiprocessing as mp
    import paper_2508_08256_b200 as F
    seed = 21
    res = str(tmp_path / "res")
    mp.spawn(_cuda_shard_worker, args=(world, _free_port(), L, Hq, Hkv, n, dt, seed, res), nprocs=world,
             join=True)
    outs = [np.load(res + f".{r}.npz") for r in range(world)]
    for r in range(world):
        assert np.array_equal(outs[r]["sel"], outs[0]["sel"])
        assert np.array_equal(outs[r]["out"], outs[0]["out"])
        assert np.array_equal(outs[r]["out0"], outs[r]["out"])
    # the unsharded step on the same inputs (same generator order as the workers)
    d, g = 128, 32
    tdt = getattr(torch, dt)
    gen = torch.Generator(device="cpu").manual_seed(seed)
    K = torch.randn((1, Hkv, L, d), generator=gen).to(tdt)
    V = torch.randn((1, Hkv, L, d), generator=gen).to(tdt)
    q = torch.randn((1, Hq, d), generator=gen).to(tdt).to(cuda)
    kn = torch.randn((1, Hkv, d), generator=gen).to(tdt).to(cuda)
    vn = torch.randn((1, Hkv, d), generator=gen).to(tdt).to(cuda)
    pos = L - 1
    layer = F.DecodeLayer(1, Hq, Hkv, L, d, g, dtype=tdt, device=cuda, K=K.to(cuda), V=V.to(cuda))
    layer.prefill(pos)
    o1, s1 = layer.step(q, kn, vn, pos, n)
    torch.cuda.synchronize()
    assert np.array_equal(outs[0]["sel"], s1.cpu().numpy()), "sharded selection differs from unsharded"
    assert np.allclose(outs[0]["out"], o1.cpu().numpy(), rtol=1e-4, atol=1e-5)


def _devx_worker(rank, world, port_no, result_path):
    """One rank: the NCCL device-API exchange (libfier_nccl.so) inside the sharded step."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2508_08256_b200 as F
    from paper_2508_08256_b200.shard import NcclDeviceExchange, ShardedDecodeLayer, sharded_step
    dev = torch.device("cuda", 0)
    L, Hq, Hkv, d, g, n = 3000, 8, 2, 128, 32, 300
    gen = torch.Generator(device="cpu").manual_seed(5)
    K = torch.randn((1, Hkv, L, d), generator=gen).to(torch.bfloat16)
    V = torch.randn((1, Hkv, L, d), generator=gen).to(torch.bfloat16)
    q = torch.randn((1, Hq, d), generator=gen).to(torch.bfloat16).to(dev)
    kn = torch.randn((1, Hkv, d), generator=gen).to(torch.bfloat16).to(dev)
    vn = torch.randn((1, Hkv, d), generator=gen).to(torch.bfloat16).to(dev)
    pos = L - 1
    ex = NcclDeviceExchange(slot_bytes=2 * Hq * n * 8, group=None)
    # the raw all-gather: slot r holds rank r's bytes
    x = (torch.arange(1000, device=dev, dtype=torch.int32) + 7 * rank)
    gx = ex.all_gather(x)
    assert gx.shape == (world, 1000) and torch.equal(gx[rank], x)
    s = ShardedDecodeLayer(1, Hq, Hkv, L, d, g, rank=rank, shards=world, dtype=torch.bfloat16, device=dev)
    s.K[:, :, : s.end - s.start].copy_(K[:, :, s.start:s.end])
    s.V[:, :, : s.end - s.start].copy_(V[:, :, s.start:s.end])
    s.prefill(pos)
    out = sharded_step(s, ex, q, kn, vn, pos, n)
    torch.cuda.synchronize()
    layer = F.DecodeLayer(1, Hq, Hkv, L, d, g, dtype=torch.bfloat16, device=dev, K=K.to(dev), V=V.to(dev))
    layer.prefill(pos)
    o1, s1 = layer.step(q, kn, vn, pos, n)
    torch.cuda.synchronize()
    ok = torch.equal(s.sel_global, s1) and torch.allclose(out, o1, rtol=1e-4, atol=1e-5)
    np.savez(result_path + f".{rank}.npz", ok=ok)
    ex.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_device_exchange_single_rank(cuda, tmp_path):
    """The NCCL device-API exchange (symmetric window, LSA stores, LSA barrier) on the one GPU
    this build has (world 1: the path a multi-GPU run takes, with the rank's own slot): the
    sharded step through it equals the unsharded GPU step."""
    import torch.multiprocessing as mp
    from paper_2508_08256_b200 import build as b
    if not b.build_nccl():
        pytest.skip("no NCCL with the device API")
    res = str(tmp_path / "res")
    mp.spawn(_devx_worker, args=(1, _free_port(), res), nprocs=1, join=True)
    assert bool(np.load(res + ".0.npz")["ok"])
