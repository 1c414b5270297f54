"""Sequence-sharded Fier decode step (X1; BASELINE config C5).

A long context is split into P contiguous token ranges, one per GPU, whose
boundaries are whole quantization groups (``fier_shard_bounds``), so each
shard's packed index is bit-identical to the matching slice of the global
``quantize`` (quant1bit.hpp:5-9, 84).  One decode step:

  1. every shard appends (only the shard that owns ``pos``), scores its tokens
     and keeps its local Top-min(n, l_r) as (score, global index) candidates
     (K1b, K2, K3 and ``fier_shard_candidates``);
  2. exchange #1 -- all-gather of the candidate lists (rows x n x 8 bytes);
  3. every shard runs the same deterministic merge (``fier_shard_merge``: K3 on
     the side-by-side lists, which are in global index order, so the reference
     tie rule of topk_oracle, core.hpp:134-148, holds globally) and keeps its
     own run of the global selection;
  4. ragged K4 over that run -> per-row (o_r, lse_r);
  5. exchange #2 -- all-gather of the partials (rows x (d+1) floats);
  6. log-sum-exp merge (``fier_lse_merge``) -> the global output, identical on
     every rank.

Nothing else crosses GPUs.  The protocol (:func:`sharded_step`) is written
against two small interfaces -- a *shard* (select_local / attend_local /
combine) and an *exchange* (all_gather) -- so the same code runs over NCCL
(one process per GPU, :class:`DistExchange`), over gloo in the CPU tests, and
over P shards held by one process (:func:`virtual_sharded_step`, single-GPU
parity at 1M tokens).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import List, Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import check
from .api import DecodeLayer, _p, _stream, make_shape


def shard_bounds(tokens: int, shards: int, group: int) -> List[Tuple[int, int]]:
    """[start, end) of every shard: whole groups, spread evenly (fier_shard_bounds)."""
    lib = _lib.load()
    out = []
    for r in range(shards):
        a, b = C.c_int64(), C.c_int64()
        check(lib.fier_shard_bounds(tokens, shards, group, r, C.byref(a), C.byref(b)))
        out.append((a.value, b.value))
    return out


class DistExchange:
    """all_gather over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        t = t.contiguous()
        if t.is_cuda:  # NCCL: one fused all-gather into a [P, ...] buffer
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return torch.stack(parts)


class HostStagedExchange(DistExchange):
    """all_gather of device tensors over a CPU backend (gloo): device -> host copy,
    gather, host -> device.  Lets several processes that share one GPU (or GPUs without
    a peer path) run the sharded protocol with the CUDA kernels on every shard."""

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        if not t.is_cuda:
            return super().all_gather(t)
        h = t.contiguous().cpu()
        parts = [torch.empty_like(h) for _ in range(self.world)]
        self.dist.all_gather(parts, h, group=self.group)
        return torch.stack(parts).to(t.device)


_NCCL_LIB = None


def _nccl_lib():
    """libfier_nccl.so (include/fier_nccl.h): the NCCL device-API exchange."""
    global _NCCL_LIB
    if _NCCL_LIB is None:
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfier_nccl.so")
        if not os.path.exists(path):
            raise RuntimeError("libfier_nccl.so is not built (paper_2508_08256_b200.build.build_nccl)")
        lib = C.CDLL(path)
        lib.fier_devx_unique_id.argtypes = [C.c_void_p]
        lib.fier_devx_create.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_size_t, C.c_int32,
                                         C.POINTER(C.c_void_p)]
        lib.fier_devx_allgather.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.POINTER(C.c_void_p)]
        lib.fier_devx_shard_candidates.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                                   C.c_int32, C.c_int32, C.c_int64, C.c_void_p,
                                                   C.POINTER(C.c_void_p)]
        lib.fier_devx_destroy.argtypes = [C.c_void_p]
        lib.fier_devx_last_error.restype = C.c_char_p
        _NCCL_LIB = lib
    return _NCCL_LIB


class _CudaBytes:
    """A uint8 view of a device allocation owned elsewhere (__cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


class NcclDeviceExchange:
    """all_gather done on the device through the NCCL 2.28 device API: a kernel
    stores this rank's slot into every peer's symmetric window over NVLink (LSA pointers) and
    closes with an LSA barrier -- no host-side collective in the step, graph-capturable like
    any launch.  `slot_bytes` bounds one rank's payload (the larger of the two exchanges)."""

    def __init__(self, slot_bytes: int, group=None, max_ctas: int = 64):
        import torch.distributed as dist
        lib = _nccl_lib()
        self.lib, self.group = lib, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            check_devx(lib, lib.fier_devx_unique_id(uid.data_ptr()))
        if self.world > 1:
            on_gpu = dist.get_backend(group) == "nccl"
            t = uid.cuda() if on_gpu else uid
            dist.broadcast(t, src=0, group=group)
            uid = t.cpu()
        self.slot = (int(slot_bytes) + 4095) // 4096 * 4096
        h = C.c_void_p()
        check_devx(lib, lib.fier_devx_create(uid.data_ptr(), self.world, self.rank, self.slot, max_ctas,
                                             C.byref(h)))
        self.handle = h
        self._win = None

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        t = t.contiguous()
        nbytes = t.numel() * t.element_size()
        pad = (-nbytes) % 16
        src = t if pad == 0 else torch.cat([t.view(torch.uint8).reshape(-1),
                                            torch.zeros(pad, dtype=torch.uint8, device=t.device)])
        out = C.c_void_p()
        check_devx(self.lib, self.lib.fier_devx_allgather(self.handle, src.data_ptr(), nbytes + pad, _stream(),
                                                          C.byref(out)))
        if self._win is None:
            self._win = torch.as_tensor(_CudaBytes(out.value, self.world * self.slot), device=t.device)
        g = self._win.view(self.world, self.slot)[:, :nbytes]
        return g.contiguous().view(t.dtype).reshape((self.world,) + tuple(t.shape))

    def gather_candidates(self, scores, ld: int, sel, rows: int, k: int, n: int, start: int):
        """fier_shard_candidates fused with the candidate all-gather (fier_devx_shard_candidates):
        returns (CS [P, rows, n] fp32, CI [P, rows, n] int32)."""
        out = C.c_void_p()
        check_devx(self.lib, self.lib.fier_devx_shard_candidates(
            self.handle, _p(scores) if scores is not None else None, ld, _p(sel) if sel is not None else None,
            rows, k, n, start, _stream(), C.byref(out)))
        dev = scores.device if scores is not None else torch.device("cuda", torch.cuda.current_device())
        if self._win is None:
            self._win = torch.as_tensor(_CudaBytes(out.value, self.world * self.slot), device=dev)
        w = self._win.view(self.world, self.slot)[:, : 2 * rows * n * 4].view(torch.int32).view(self.world, 2, rows, n)
        return w[:, 0].contiguous().view(torch.float32), w[:, 1].contiguous()

    def close(self):
        if self.handle:
            self.lib.fier_devx_destroy(self.handle)
            self.handle = None


def check_devx(lib, rc: int) -> None:
    if rc:
        raise RuntimeError(lib.fier_devx_last_error().decode())


def _pack_candidates(cs: torch.Tensor, ci: torch.Tensor) -> torch.Tensor:
    return torch.stack([cs.view(torch.int32), ci])


def _unpack_candidates(g: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    # g: [P, 2, rows, n]
    return g[:, 0].contiguous().view(torch.float32), g[:, 1].contiguous()


def _pack_partial(out: torch.Tensor, lse: torch.Tensor) -> torch.Tensor:
    return torch.cat([out, lse.unsqueeze(-1)], dim=-1)


def _unpack_partial(g: torch.Tensor, d: int) -> Tuple[torch.Tensor, torch.Tensor]:
    # g: [P, rows, d + 1]
    return g[..., :d].contiguous(), g[..., d].contiguous()


def sharded_step(shard, exchange, q, k_new, v_new, pos: int, n: int) -> torch.Tensor:
    """One decode step of a sequence-sharded layer; returns out [B, Hq, d] (fp32),
    identical on every rank.  The two all-gathers are the only communication."""
    if hasattr(exchange, "gather_candidates"):  # candidates stored straight into the peers' windows
        CS, CI = shard.select_local(q, k_new, v_new, pos, n, exchange=exchange)
    else:
        cs, ci = shard.select_local(q, k_new, v_new, pos, n)
        CS, CI = _unpack_candidates(exchange.all_gather(_pack_candidates(cs, ci)))
    o, lse = shard.attend_local(q, CS, CI, n)
    O, LSE = _unpack_partial(exchange.all_gather(_pack_partial(o, lse)), o.shape[-1])
    return shard.combine(O, LSE)


def virtual_sharded_step(shards: Sequence, q, k_new, v_new, pos: int, n: int) -> torch.Tensor:
    """The same protocol with all P shards in one process (the all-gathers become stacks)."""
    cands = [_pack_candidates(*s.select_local(q, k_new, v_new, pos, n)) for s in shards]
    CS, CI = _unpack_candidates(torch.stack(cands))
    parts = [_pack_partial(*s.attend_local(q, CS, CI, n)) for s in shards]
    O, LSE = _unpack_partial(torch.stack(parts), shards[0].d)
    return shards[0].combine(O, LSE)


class ShardedDecodeLayer:
    """Shard ``rank`` of ``shards`` of one attention layer over a context of
    ``context`` tokens, on this process's GPU.  The local KV cache holds global
    tokens [start, end) as local rows [0, end - start)."""

    def __init__(self, batch, q_heads, kv_heads, context, dim, group=32, rank=0, shards=1,
                 dtype=torch.bfloat16, device="cuda", K=None, V=None):
        self.B, self.Hq, self.Hkv, self.d, self.g = batch, q_heads, kv_heads, dim, group
        self.rank, self.P, self.context = rank, shards, context
        self.start, self.end = shard_bounds(context, shards, group)[rank]
        self.cap = max(self.end - self.start, group)
        self.device = torch.device(device)
        self.layer = DecodeLayer(batch, q_heads, kv_heads, self.cap, dim, group, dtype=dtype, device=device,
                                 K=K, V=V)
        self.rows = batch * q_heads
        self.local_tokens = 0
        self.sel_global: Optional[torch.Tensor] = None
        self._bufs = {}

    # -- helpers ---------------------------------------------------------------
    def _buf(self, name, shape, dtype):
        t = self._bufs.get(name)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t

    def _local(self, pos: int) -> int:
        return min(max(pos + 1 - self.start, 0), self.end - self.start)

    @property
    def K(self):
        return self.layer.K

    @property
    def V(self):
        return self.layer.V

    def prefill(self, tokens: int) -> None:
        """Pack this shard's part of the prefix [0, tokens)."""
        lt = min(max(tokens - self.start, 0), self.end - self.start)
        if lt > 0:
            self.layer.prefill(lt)
        self.local_tokens = lt

    # -- protocol steps -----------------------------------------------------------
    def select_local(self, q, k_new, v_new, pos: int, n: int, exchange=None):
        """Append (the shard holding pos), score, local Top-min(n, l); returns the (score, global
        index) candidate lists -- or, with an exchange that fuses the candidate construction
        into its all-gather (NcclDeviceExchange), the gathered [P, rows, n] lists."""
        lib = _lib.load()
        sh = C.byref(self.layer.shape)
        if self.start <= pos < self.end:
            check(lib.fier_append(sh, _p(self.layer.K), _p(self.layer.V), _p(k_new), _p(v_new),
                                  pos - self.start, _p(self.layer.pk.bits), _p(self.layer.pk.params), None,
                                  _stream()))
            self.layer.pk.tokens = max(self.layer.pk.tokens, pos - self.start + 1)
        lt = self._local(pos)
        self.local_tokens = lt
        cs = self._buf("cs", (self.rows, n), torch.float32)
        ci = self._buf("ci", (self.rows, n), torch.int32)
        k = min(n, lt)
        fused = exchange is not None and hasattr(exchange, "gather_candidates")
        if k == 0:
            if fused:
                return exchange.gather_candidates(None, 1, None, self.rows, 0, n, self.start)
            check(lib.fier_shard_candidates(None, self.rows, 1, None, 0, n, self.start, _p(cs), _p(ci),
                                            _stream()))
            return cs, ci
        ld = lib.fier_step_scores_ld(lt)
        scores = self._buf("scores", (self.rows, ld), torch.float32)
        sel = self._buf(f"sel{k}", (self.rows, k), torch.int32)
        check(lib.fier_score(sh, _p(q), _p(self.layer.pk.bits), _p(self.layer.pk.params), lt, _p(scores), ld,
                             _stream()))
        twb = lib.fier_topk_workspace(self.rows, lt, k)
        tws = self._buf("tws", (max(twb, 1),), torch.uint8)
        check(lib.fier_topk(_p(scores), self.rows, lt, ld, k, _p(sel), _p(tws), twb, _stream()))
        if fused:
            return exchange.gather_candidates(scores, ld, sel, self.rows, k, n, self.start)
        check(lib.fier_shard_candidates(_p(scores), self.rows, ld, _p(sel), k, n, self.start, _p(cs), _p(ci),
                                        _stream()))
        return cs, ci

    def attend_local(self, q, CS, CI, n: int, scale: Optional[float] = None):
        lib = _lib.load()
        P = CS.shape[0]
        ws = self._buf("mws", (lib.fier_shard_merge_workspace(P, self.rows, n, n),), torch.uint8)
        self.sel_global = self._buf("selg", (self.B, self.Hq, n), torch.int32)
        sel_local = self._buf("sell", (self.B, self.Hq, n), torch.int32)
        counts = self._buf("counts", (self.B, self.Hq), torch.int32)
        check(lib.fier_shard_merge(_p(CS), _p(CI), P, self.rows, n, n, self.rank, self.start,
                                   _p(self.sel_global), _p(sel_local), _p(counts), _p(ws), ws.numel(),
                                   _stream()))
        out = self._buf("o", (self.B, self.Hq, self.d), torch.float32)
        lse = self._buf("lse", (self.B, self.Hq), torch.float32)
        if self.local_tokens == 0:
            out.zero_()
            lse.fill_(-math.inf)
            return out, lse
        scale = 1.0 / math.sqrt(self.d) if scale is None else scale
        aws = self._buf("aws", (max(4, lib.fier_sparse_attention_workspace(C.byref(self.layer.shape), n)),),
                        torch.uint8)
        check(lib.fier_sparse_attention_ragged(C.byref(self.layer.shape), _p(q), _p(self.layer.K),
                                               _p(self.layer.V), _p(sel_local), _p(counts), n,
                                               self.local_tokens, scale, _p(out), _p(lse), _p(aws), aws.numel(),
                                               _stream()))
        return out, lse

    def combine(self, O, LSE) -> torch.Tensor:
        lib = _lib.load()
        P = O.shape[0]
        out = torch.empty((self.B, self.Hq, self.d), dtype=torch.float32, device=self.device)
        check(lib.fier_lse_merge(_p(O), _p(LSE), P, self.rows, self.d, _p(out), None, _stream()))
        return out
