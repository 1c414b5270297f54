"""Torch-facing mirror of the reference's Fier API, running on the sm_100a kernels.

Same names, argument meaning and error behaviour as the reference's C++ entry
points (proj/include/fier/):

=====================  =========================================  ==============================
this module            reference                                   kernel
=====================  =========================================  ==============================
quantize               quantize            quant1bit.hpp:65-103    K1 pack  (fier_pack_keys)
append_token           (decode-time growth, quant1bit.hpp:84)      K1 append (fier_append)
approx_scores          approx_scores       quant1bit.hpp:121-140   K2 score (fier_score)
topk_oracle            topk_oracle         core.hpp:134-148        K3 top-k (fier_topk)
gather_attention       gather_attention    core.hpp:152-179        K4 sparse attention
full_attention         full policy         retrieval.hpp:159-166   K0 full-KV attention
fier_select            fier_select         retrieval.hpp:130-133   K2 -> K3
fier_attend            fier_attend         retrieval.hpp:136-146   K2 -> K3 -> K4
DecodeLayer.step       fier_attend per decode step, batched       fier_decode_step
=====================  =========================================  ==============================

Tensors live on the GPU.  Single-head calls take the reference's shapes
(K: [l, d], q: [d]); batched calls take K: [B, Hkv, l, d], q: [B, Hq, d].
Precondition failures raise ValueError with the reference's message
(std::invalid_argument from require(), core.hpp:19-21); malformed FIER bytes
raise FierDataError (fier::DataError, io.hpp:29-31).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import FierShape, check

_DT = {torch.float32: _lib.FIER_F32, torch.float16: _lib.FIER_F16, torch.bfloat16: _lib.FIER_BF16}
# fp64 keys (the reference's own KeyCache type) are accepted by quantize / append_token only
_DT_KEYS = {**_DT, torch.float64: _lib.FIER_F64}


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: Optional[torch.Tensor]) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else 0)


def _require(ok: bool, msg: str) -> None:
    if not ok:
        raise ValueError(msg)


def _dtype_code(t: torch.Tensor, keys: bool = False) -> int:
    table = _DT_KEYS if keys else _DT
    _require(t.dtype in table, f"unsupported dtype {t.dtype}: expected float32, float16 or bfloat16"
             + (" (or float64 keys)" if keys else ""))
    return table[t.dtype]


def _cuda(t: torch.Tensor, what: str) -> torch.Tensor:
    _require(isinstance(t, torch.Tensor) and t.is_cuda, f"{what}: expected a CUDA tensor")
    return t.contiguous()


def _as4(K: torch.Tensor) -> torch.Tensor:
    if K.dim() == 2:
        return K.unsqueeze(0).unsqueeze(0)
    _require(K.dim() == 4, "expected a [l, d] or [B, H, l, d] cache")
    return K


def _as3(q: torch.Tensor) -> torch.Tensor:
    if q.dim() == 1:
        return q.view(1, 1, -1)
    _require(q.dim() == 3, "expected a [d] or [B, H, d] query")
    return q


def make_shape(batch, q_heads, kv_heads, capacity, dim, group, dtype) -> FierShape:
    return FierShape(batch, q_heads, kv_heads, capacity, dim, group, dtype)


@dataclass
class PackedKeys:
    """Device-resident Fier index (PackedKeys, quant1bit.hpp:32-63).

    bits   : int32 view of uint32 [B, Hkv, cap, ceil(d/32)] (bit i of word w = channel 32w+i)
    params : float16 [B, Hkv, ceil(cap/g), d, 2] = (s, z) rounded to binary16
    """
    bits: torch.Tensor
    params: torch.Tensor
    tokens: int
    dim: int
    group_size: int
    batch: int
    kv_heads: int
    capacity: int
    single: bool = False

    @property
    def groups_per_channel(self) -> int:
        return (self.tokens + self.group_size - 1) // self.group_size

    def payload_bytes(self) -> int:
        """Per (sequence, kv head): l*ceil(d/8) + d*ceil(l/g)*4 (quant1bit.hpp:60-62)."""
        return int(_lib.load().fier_payload_bytes(self.tokens, self.dim, self.group_size))

    def scales(self) -> torch.Tensor:
        """(s) as fp64, [B, Hkv, G, d] (or [G*d] single-head) -- half-rounded."""
        s = self.params[:, :, : self.groups_per_channel, :, 0].double()
        return s.reshape(-1) if self.single else s

    def zeros(self) -> torch.Tensor:
        z = self.params[:, :, : self.groups_per_channel, :, 1].double()
        return z.reshape(-1) if self.single else z

    def to_fier(self, b: int = 0, h: int = 0) -> bytes:
        """serialize_packed_keys (io.hpp:197-225) of sequence b, kv head h."""
        W = (self.dim + 31) // 32
        bits = self.bits[b, h, : self.tokens].contiguous().cpu().numpy().view(np.uint32)
        par = self.params[b, h, : self.groups_per_channel].contiguous().cpu().numpy().view(np.uint16)
        out = np.zeros(18 + self.payload_bytes(), np.uint8)
        check(_lib.load().fier_index_to_fier(bits.ctypes.data, par.ctypes.data, self.tokens, self.dim,
                                             self.group_size, out.ctypes.data, out.size))
        assert bits.size == self.tokens * W
        return out.tobytes()

    @staticmethod
    def from_fier(buf: bytes, device="cuda", capacity: Optional[int] = None) -> "PackedKeys":
        """parse_packed_keys (io.hpp:227-277) into a device index."""
        lib = _lib.load()
        b = np.frombuffer(buf, np.uint8)
        l, d, g = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib.fier_fier_to_index(b.ctypes.data, b.size, C.byref(l), C.byref(d), C.byref(g),
                                     None, 0, None, 0))
        l, d, g = l.value, d.value, g.value
        cap = capacity or l
        W, G = (d + 31) // 32, (cap + g - 1) // g
        bits = np.zeros((1, 1, cap, W), np.uint32)
        par = np.zeros((1, 1, G, d, 2), np.uint16)
        check(lib.fier_fier_to_index(b.ctypes.data, b.size, C.byref(C.c_int32()), C.byref(C.c_int32()),
                                     C.byref(C.c_int32()), bits.ctypes.data, bits.size, par.ctypes.data,
                                     par.size))
        return PackedKeys(torch.from_numpy(bits.view(np.int32)).to(device),
                          torch.from_numpy(par.view(np.float16)).to(device), l, d, g, 1, 1, cap,
                          single=True)


    def to_fier_device(self, b: int = 0, h: int = 0) -> torch.Tensor:
        """serialize_packed_keys (io.hpp:197-225) of sequence b, kv head h into a CUDA uint8
        tensor, written by kernels (fier_index_export): persist it with one D2H copy."""
        _require(self.bits.is_cuda, "to_fier_device: the index is not on a GPU")
        out = torch.empty(18 + self.payload_bytes(), dtype=torch.uint8, device=self.bits.device)
        check(_lib.load().fier_index_export(_p(self.bits[b, h]), _p(self.params[b, h]), self.tokens, self.dim,
                                            self.group_size, _p(out), out.numel(), _stream()))
        return out

    @staticmethod
    def from_fier_device(buf: torch.Tensor, capacity: Optional[int] = None) -> "PackedKeys":
        """parse_packed_keys (io.hpp:227-277) of a FIER stream held in a CUDA uint8 tensor,
        decoded on the device (fier_index_import)."""
        _require(isinstance(buf, torch.Tensor) and buf.is_cuda and buf.dtype == torch.uint8,
                 "from_fier_device: expected a CUDA uint8 tensor")
        lib = _lib.load()
        buf = buf.contiguous()
        l, d, g = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib.fier_index_import(_p(buf), buf.numel(), C.byref(l), C.byref(d), C.byref(g), None, 0, None, 0,
                                    _stream()))
        l, d, g = l.value, d.value, g.value
        cap = capacity or l
        _require(cap >= l, "from_fier_device: capacity below the stored token count")
        pk = alloc_index(1, 1, cap, d, g, buf.device)
        check(lib.fier_index_import(_p(buf), buf.numel(), None, None, None, _p(pk.bits), pk.bits.numel(),
                                    _p(pk.params), pk.params.numel() // 2, _stream()))
        pk.tokens, pk.single = l, True
        return pk


@dataclass(frozen=True)
class LoadRatio:
    """LoadRatio (quant1bit.hpp:162-171): exact bit counts of estimation vs a 16-bit key cache."""
    numerator_bits: int
    denominator_bits: int
    formula: bool  # False when a short final group forces exact byte accounting

    def ratio(self) -> Tuple[int, int]:
        """Rational(numerator_bits, denominator_bits) reduced (quant1bit.hpp:143-160)."""
        g = math.gcd(self.numerator_bits, self.denominator_bits)
        return self.numerator_bits // g, self.denominator_bits // g

    def value(self) -> float:
        n, d = self.ratio()
        return n / d


def load_ratio_fier(l: int, g: int) -> LoadRatio:
    """load_ratio_fier (quant1bit.hpp:176-184) through the C ABI (fier_load_ratio_fier)."""
    num, den, formula = C.c_int64(), C.c_int64(), C.c_int32()
    check(_lib.load().fier_load_ratio_fier(l, g, C.byref(num), C.byref(den), C.byref(formula)))
    return LoadRatio(num.value, den.value, bool(formula.value))


def alloc_index(batch, kv_heads, capacity, dim, group, device="cuda") -> PackedKeys:
    W, G = (dim + 31) // 32, (capacity + group - 1) // group
    bits = torch.zeros((batch, kv_heads, capacity, W), dtype=torch.int32, device=device)
    params = torch.zeros((batch, kv_heads, G, dim, 2), dtype=torch.float16, device=device)
    return PackedKeys(bits, params, 0, dim, group, batch, kv_heads, capacity)


def _shape_of(pk: PackedKeys, q_heads: int, dtype: int) -> FierShape:
    return make_shape(pk.batch, q_heads, pk.kv_heads, pk.capacity, pk.dim, pk.group_size, dtype)


def quantize(K: torch.Tensor, group_size: int = 32, tokens: Optional[int] = None,
             out: Optional[PackedKeys] = None) -> PackedKeys:
    """quantize (quant1bit.hpp:65-103) on the GPU.  K: [l, d] or [B, Hkv, cap, d]."""
    _require(group_size >= 1, "quantize: group size must be >= 1")
    single = K.dim() == 2
    K4 = _as4(_cuda(K, "quantize"))
    B, H, cap, d = K4.shape
    _require(cap >= 1 and d >= 1, "quantize: empty key cache")
    tokens = cap if tokens is None else tokens
    _require(1 <= tokens <= cap, "quantize: empty key cache")
    pk = out or alloc_index(B, H, cap, d, group_size, K4.device)
    flag = torch.zeros(1, dtype=torch.int32, device=K4.device)
    shape = make_shape(B, H, H, cap, d, group_size, _dtype_code(K4, keys=True))
    check(_lib.load().fier_pack_keys(C.byref(shape), _p(K4), tokens, _p(pk.bits), _p(pk.params),
                                     _p(flag), _stream()))
    if int(flag.item()) != 0:
        raise ValueError("quantize: non-finite key entry")
    pk.tokens, pk.single = tokens, single
    return pk


def append_token(K: torch.Tensor, V: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
                 pos: int, pk: PackedKeys, check_finite: bool = True) -> PackedKeys:
    """Write token `pos` of K/V and re-pack its open group in place (K1b)."""
    K4, V4 = _as4(K), _as4(V)
    B, H, cap, d = K4.shape
    flag = torch.zeros(1, dtype=torch.int32, device=K4.device) if check_finite else None
    shape = make_shape(B, H, H, cap, d, pk.group_size, _dtype_code(K4, keys=True))
    check(_lib.load().fier_append(C.byref(shape), _p(K4), _p(V4), _p(k_new.contiguous()),
                                  _p(v_new.contiguous()), pos, _p(pk.bits), _p(pk.params), _p(flag),
                                  _stream()))
    if check_finite and int(flag.item()) != 0:
        raise ValueError("quantize: non-finite key entry")
    pk.tokens = max(pk.tokens, pos + 1)
    return pk


def approx_scores(q: torch.Tensor, pk: PackedKeys) -> torch.Tensor:
    """approx_scores (quant1bit.hpp:121-140): fp32 [l] or [B, Hq, l]."""
    single = q.dim() == 1
    _require(q.shape[-1] == pk.dim, "approx_scores: query length does not match key dim")
    q3 = _as3(_cuda(q, "approx_scores"))
    B, Hq, d = q3.shape
    _require(B == pk.batch and Hq % pk.kv_heads == 0, "approx_scores: query heads do not match index")
    ld = pk.tokens
    scores = torch.empty((B, Hq, ld), dtype=torch.float32, device=q3.device)
    shape = _shape_of(pk, Hq, _dtype_code(q3))
    check(_lib.load().fier_score(C.byref(shape), _p(q3), _p(pk.bits), _p(pk.params), pk.tokens,
                                 _p(scores), ld, _stream()))
    return scores.view(-1) if single else scores


def topk_oracle(scores: torch.Tensor, k: int, wide: bool = True) -> torch.Tensor:
    """topk_oracle (core.hpp:134-148): int32 ascending indices [k] or [..., k].

    float32 scores take the decode path's select (fier_topk: with ``wide``, launches of
    millions of keys use the wide-grid radix select and its workspace, else the per-row
    cluster select); float64 scores (the reference's own ScoreVector type) the exact fp64
    select (fier_topk_f64)."""
    s = _cuda(scores, "topk_oracle")
    _require(s.dtype in (torch.float32, torch.float64), "topk_oracle: scores must be float32 or float64")
    l = s.shape[-1]
    _require(1 <= k <= l, "topk_oracle: k out of range")
    rows = s.numel() // l
    sel = torch.empty(s.shape[:-1] + (k,), dtype=torch.int32, device=s.device)
    if s.dtype == torch.float64:
        check(_lib.load().fier_topk_f64(_p(s), rows, l, l, k, _p(sel), _stream()))
    else:
        lib = _lib.load()
        wsb = lib.fier_topk_workspace(rows, l, k) if wide else 0
        ws = torch.empty(wsb, dtype=torch.uint8, device=s.device) if wsb else None
        check(lib.fier_topk(_p(s), rows, l, l, k, _p(sel), _p(ws) if ws is not None else None, wsb, _stream()))
    return sel


def _validate_selection(sel: torch.Tensor, tokens: int) -> None:
    # Selection::valid_against (core.hpp:86-93)
    _require(sel.shape[-1] >= 1, "gather_attention: empty selection")
    ok = bool(((sel >= 0) & (sel < tokens)).all().item())
    if sel.shape[-1] > 1:
        ok = ok and bool((sel[..., 1:] > sel[..., :-1]).all().item())
    _require(ok, "gather_attention: selection invalid for cache")


def gather_attention(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, sel: torch.Tensor,
                     scaled: bool = True, tokens: Optional[int] = None,
                     validate: bool = True) -> torch.Tensor:
    """gather_attention (core.hpp:152-179): fp32 [d] or [B, Hq, d]."""
    single = q.dim() == 1
    K4, V4 = _as4(_cuda(K, "gather_attention")), _as4(_cuda(V, "gather_attention"))
    _require(K4.shape == V4.shape, "gather_attention: K and V are not row-aligned")
    q3 = _as3(_cuda(q, "gather_attention"))
    B, Hkv, cap, d = K4.shape
    _require(q3.shape[-1] == d, "gather_attention: query length does not match key dim")
    Hq = q3.shape[1]
    sel3 = sel.to(torch.int32).reshape(B, Hq, -1).contiguous()
    n = sel3.shape[-1]
    tokens = cap if tokens is None else tokens
    if validate:
        _validate_selection(sel3, tokens)
    shape = make_shape(B, Hq, Hkv, cap, d, 32, _dtype_code(K4))
    lib = _lib.load()
    ws_bytes = lib.fier_sparse_attention_workspace(C.byref(shape), n)
    ws = torch.empty(max(ws_bytes, 4), dtype=torch.uint8, device=q3.device)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=q3.device)
    scale = 1.0 / math.sqrt(d) if scaled else 1.0
    check(lib.fier_sparse_attention(C.byref(shape), _p(q3.to(K4.dtype)), _p(K4), _p(V4), _p(sel3), n,
                                    tokens, scale, _p(out), _p(ws), ws.numel(), _stream()))
    return out.view(-1) if single else out


def full_attention(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, scaled: bool = True,
                   tokens: Optional[int] = None) -> torch.Tensor:
    """gather_attention over every index (`full` policy, retrieval.hpp:159-166) -- K0."""
    single = q.dim() == 1
    K4, V4 = _as4(_cuda(K, "gather_attention")), _as4(_cuda(V, "gather_attention"))
    q3 = _as3(_cuda(q, "gather_attention"))
    B, Hkv, cap, d = K4.shape
    Hq = q3.shape[1]
    tokens = cap if tokens is None else tokens
    shape = make_shape(B, Hq, Hkv, cap, d, 32, _dtype_code(K4))
    lib = _lib.load()
    ws = torch.empty(max(lib.fier_full_attention_workspace(C.byref(shape), tokens), 4),
                     dtype=torch.uint8, device=q3.device)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=q3.device)
    scale = 1.0 / math.sqrt(d) if scaled else 1.0
    check(lib.fier_full_attention(C.byref(shape), _p(q3.to(K4.dtype)), _p(K4), _p(V4), tokens, scale,
                                  _p(out), _p(ws), ws.numel(), _stream()))
    return out.view(-1) if single else out


def fier_select(q: torch.Tensor, pk: PackedKeys, n: int) -> torch.Tensor:
    """fier_select (retrieval.hpp:130-133)."""
    _require(1 <= n <= pk.tokens, "fier_select: budget out of range")
    return topk_oracle(approx_scores(q, pk), n)


@dataclass
class RetrievalResult:
    """RetrievalResult (retrieval.hpp:122-127)."""
    selection: torch.Tensor
    output: torch.Tensor
    est_scores: torch.Tensor
    bytes_loaded_for_estimation: int


def fier_attend(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, pk: PackedKeys,
                n: int) -> RetrievalResult:
    """fier_attend (retrieval.hpp:136-146): estimate, select, exact attention on the subset."""
    K4 = _as4(K)
    _require(pk.tokens == K4.shape[2] and pk.dim == K4.shape[3],
             "fier_attend: packed keys do not match cache")
    est = approx_scores(q, pk)
    _require(1 <= n <= pk.tokens, "topk_oracle: k out of range")
    sel = topk_oracle(est, n)
    out = gather_attention(q, K, V, sel, scaled=True, validate=False)
    return RetrievalResult(sel, out, est, pk.payload_bytes())


class DecodeLayer:
    """One attention layer's decode-time state on the GPU, batched over B sequences.

    Holds the KV cache [B, Hkv, cap, d], the Fier index, and the workspace of
    ``fier_decode_step``; ``step`` is graph-capturable (no host sync, no
    allocation).
    """

    def __init__(self, batch, q_heads, kv_heads, capacity, dim, group=32, dtype=torch.bfloat16,
                 device="cuda", K=None, V=None):
        self.B, self.Hq, self.Hkv, self.cap, self.d, self.g = batch, q_heads, kv_heads, capacity, dim, group
        self.dtype = dtype
        self.device = torch.device(device)
        self.K = K if K is not None else torch.zeros((batch, kv_heads, capacity, dim), dtype=dtype,
                                                     device=device)
        self.V = V if V is not None else torch.zeros_like(self.K)
        self.pk = alloc_index(batch, kv_heads, capacity, dim, group, device)
        self.shape = make_shape(batch, q_heads, kv_heads, capacity, dim, group, _DT[dtype])
        self.tokens = 0
        self._ws = None
        self._ws_key = None

    def prefill(self, tokens: int) -> None:
        """Pack the prefix [0, tokens) of the cache (hoisted quantize)."""
        quantize(self.K, self.g, tokens=tokens, out=self.pk)
        self.tokens = tokens

    def workspace(self, tokens: int, n: int) -> torch.Tensor:
        key = (tokens, n)
        need = _lib.load().fier_decode_workspace(C.byref(self.shape), tokens, n)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        self._ws_key = key
        return self._ws

    def step(self, q, k_new, v_new, pos: int, n: int, out=None, sel=None, scores_out=None,
             scale: Optional[float] = None, rope: Optional[Tuple[float, int, bool]] = None,
             host_inputs: bool = False, separate: bool = False,
             nonfinite: Optional[torch.Tensor] = None):
        """fier_attend for a decode step: append token `pos`, score, select n, attend.

        rope = (base, rotary_dim, interleaved): rotate q and k_new by position `pos`
        inside the step (fier_decode_step_ex; the cache stores the rotated k row).
        host_inputs: q / k_new / v_new are pinned host tensors (FIER_STEP_HOST_INPUTS).
        separate: force the separate-kernel path (FIER_STEP_SEPARATE).
        nonfinite: an int32 device tensor the step ORs FIER_NONFINITE_KEY (1) /
        FIER_NONFINITE_QUERY (2) into; check it with ``raise_nonfinite``."""
        lib = _lib.load()
        tokens = pos + 1
        ws = self.workspace(tokens, n) if self._ws_key != (tokens, n) else self._ws
        if out is None:
            out = torch.empty((self.B, self.Hq, self.d), dtype=torch.float32, device=self.device)
        if sel is None:
            sel = torch.empty((self.B, self.Hq, n), dtype=torch.int32, device=self.device)
        scale = 1.0 / math.sqrt(self.d) if scale is None else scale
        rp = None
        if rope is not None:
            base, rd, inter = rope
            rp = C.byref(_lib.FierRope(float(base), int(rd), 1 if inter else 0))
        flags = (_lib.FIER_STEP_HOST_INPUTS if host_inputs else 0) | (_lib.FIER_STEP_SEPARATE if separate else 0)
        check(lib.fier_decode_step_ex(C.byref(self.shape), _p(q), _p(k_new), _p(v_new), pos, _p(self.K),
                                      _p(self.V), _p(self.pk.bits), _p(self.pk.params), n, scale, rp, flags,
                                      _p(nonfinite), _p(out), _p(sel), _p(scores_out), _p(ws), ws.numel(),
                                      _stream()))
        self.pk.tokens = max(self.pk.tokens, tokens)
        self.tokens = max(self.tokens, tokens)
        return out, sel

    def launches(self, tokens: int, n: int, host_inputs: bool = False, rope: bool = False,
                 separate: bool = False) -> int:
        """Kernel launches one step issues (fier_decode_step_launches)."""
        flags = (_lib.FIER_STEP_HOST_INPUTS if host_inputs else 0) | (_lib.FIER_STEP_SEPARATE if separate else 0)
        return int(_lib.load().fier_decode_step_launches(C.byref(self.shape), tokens, n, flags, 1 if rope else 0))

    def full_step(self, q, tokens: int, out=None, ws=None, scale: Optional[float] = None):
        """K0: full-KV decode attention over [0, tokens) (the baseline)."""
        lib = _lib.load()
        need = lib.fier_full_attention_workspace(C.byref(self.shape), tokens)
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        if out is None:
            out = torch.empty((self.B, self.Hq, self.d), dtype=torch.float32, device=self.device)
        scale = 1.0 / math.sqrt(self.d) if scale is None else scale
        check(lib.fier_full_attention(C.byref(self.shape), _p(q), _p(self.K), _p(self.V), tokens, scale,
                                      _p(out), _p(ws), ws.numel(), _stream()))
        return out


def raise_nonfinite(flag: torch.Tensor) -> None:
    """Raise the reference's error for a decode step's non-finite status word (a host sync):
    "quantize: non-finite key entry" (quant1bit.hpp:68) or "softmax: non-finite logit"
    (core.hpp:122)."""
    v = int(flag.item())
    if v & _lib.FIER_NONFINITE_KEY:
        raise ValueError("quantize: non-finite key entry")
    if v & _lib.FIER_NONFINITE_QUERY:
        raise ValueError("softmax: non-finite logit")


# ---- KVD1 cache dumps straight to/from the device (io.hpp:110-185) -----------------

def load_cache_dump(buf, device="cuda") -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """parse_cache_dump (io.hpp:140-185) decoded on the GPU (fier_kvd1_load).  buf: bytes or a
    CUDA uint8 tensor.  Returns fp32 CUDA tensors K [l, d], V [l, d], queries [nq, d] (exact)."""
    if not isinstance(buf, torch.Tensor):
        buf = torch.from_numpy(np.frombuffer(bytes(buf), np.uint8).copy()).to(device)
    _require(buf.is_cuda and buf.dtype == torch.uint8, "load_cache_dump: expected bytes or a CUDA uint8 tensor")
    buf = buf.contiguous()
    lib = _lib.load()
    l, d, nq, dt = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    check(lib.fier_kvd1_load(_p(buf), buf.numel(), C.byref(l), C.byref(d), C.byref(nq), C.byref(dt), None, 0,
                             _stream()))
    l, d, nq = l.value, d.value, nq.value
    vals = torch.empty((2 * l + nq) * d, dtype=torch.float32, device=buf.device)
    check(lib.fier_kvd1_load(_p(buf), buf.numel(), None, None, None, None, _p(vals), vals.numel(), _stream()))
    vals = vals.view(2 * l + nq, d)
    return vals[:l], vals[l:2 * l], vals[2 * l:]


def save_cache_dump(K: torch.Tensor, V: torch.Tensor, queries: Optional[torch.Tensor] = None,
                    dtype: str = "f16") -> torch.Tensor:
    """serialize_cache_dump (io.hpp:110-137) encoded on the GPU (fier_kvd1_store) into a CUDA
    uint8 tensor.  K, V: [l, d]; queries: [nq, d]; dtype "f16" (round to nearest even) or "f32"."""
    _require(K.dim() == 2 and K.shape == V.shape, "serialize_cache_dump: K and V shapes differ")
    l, d = K.shape
    Q = queries if queries is not None else K.new_zeros((0, d))
    _require(Q.dim() == 2 and Q.shape[1] == d, "serialize_cache_dump: query length does not match dim")
    _require(dtype in ("f16", "f32"), "serialize_cache_dump: dtype must be f16 or f32")
    vals = torch.cat([_cuda(K, "K").float(), _cuda(V, "V").float(), _cuda(Q, "queries").float()]).contiguous()
    code = 0 if dtype == "f16" else 1
    out = torch.empty(20 + vals.numel() * (2 if code == 0 else 4), dtype=torch.uint8, device=vals.device)
    check(_lib.load().fier_kvd1_store(_p(vals), l, d, Q.shape[0], code, _p(out), out.numel(), _stream()))
    return out


# ---- Quest page retrieval (baselines.hpp) ------------------------

_VARIANTS = {"sum": 1, "sum_over_channels": 1, "max": 0, "max_over_channels": 0}


@dataclass
class PageSummaries:
    """build_page_summaries (baselines.hpp:16-56) on the device: fp32 [B, Hkv, P, d]."""
    max_vecs: torch.Tensor
    min_vecs: torch.Tensor
    page_size: int
    tokens: int
    dim: int
    single: bool = False

    def page_count(self) -> int:
        return self.max_vecs.shape[-2]


def build_page_summaries(K: torch.Tensor, page_size: int = 16, tokens: Optional[int] = None) -> PageSummaries:
    """build_page_summaries (baselines.hpp:34-56).  K: [l, d] or [B, Hkv, cap, d]."""
    _require(page_size >= 1, "build_page_summaries: page size must be >= 1")
    single = K.dim() == 2
    K4 = _as4(_cuda(K, "build_page_summaries"))
    B, H, cap, d = K4.shape
    tokens = cap if tokens is None else tokens
    _require(1 <= tokens <= cap, "build_page_summaries: empty key cache")
    P = (tokens + page_size - 1) // page_size
    kmax = torch.empty((B, H, P, d), dtype=torch.float32, device=K4.device)
    kmin = torch.empty_like(kmax)
    shape = make_shape(B, H, H, cap, d, 1, _dtype_code(K4))
    check(_lib.load().fier_quest_summaries(C.byref(shape), _p(K4), tokens, page_size, _p(kmax), _p(kmin),
                                           _stream()))
    return PageSummaries(kmax, kmin, page_size, tokens, d, single)


def quest_page_scores(q: torch.Tensor, ps: PageSummaries, variant: str = "sum") -> torch.Tensor:
    """quest_page_scores (baselines.hpp:60-79): fp32 [P] or [B, Hq, P] (fp64 evaluation)."""
    _require(variant in _VARIANTS, "quest_page_scores: variant must be sum or max")
    _require(q.shape[-1] == ps.dim, "quest_page_scores: query length does not match dim")
    single = q.dim() == 1
    q3 = _as3(_cuda(q, "quest_page_scores"))
    B, Hq, d = q3.shape
    Hkv = ps.max_vecs.shape[1]
    _require(B == ps.max_vecs.shape[0] and Hq % Hkv == 0, "quest_page_scores: query heads do not match")
    P = ps.page_count()
    out = torch.empty((B, Hq, P), dtype=torch.float32, device=q3.device)
    shape = make_shape(B, Hq, Hkv, max(ps.tokens, 1), d, 1, _dtype_code(q3))
    check(_lib.load().fier_quest_page_scores(C.byref(shape), _p(q3), _p(ps.max_vecs), _p(ps.min_vecs), ps.tokens,
                                             ps.page_size, _VARIANTS[variant], _p(out), P, _stream()))
    return out.view(-1) if single else out


def select_by_page_scores(page_scores: torch.Tensor, tokens: int, page_size: int, n: int) -> torch.Tensor:
    """detail::select_by_page_scores (baselines.hpp:85-111): int32 ascending [n] or [..., n]."""
    s = _cuda(page_scores, "page selection")
    _require(s.dtype == torch.float32, "page selection: page scores must be float32")
    _require(1 <= n <= tokens, "page selection: budget out of range")
    P = s.shape[-1]
    _require(P == (tokens + page_size - 1) // page_size, "page selection: page count does not match tokens")
    rows = s.numel() // P
    lib = _lib.load()
    ws = torch.empty(max(1, lib.fier_page_select_workspace(rows, tokens, page_size, n)), dtype=torch.uint8,
                     device=s.device)
    sel = torch.empty(s.shape[:-1] + (n,), dtype=torch.int32, device=s.device)
    check(lib.fier_page_select(_p(s), rows, tokens, P, page_size, n, _p(sel), _p(ws), ws.numel(), _stream()))
    return sel


def quest_select(q: torch.Tensor, K: torch.Tensor, ps: PageSummaries, n: int, variant: str = "sum") -> torch.Tensor:
    """quest_select (baselines.hpp:113-118)."""
    _require(K.shape[-2] >= ps.tokens and K.shape[-1] == ps.dim, "quest_select: summaries do not match cache")
    return select_by_page_scores(quest_page_scores(q, ps, variant), ps.tokens, ps.page_size, n)


def quest_select_quantized(q: torch.Tensor, pk: PackedKeys, page_size: int, n: int) -> torch.Tensor:
    """quest_select_quantized (baselines.hpp:120-140): pages scored by the mean of the
    members' approx_scores (K2 on the GPU), ranked and filled like quest_select."""
    _require(page_size >= 1, "quest_select_quantized: page size must be >= 1")
    est = approx_scores(q, pk)
    rows, l = est.numel() // pk.tokens, pk.tokens
    P = (l + page_size - 1) // page_size
    pscores = torch.empty(est.shape[:-1] + (P,), dtype=torch.float32, device=est.device)
    check(_lib.load().fier_page_mean(_p(est), rows, l, l, page_size, _p(pscores), P, _stream()))
    return select_by_page_scores(pscores, l, page_size, n)

