"""ctypes loaders for the parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import
this module.  The product package (``paper_2508_08256_b200``) never does.

* :class:`Port` -- the C restatement (``oracle/fier_oracle.c``).
* :class:`Ref`  -- the reference itself, compiled from its own headers
  (``oracle/_ref/libfier_ref.so``, built by ``oracle/Makefile``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfier_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def build() -> None:
    """Compile the port (and the reference, where its headers exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(ValueError):
    pass


class Port:
    """C restatement of quant1bit.hpp / core.hpp / io.hpp / half.hpp."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.fo_half_to_double.argtypes = [C.c_uint16]
        L.fo_half_to_double.restype = C.c_double
        L.fo_double_to_half.argtypes = [C.c_double]
        L.fo_double_to_half.restype = C.c_uint16
        L.fo_payload_bytes.argtypes = [_sz, _sz, _sz]
        L.fo_payload_bytes.restype = _sz
        L.fo_quantize.argtypes = [_dp, _sz, _sz, _sz, _u64p, _dp, _dp]
        L.fo_serialize_packed.argtypes = [_sz, _sz, _sz, _u64p, _dp, _dp, _u8p]
        L.fo_serialize_packed.restype = _sz
        L.fo_parse_header.argtypes = [_u8p, _sz, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(_sz)]
        L.fo_parse_packed.argtypes = [_u8p, _sz, _u64p, _dp, _dp]
        L.fo_approx_scores.argtypes = [_dp, _sz, _sz, _sz, _u64p, _dp, _dp, _dp]
        L.fo_approx_scores.restype = None
        L.fo_exact_scores.argtypes = [_dp, _dp, _sz, _sz, C.c_int, _dp]
        L.fo_exact_scores.restype = None
        L.fo_topk.argtypes = [_dp, _sz, _sz, _i64p]
        L.fo_gather_attention.argtypes = [_dp, _dp, _dp, _sz, _sz, _i64p, _sz, C.c_int, _dp]
        L.fo_recall.argtypes = [_i64p, _i64p, _sz]
        L.fo_recall.restype = C.c_double
        L.fo_relative_l2_error.argtypes = [_dp, _dp, _sz]
        L.fo_relative_l2_error.restype = C.c_double
        L.fo_fier_attend.argtypes = [_dp, _dp, _dp, _sz, _sz, _sz, _u64p, _dp, _dp, _sz, _i64p, _dp]
        L.fo_page_summaries.argtypes = [_dp, _sz, _sz, _sz, _dp, _dp]
        L.fo_quest_page_scores.argtypes = [_dp, _dp, _dp, _sz, _sz, C.c_int, _dp]
        L.fo_page_mean.argtypes = [_dp, _sz, _sz, _dp]
        L.fo_select_by_page_scores.argtypes = [_dp, _sz, _sz, _sz, _i64p]

    # half.hpp
    def double_to_half(self, x: float) -> int:
        return int(self.lib.fo_double_to_half(float(x)))

    def half_to_double(self, h: int) -> float:
        return float(self.lib.fo_half_to_double(int(h)))

    # quant1bit.hpp
    def quantize(self, K, g: int):
        K = _c64(K)
        l, d = K.shape
        G = (l + g - 1) // g
        cw = np.zeros(l * ((d + 63) // 64), np.uint64)
        s = np.zeros(G * d)
        z = np.zeros(G * d)
        if self.lib.fo_quantize(K, l, d, g, cw, s, z):
            raise OracleError("quantize: invalid input")
        return cw, s, z

    def serialize(self, l, d, g, cw, s, z) -> bytes:
        out = np.zeros(18 + self.lib.fo_payload_bytes(l, d, g), np.uint8)
        n = self.lib.fo_serialize_packed(l, d, g, cw, s, z, out)
        return out[:n].tobytes()

    def quantize_fier(self, K, g: int) -> bytes:
        K = _c64(K)
        l, d = K.shape
        return self.serialize(l, d, g, *self.quantize(K, g))

    def parse(self, buf: bytes):
        b = np.frombuffer(buf, np.uint8).copy()
        l, d, g = _sz(), _sz(), _sz()
        if self.lib.fo_parse_header(b, len(b), C.byref(l), C.byref(d), C.byref(g)):
            raise OracleError("parse: bad FIER buffer")
        l, d, g = l.value, d.value, g.value
        G = (l + g - 1) // g
        cw = np.zeros(l * ((d + 63) // 64), np.uint64)
        s = np.zeros(G * d)
        z = np.zeros(G * d)
        self.lib.fo_parse_packed(b, len(b), cw, s, z)
        return (l, d, g), cw, s, z

    def approx_scores_fier(self, q, buf: bytes) -> np.ndarray:
        (l, d, g), cw, s, z = self.parse(buf)
        out = np.zeros(l)
        self.lib.fo_approx_scores(_c64(q), l, d, g, cw, s, z, out)
        return out

    def approx_scores_packed(self, q, l, d, g, cw, s, z) -> np.ndarray:
        out = np.zeros(l)
        self.lib.fo_approx_scores(_c64(q), l, d, g, cw, _c64(s), _c64(z), out)
        return out

    # core.hpp
    def exact_scores(self, q, K, scaled=False) -> np.ndarray:
        K = _c64(K)
        out = np.zeros(K.shape[0])
        self.lib.fo_exact_scores(_c64(q), K, K.shape[0], K.shape[1], int(scaled), out)
        return out

    def topk(self, scores, k: int) -> np.ndarray:
        scores = _c64(scores)
        out = np.zeros(k, np.int64)
        if self.lib.fo_topk(scores, scores.size, k, out):
            raise OracleError("topk_oracle: k out of range")
        return out

    def gather_attention(self, q, K, V, idx, scaled=True) -> np.ndarray:
        K, V = _c64(K), _c64(V)
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.zeros(K.shape[1])
        if self.lib.fo_gather_attention(_c64(q), K, V, K.shape[0], K.shape[1], idx, idx.size,
                                        int(scaled), out):
            raise OracleError("gather_attention: invalid selection")
        return out

    def recall(self, got, want) -> float:
        got = np.ascontiguousarray(got, np.int64)
        want = np.ascontiguousarray(want, np.int64)
        return float(self.lib.fo_recall(got, want, got.size))

    def relative_l2_error(self, got, want) -> float:
        got, want = _c64(got), _c64(want)
        return float(self.lib.fo_relative_l2_error(got, want, got.size))

    def fier_attend_fier(self, q, K, V, buf: bytes, n: int):
        """fier_attend (retrieval.hpp:136) over a FIER-serialized index."""
        (l, d, g), cw, s, z = self.parse(buf)
        sel = np.zeros(n, np.int64)
        out = np.zeros(d)
        if self.lib.fo_fier_attend(_c64(q), _c64(K), _c64(V), l, d, g, cw, s, z, n, sel, out):
            raise OracleError("fier_attend: invalid input")
        return sel, out


    # baselines.hpp (Quest page retrieval)
    def page_summaries(self, K, L: int):
        """build_page_summaries (baselines.hpp:34): (kmax, kmin) [ceil(l/L), d]."""
        K = _c64(K)
        l, d = K.shape
        P = (l + L - 1) // L
        kmax, kmin = np.zeros((P, d)), np.zeros((P, d))
        if self.lib.fo_page_summaries(K, l, d, L, kmax, kmin):
            raise OracleError("build_page_summaries: page size must be >= 1")
        return kmax, kmin

    def quest_page_scores(self, q, kmax, kmin, variant: str = "sum") -> np.ndarray:
        """quest_page_scores (baselines.hpp:60); variant "sum" or "max" over channels."""
        kmax, kmin = _c64(kmax), _c64(kmin)
        out = np.zeros(kmax.shape[0])
        self.lib.fo_quest_page_scores(_c64(q), kmax, kmin, kmax.shape[0], kmax.shape[1], int(variant == "sum"), out)
        return out

    def page_mean(self, est, L: int) -> np.ndarray:
        """quest_select_quantized's page scores (baselines.hpp:131-139)."""
        est = _c64(est)
        out = np.zeros((est.size + L - 1) // L)
        if self.lib.fo_page_mean(est, est.size, L, out):
            raise OracleError("quest_select_quantized: page size must be >= 1")
        return out

    def select_by_page_scores(self, page_scores, l: int, L: int, n: int) -> np.ndarray:
        """detail::select_by_page_scores (baselines.hpp:85)."""
        out = np.zeros(n, np.int64)
        if self.lib.fo_select_by_page_scores(_c64(page_scores), l, L, n, out):
            raise OracleError("page selection: budget out of range")
        return out

    def quest_select(self, q, K, L: int, n: int, variant: str = "sum") -> np.ndarray:
        kmax, kmin = self.page_summaries(K, L)
        return self.select_by_page_scores(self.quest_page_scores(q, kmax, kmin, variant), len(K), L, n)


class Ref:
    """The reference's own functions (oracle/_ref/libfier_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_double_to_half.argtypes = [C.c_double]
        L.ref_double_to_half.restype = C.c_uint16
        L.ref_half_to_double.argtypes = [C.c_uint16]
        L.ref_half_to_double.restype = C.c_double
        L.ref_quantize_fier.argtypes = [_dp, _sz, _sz, _sz, C.c_void_p, _sz, C.POINTER(_sz)]
        L.ref_quantize_inmem.argtypes = [_dp, _sz, _sz, _sz, _u64p, _dp, _dp]
        L.ref_approx_scores_fier.argtypes = [_dp, _u8p, _sz, _dp]
        L.ref_topk.argtypes = [_dp, _sz, _sz, _i64p]
        L.ref_load_ratio_fier.argtypes = [_sz, _sz, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                          C.POINTER(C.c_int)]
        L.ref_gather_attention.argtypes = [_dp, _dp, _dp, _sz, _sz, _i64p, _sz, C.c_int, _dp]
        L.ref_exact_scores.argtypes = [_dp, _dp, _sz, _sz, C.c_int, _dp]
        L.ref_fier_attend_fier.argtypes = [_dp, _dp, _dp, _sz, _sz, _u8p, _sz, _sz, _i64p, _dp, _dp,
                                           C.POINTER(C.c_uint64)]
        L.ref_generate.argtypes = [_sz, _sz, C.c_int, _sz, C.c_double, C.c_uint64, _sz, _dp, _dp, _dp]
        L.ref_layer_build.argtypes = [_fp, _fp, _sz, _sz, _sz, _sz, _sz]
        L.ref_layer_build.restype = C.c_void_p
        L.ref_layer_free.argtypes = [C.c_void_p]
        L.ref_layer_step.argtypes = [C.c_void_p, _fp, _sz, _sz, _sz, _sz, _sz, C.c_void_p, C.c_void_p]
        L.ref_layer_step.restype = C.c_double
        L.ref_page_summaries.argtypes = [_dp, _sz, _sz, _sz, _dp, _dp]
        L.ref_quest_page_scores.argtypes = [_dp, _dp, _sz, _sz, _sz, C.c_int, _dp]
        L.ref_quest_select.argtypes = [_dp, _dp, _sz, _sz, _sz, _sz, C.c_int, _i64p]
        L.ref_quest_select_quantized.argtypes = [_dp, _u8p, _sz, _sz, _sz, _i64p]
        L.ref_select_by_page_scores.argtypes = [_dp, _sz, _sz, _sz, _i64p]
        L.ref_margin_and_errors.argtypes = [_dp, _dp, _sz, _sz, _u8p, _sz, _sz, _dp]
        L.ref_run_trial.argtypes = [_dp, _dp, _sz, _sz, _dp, _sz, _sz, _sz, C.c_int, C.POINTER(_sz), _sz, _dp, _dp]

    def _check(self, rc: int):
        if rc:
            raise OracleError(self.lib.ref_last_error().decode())

    def double_to_half(self, x):
        return int(self.lib.ref_double_to_half(float(x)))

    def half_to_double(self, h):
        return float(self.lib.ref_half_to_double(int(h)))

    def quantize_fier(self, K, g: int) -> bytes:
        K = _c64(K)
        l, d = K.shape
        n = _sz()
        self._check(self.lib.ref_quantize_fier(K, l, d, g, None, 0, C.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        self._check(self.lib.ref_quantize_fier(K, l, d, g, buf.ctypes.data, n.value, C.byref(n)))
        return buf.tobytes()

    def quantize_inmem(self, K, g: int):
        K = _c64(K)
        l, d = K.shape
        G = (l + g - 1) // g
        cw = np.zeros(l * ((d + 63) // 64), np.uint64)
        s = np.zeros(G * d)
        z = np.zeros(G * d)
        self._check(self.lib.ref_quantize_inmem(K, l, d, g, cw, s, z))
        return cw, s, z

    def approx_scores_fier(self, q, buf: bytes) -> np.ndarray:
        b = np.frombuffer(buf, np.uint8).copy()
        l = int.from_bytes(buf[6:10], "little")
        out = np.zeros(l)
        self._check(self.lib.ref_approx_scores_fier(_c64(q), b, len(b), out))
        return out

    def topk(self, scores, k: int) -> np.ndarray:
        scores = _c64(scores)
        out = np.zeros(k, np.int64)
        self._check(self.lib.ref_topk(scores, scores.size, k, out))
        return out

    def load_ratio_fier(self, l: int, g: int):
        """load_ratio_fier (quant1bit.hpp:176-184): ((num_bits, den_bits), (num, den) reduced, formula)."""
        bits = (C.c_longlong * 2)()
        ratio = (C.c_longlong * 2)()
        formula = C.c_int()
        self._check(self.lib.ref_load_ratio_fier(l, g, bits, ratio, C.byref(formula)))
        return (bits[0], bits[1]), (ratio[0], ratio[1]), bool(formula.value)

    def gather_attention(self, q, K, V, idx, scaled=True) -> np.ndarray:
        K, V = _c64(K), _c64(V)
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.zeros(K.shape[1])
        self._check(self.lib.ref_gather_attention(_c64(q), K, V, K.shape[0], K.shape[1], idx,
                                                  idx.size, int(scaled), out))
        return out

    def exact_scores(self, q, K, scaled=False) -> np.ndarray:
        K = _c64(K)
        out = np.zeros(K.shape[0])
        self._check(self.lib.ref_exact_scores(_c64(q), K, K.shape[0], K.shape[1], int(scaled), out))
        return out

    def fier_attend_fier(self, q, K, V, buf: bytes, n: int):
        K, V = _c64(K), _c64(V)
        l, d = K.shape
        b = np.frombuffer(buf, np.uint8).copy()
        sel = np.zeros(n, np.int64)
        out = np.zeros(d)
        est = np.zeros(l)
        nbytes = C.c_uint64()
        self._check(self.lib.ref_fier_attend_fier(_c64(q), K, V, l, d, b, len(b), n, sel, out, est,
                                                  C.byref(nbytes)))
        return sel, out, est, int(nbytes.value)

    def page_summaries(self, K, L: int):
        K = _c64(K)
        l, d = K.shape
        P = (l + L - 1) // L
        kmax, kmin = np.zeros((P, d)), np.zeros((P, d))
        self._check(self.lib.ref_page_summaries(K, l, d, L, kmax, kmin))
        return kmax, kmin

    def quest_page_scores(self, q, K, L: int, variant: str = "sum") -> np.ndarray:
        K = _c64(K)
        out = np.zeros((K.shape[0] + L - 1) // L)
        self._check(self.lib.ref_quest_page_scores(_c64(q), K, K.shape[0], K.shape[1], L, int(variant == "sum"),
                                                   out))
        return out

    def quest_select(self, q, K, L: int, n: int, variant: str = "sum") -> np.ndarray:
        K = _c64(K)
        out = np.zeros(n, np.int64)
        self._check(self.lib.ref_quest_select(_c64(q), K, K.shape[0], K.shape[1], L, n, int(variant == "sum"),
                                              out))
        return out

    def quest_select_quantized(self, q, buf: bytes, L: int, n: int) -> np.ndarray:
        b = np.frombuffer(buf, np.uint8).copy()
        out = np.zeros(n, np.int64)
        self._check(self.lib.ref_quest_select_quantized(_c64(q), b, len(b), L, n, out))
        return out

    def select_by_page_scores(self, page_scores, l: int, L: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.int64)
        self._check(self.lib.ref_select_by_page_scores(_c64(page_scores), l, L, n, out))
        return out

    def margin_and_errors(self, q, K, buf: bytes, k: int) -> np.ndarray:
        """evalharness.hpp:63 -> (margin, max_err, l2_loss, hinge_loss, hinge_loss_symmetric)."""
        K = _c64(K)
        b = np.frombuffer(buf, np.uint8).copy()
        out = np.zeros(5)
        self._check(self.lib.ref_margin_and_errors(_c64(q), K, K.shape[0], K.shape[1], b, len(b), k, out))
        return out

    def run_trial(self, K, V, Q, g: int, L: int, budgets, variant: str = "sum"):
        """run_trial (evalharness.hpp:184), policies fier, quest, quest_quant, oracle, full:
        cells [5, len(budgets), 3] = (recall, out_err, max_err), margins [len(budgets)]."""
        K, V, Q = _c64(K), _c64(V), _c64(np.atleast_2d(Q))
        nb = len(budgets)
        bud = (_sz * nb)(*budgets)
        cells = np.zeros((5, nb, 3))
        margins = np.zeros(nb)
        self._check(self.lib.ref_run_trial(K, V, K.shape[0], K.shape[1], Q, Q.shape[0], g, L, int(variant == "sum"),
                                           bud, nb, cells, margins))
        return cells, margins

    def generate(self, l, d, planted=False, spike_count=4, spike_gain=1e3, seed=0, query_count=1):
        K = np.zeros((l, d))
        V = np.zeros((l, d))
        Q = np.zeros((query_count, d))
        self._check(self.lib.ref_generate(l, d, int(planted), spike_count, spike_gain, seed,
                                          query_count, K, V, Q))
        return K, V, Q


class RefLayer:
    """Multi-head decode step on the reference (hoisted index, std::thread pool)."""

    def __init__(self, ref: Ref, K: np.ndarray, V: np.ndarray, g: int = 32, threads: int = 0):
        K = np.ascontiguousarray(K, np.float32)
        V = np.ascontiguousarray(V, np.float32)
        self.ref = ref
        self.hkv, self.l, self.d = K.shape
        self.threads = threads or os.cpu_count() or 1
        self.h = ref.lib.ref_layer_build(K, V, self.hkv, self.l, self.d, g, self.threads)

    def step(self, Q: np.ndarray, n: int, heads=None, want_outputs=False):
        Q = np.ascontiguousarray(Q, np.float32)
        hq = Q.shape[0]
        h0, h1 = (0, hq) if heads is None else heads
        sel = np.zeros((hq, n), np.int32) if want_outputs else None
        out = np.zeros((hq, self.d)) if want_outputs else None
        secs = self.ref.lib.ref_layer_step(self.h, Q, hq, h0, h1, n, self.threads,
                                           sel.ctypes.data if want_outputs else None,
                                           out.ctypes.data if want_outputs else None)
        if secs < 0:
            raise OracleError(self.ref.lib.ref_last_error().decode())
        return secs, sel, out

    def close(self):
        if self.h:
            self.ref.lib.ref_layer_free(self.h)
            self.h = None

    def __del__(self):
        self.close()
