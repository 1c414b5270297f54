"""ctypes binding of libfier_cuda.so (include/fier_cuda.h).

There is no fallback: if the library is missing or no CUDA device is present,
every compute entry point raises.  The .so is built in-tree by
``python -m paper_2508_08256_b200.build`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

# FIER_LIB: load another in-tree build of the same sources (tools: the -DFIER_STEP_TRACE variant)
LIB_PATH = os.environ.get("FIER_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfier_cuda.so")

FIER_OK, FIER_EINVAL, FIER_EDATA, FIER_ECUDA = 0, 1, 2, 3
FIER_F32, FIER_F16, FIER_BF16, FIER_F64 = 0, 1, 2, 3
FIER_STEP_HOST_INPUTS, FIER_STEP_SEPARATE = 1, 2
FIER_NONFINITE_KEY, FIER_NONFINITE_QUERY = 1, 2

# every symbol include/fier_cuda.h declares
EXPORTS = (
    "fier_last_error", "fier_version", "fier_bits_bytes", "fier_params_bytes", "fier_payload_bytes",
    "fier_pack_keys", "fier_append", "fier_score", "fier_topk_workspace", "fier_topk",
    "fier_sparse_attention_workspace", "fier_sparse_attention", "fier_full_attention_workspace",
    "fier_full_attention", "fier_decode_workspace", "fier_step_scores_ld", "fier_decode_step",
    "fier_decode_step_launches", "fier_decode_step_ex",
    "fier_index_to_fier", "fier_fier_to_index", "fier_sparse_attention_ragged", "fier_shard_bounds",
    "fier_shard_candidates", "fier_shard_merge_workspace", "fier_shard_merge", "fier_lse_merge",
    "fier_index_export", "fier_index_import", "fier_kvd1_load", "fier_kvd1_store",
    "fier_quest_summaries", "fier_quest_page_scores", "fier_page_mean", "fier_page_select_workspace",
    "fier_page_select", "fier_exact_scores", "fier_margin_errors_workspace", "fier_margin_errors", "fier_overlap",
    "fier_topk_f64", "fier_load_ratio_fier",
)


class FierShape(C.Structure):
    _fields_ = [("batch", C.c_int32), ("q_heads", C.c_int32), ("kv_heads", C.c_int32),
                ("capacity", C.c_int32), ("dim", C.c_int32), ("group", C.c_int32),
                ("dtype", C.c_int32)]


class FierRope(C.Structure):
    """fier_rope: rotary embedding fused into the decode step (include/fier_cuda.h)."""
    _fields_ = [("base", C.c_float), ("rotary_dim", C.c_int32), ("interleaved", C.c_int32)]


class FierDataError(RuntimeError):
    """fier::DataError (io.hpp:29-31)."""


class FierCudaError(RuntimeError):
    """A CUDA launch/runtime failure inside the library."""


_vp = C.c_void_p
_sz = C.c_size_t
_i32 = C.c_int32
_i64 = C.c_int64
_SP = C.POINTER(FierShape)

_SIGS = {
    "fier_last_error": ([], C.c_char_p),
    "fier_version": ([], C.c_int),
    "fier_bits_bytes": ([_SP], _sz),
    "fier_params_bytes": ([_SP], _sz),
    "fier_payload_bytes": ([_i32, _i32, _i32], _sz),
    "fier_pack_keys": ([_SP, _vp, _i32, _vp, _vp, _vp, _vp], C.c_int),
    "fier_append": ([_SP, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp], C.c_int),
    "fier_score": ([_SP, _vp, _vp, _vp, _i32, _vp, _i64, _vp], C.c_int),
    "fier_topk_workspace": ([_i32, _i32, _i32], _sz),
    "fier_topk_f64": ([_vp, _i32, _i32, _i64, _i32, _vp, _vp], C.c_int),
    "fier_load_ratio_fier": ([_i64, _i64, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i32)], C.c_int),
    "fier_topk": ([_vp, _i32, _i32, _i64, _i32, _vp, _vp, _sz, _vp], C.c_int),
    "fier_sparse_attention_workspace": ([_SP, _i32], _sz),
    "fier_sparse_attention": ([_SP, _vp, _vp, _vp, _vp, _i32, _i32, C.c_float, _vp, _vp, _sz, _vp],
                              C.c_int),
    "fier_full_attention_workspace": ([_SP, _i32], _sz),
    "fier_full_attention": ([_SP, _vp, _vp, _vp, _i32, C.c_float, _vp, _vp, _sz, _vp], C.c_int),
    "fier_decode_workspace": ([_SP, _i32, _i32], _sz),
    "fier_step_scores_ld": ([_i32], _i64),
    "fier_decode_step_launches": ([_SP, _i32, _i32, C.c_uint32, _i32], _i32),
    "fier_decode_step_ex": ([_SP, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _i32, C.c_float, C.POINTER(FierRope),
                             C.c_uint32, _vp, _vp, _vp, _vp, _vp, _sz, _vp], C.c_int),
    "fier_decode_step": ([_SP, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _i32, C.c_float, _vp, _vp,
                          _vp, _vp, _sz, _vp], C.c_int),
    "fier_sparse_attention_ragged": ([_SP, _vp, _vp, _vp, _vp, _vp, _i32, _i32, C.c_float, _vp, _vp, _vp,
                                      _sz, _vp], C.c_int),
    "fier_shard_bounds": ([_i64, _i32, _i32, _i32, C.POINTER(_i64), C.POINTER(_i64)], C.c_int),
    "fier_shard_candidates": ([_vp, _i32, _i64, _vp, _i32, _i32, _i32, _vp, _vp, _vp], C.c_int),
    "fier_shard_merge_workspace": ([_i32, _i32, _i32, _i32], _sz),
    "fier_shard_merge": ([_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp], C.c_int),
    "fier_lse_merge": ([_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp], C.c_int),
    "fier_index_to_fier": ([_vp, _vp, _i32, _i32, _i32, _vp, _sz], C.c_int),
    "fier_fier_to_index": ([_vp, _sz, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), _vp, _sz, _vp,
                            _sz], C.c_int),
    "fier_index_export": ([_vp, _vp, _i32, _i32, _i32, _vp, _sz, _vp], C.c_int),
    "fier_index_import": ([_vp, _sz, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), _vp, _i64, _vp, _i64,
                           _vp], C.c_int),
    "fier_kvd1_load": ([_vp, _sz, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), _vp, _i64,
                        _vp], C.c_int),
    "fier_kvd1_store": ([_vp, _i32, _i32, _i32, _i32, _vp, _sz, _vp], C.c_int),
    "fier_quest_summaries": ([C.POINTER(FierShape), _vp, _i32, _i32, _vp, _vp, _vp], C.c_int),
    "fier_quest_page_scores": ([C.POINTER(FierShape), _vp, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _vp], C.c_int),
    "fier_page_mean": ([_vp, _i32, _i32, _i64, _i32, _vp, _i64, _vp], C.c_int),
    "fier_page_select_workspace": ([_i32, _i32, _i32, _i32], _sz),
    "fier_page_select": ([_vp, _i32, _i32, _i64, _i32, _i32, _vp, _vp, _sz, _vp], C.c_int),
    "fier_exact_scores": ([C.POINTER(FierShape), _vp, _vp, _i32, _i32, _vp, _vp, _i64, _vp], C.c_int),
    "fier_margin_errors_workspace": ([_i32, _i32], _sz),
    "fier_margin_errors": ([_vp, _vp, _vp, _i32, _i32, _i64, _i32, _vp, _vp, _sz, _vp], C.c_int),
    "fier_overlap": ([_vp, _i32, _vp, _i32, _i32, _vp, _vp], C.c_int),
}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the library (once).  Raises if it is missing: no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: the Fier CUDA library is required (build it with "
            "`python -m paper_2508_08256_b200.build`); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def last_error() -> str:
    return load().fier_last_error().decode()


def check(rc: int) -> None:
    if rc == FIER_OK:
        return
    msg = last_error()
    if rc == FIER_EINVAL:
        raise ValueError(msg)  # std::invalid_argument (core.hpp:19-21)
    if rc == FIER_EDATA:
        raise FierDataError(msg)
    raise FierCudaError(msg)
