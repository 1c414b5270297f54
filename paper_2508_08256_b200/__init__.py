"""B200-native (sm_100a) Fier decode-time KV retrieval (arxiv 2508.08256).

Hot path: 1-bit key packing -> packed q.K scoring -> per-head Top-k -> sparse
attention over the selected K/V rows, as hand-written CUDA kernels behind the
C ABI in include/fier_cuda.h.  ``api`` mirrors the reference's C++ entry points
(quantize, approx_scores, topk_oracle, gather_attention, fier_select,
fier_attend) on torch CUDA tensors.
"""
from . import _lib  # noqa: F401
from .api import (  # noqa: F401
    DecodeLayer,
    LoadRatio,
    load_ratio_fier,
    raise_nonfinite,
    PackedKeys,
    RetrievalResult,
    alloc_index,
    append_token,
    PageSummaries,
    approx_scores,
    build_page_summaries,
    fier_attend,
    fier_select,
    full_attention,
    gather_attention,
    load_cache_dump,
    quantize,
    quest_page_scores,
    quest_select,
    quest_select_quantized,
    save_cache_dump,
    select_by_page_scores,
    topk_oracle,
)

__all__ = [
    "DecodeLayer", "PackedKeys", "RetrievalResult", "alloc_index", "append_token", "approx_scores",
    "fier_attend", "fier_select", "full_attention", "gather_attention", "load_cache_dump", "quantize",
    "save_cache_dump", "topk_oracle", "PageSummaries", "build_page_summaries", "quest_page_scores",
    "quest_select", "quest_select_quantized", "select_by_page_scores", "LoadRatio", "load_ratio_fier", "raise_nonfinite",
]
