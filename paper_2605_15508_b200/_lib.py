"""ctypes binding of libsts_b200.so (the C-ABI in include/sts_b200.h).

There is no fallback: if the library is missing or does not load, importing a
compute entry point raises immediately.  ``load()`` is idempotent.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import raise_for_status

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["STS_B200_LIB"]) if os.environ.get("STS_B200_LIB") else _PKG / "_lib" / "libsts_b200.so"
HEADER = _PKG.parent / "include" / "sts_b200.h"

STS_DTYPE_F32 = 0
STS_DTYPE_BF16 = 1
STS_SEL_CURRENT = 0x1
STS_SEL_SINK = 0x2
STS_DEV_IDX_CAPACITY = 0x1
STS_DEV_EMPTY_ROW = 0x2
STS_DEV_BAD_INDEX = 0x4
STS_DEV_SELECT_INCONSISTENT = 0x8
STS_BLOCK_INCLUDE_SELF = 0x1
ABI_VERSION = 8

_i32, _i64, _u32, _f32, _f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_float, C.c_double
_p, _sz = C.c_void_p, C.c_size_t

# symbol -> (restype, argtypes); must list every function the header declares
SIGNATURES = {
    "sts_last_error": (C.c_char_p, []),
    "sts_abi_version": (C.c_int, []),
    "sts_launch_count": (C.c_ulonglong, []),
    "sts_select_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "sts_select_topk": (C.c_int, [_p, _i64, _p, _i32, _i64, _p, _i32, _f64, _i32, _i32, _u32, _i32,
                                  _i32, _p, _i64, _p, _p, _p, _sz, _p]),
    "sts_page_aggregate": (C.c_int, [_p, _i64, _i64, _p, _i32, _i32, _p, _i64, _p]),
    "sts_sparse_decode_workspace_bytes": (_sz, [_i64, _i32, _i32, _i32]),
    "sts_auto_splits": (_i32, [_i64, _i64]),
    "sts_sparse_decode_schedule": (_i32, [_i64, _i32, _i32, _i64, _i32]),
    "sts_sparse_decode": (C.c_int, [_i32, _i32, _p, _p, _p, _i64, _i64, _i64, _i32, _i32, _p, _i64, _p, _i32, _p,
                                    _i32, _i32, _i32, _f32, _p, _p, _i32, _p, _p, _sz, _p]),
    "sts_sparse_prefill": (C.c_int, [_i32, _i32, _p, _p, _p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _i64, _p,
                                     _f32, _p, _p, _p, _p, _sz, _p]),
    "sts_draft_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "sts_draft_lse": (C.c_int, [_i32, _p, _p, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _f32,
                                _p, _p, _sz, _p]),
    "sts_draft_probs": (C.c_int, [_i32, _p, _p, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _f32,
                                  _p, _i32, _p, _i64, _p]),
    "sts_kv_prefetch_l2": (C.c_int, [_p, _p, _i64, _i64, _i64, _i32, _i32, _p, _i64, _p, _i32, _i32, _p]),
    "sts_draft_scores": (C.c_int, [_i32, _p, _p, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _f32,
                                   _p, _i64, _p]),
    "sts_lse_merge": (C.c_int, [_p, _p, _i32, _i64, _i32, _i32, _p, _p, _p]),
    "sts_lse_merge_ptrs": (C.c_int, [_p, _i32, _i64, _i32, _i64, _i64, _i32, _p, _p, _p]),
    "sts_row_union": (C.c_int, [_p, _i64, _p, _p, _i64, _i32, _i32, _p, _p, _p, _i64, _p, _p, _p]),
    "sts_topk_bitsets": (C.c_int, [_p, _i64, _p, _i64, _i32, _p, _p]),
    "sts_bitset_overlap": (C.c_int, [_p, _i32, _p, _i32, _i64, _p, _p]),
    "sts_block_attention_f64": (C.c_int, [_p, _p, _p, _i64, _i64, _i32, _i32, _i32, _i32, _f64, _p, _i64, _p, _p,
                                          _i32, _p, _i64, _p, _p, _i64, _p, _p]),
    "sts_page_plan": (C.c_int, [_p, _i64, _p, _i64, _i32, _i32, _i32, _p, _i64, _p, _p, _p, _p]),
    "sts_page_copy": (C.c_int, [_p, _p, _i64, _i64, _i32, _p, _p, _i64, _i32, _i32, _p, _i64, _p, _p, _i64, _i64,
                                _i32, _i32, _i32, _i32, _p]),
    "sts_page_cache_plan": (C.c_int, [_p, _i64, _p, _i64, _i32, _i32, _i32, _p, _p, _i64, _i32, _i32, _p, _p, _p, _p,
                                      _p, _p]),
    "sts_prefill_blocksparse": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _i32, _i64, _i64, _i64, _f32, _p, _i64, _p,
                                          _p, _p, _p]),
    "sts_dist_select_rounds": (_i32, [_i32]),
    "sts_dist_select_bins": (_i32, []),
    "sts_dist_select_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "sts_dist_select_begin": (C.c_int, [_p, _p, _p, _sz, _p]),
    "sts_dist_select_round": (C.c_int, [_p, _i32, _p, _p, _p, _p, _sz, _p]),
    "sts_dist_select_finish": (C.c_int, [_p, _i32, _i32, _p, _u32, _i32, _i32, _i32, _p, _i64, _p, _p, _p, _sz,
                                         _p]),
}

STS_DIST_BINS = 2048


class DistRows(C.Structure):
    """struct sts_dist_rows (include/sts_b200.h)."""

    _fields_ = [
        ("scores_dev", _p),
        ("ld", _i64),
        ("row_src_dev", _p),
        ("nsrc", _i32),
        ("rows", _i64),
        ("n_global", _i32),
        ("lo", _i32),
        ("n_local", _i32),
        ("k_top", _i32),
        ("page_size", _i32),
    ]

_LIB = None


def load(build_if_missing: bool = False):
    """Load (optionally building) the native library; raise if unavailable."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        if build_if_missing or os.environ.get("STS_B200_BUILD") == "1":
            from .build import build

            build()
        else:
            raise ImportError(
                f"libsts_b200.so not found at {LIB_PATH}; run `python -m paper_2605_15508_b200.build` "
                "(there is no CPU fallback)"
            )
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    # a stale build would run a different protocol from this binding: refuse it
    if lib.sts_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI {lib.sts_abi_version()} != {ABI_VERSION}; rebuild "
                          "(python -m paper_2605_15508_b200.build)")
    if lib.sts_dist_select_bins() != STS_DIST_BINS:
        raise ImportError(f"{LIB_PATH}: sharded select uses {lib.sts_dist_select_bins()} bins, binding expects "
                          f"{STS_DIST_BINS}; rebuild")
    _LIB = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise the mapped exception."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.sts_last_error()
        raise_for_status(rc, msg.decode() if msg else "")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
