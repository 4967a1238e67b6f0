"""ctypes binding of the C ABI declared in ``include/mosaic_b200.h``.

There is deliberately no fallback: if ``libmosaic_b200.so`` is missing the
first call raises, so a GPU run can never silently route through a CPU or
PyTorch re-implementation.
"""
from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_uint32, c_uint64, c_void_p
from pathlib import Path

from .errors import raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libmosaic_b200.so"

_i32p = POINTER(c_int32)
_u64p = POINTER(c_uint64)

# name -> (restype, argtypes); mirrors include/mosaic_b200.h one to one.
SIGNATURES: dict[str, tuple[object, list[object]]] = {
    "mosaic_abi_version": (c_int, []),
    "mosaic_last_error": (c_char_p, []),
    "mosaic_first_fit": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, POINTER(c_int64)]),
    "mosaic_l2_persisting_limit": (c_int, [c_int64, POINTER(c_int64)]),
    "mosaic_mask_compact_scratch_bytes": (c_size_t, [c_int64]),
    "mosaic_mask_compact": (c_int, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mosaic_gather_rows": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p],
    ),
    "mosaic_gather_rows_scattered": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_int64, c_int32, c_int32, c_void_p,
         c_void_p],
    ),
    "mosaic_lmhead_plan": (c_int, [c_int64, c_int64, c_int64, _i32p, _i32p]),
    "mosaic_lmhead_stats": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32,
         c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_lmhead_stats_die": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_die_map_scratch_bytes": (c_size_t, [c_int32]),
    "mosaic_die_map": (c_int, [c_void_p, c_int32, c_void_p, POINTER(c_int32), POINTER(c_int32), c_void_p]),
    "mosaic_lmhead_stats_gather": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
         c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_lmhead_stats_gather_die": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
         c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_lmhead_stats_runs": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64,
         c_int64, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_remask_commit_segmented": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p, c_int64, c_void_p,
         c_void_p, c_void_p],
    ),
    "mosaic_window_rows": (
        c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int32, c_void_p, c_void_p],
    ),
    "mosaic_lmhead_sample": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p, c_float,
         c_uint32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_sample_merge": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_lmhead_logits": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p],
    ),
    "mosaic_stats_merge": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_stats_exchange_push": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p,
         c_int32, c_int32, c_uint32, c_void_p, c_void_p],
    ),
    "mosaic_stats_exchange_wait": (c_int, [c_void_p, c_int32, c_uint32, c_void_p]),
    "mosaic_remask_scratch_bytes": (c_size_t, []),
    "mosaic_remask_commit": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p,
         c_void_p, c_void_p],
    ),
    "mosaic_lmhead_logits_gather": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
         c_void_p, c_int64, c_void_p],
    ),
    "mosaic_lmhead_config": (c_int, [c_int64, c_int32, c_void_p]),
    "mosaic_swiglu": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "mosaic_rope_qk": (c_int, [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int64, c_void_p, c_int64, c_void_p]),
    "mosaic_moe_route_scratch_bytes": (c_size_t, [c_int64, c_int32]),
    "mosaic_moe_route": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p],
    ),
    "mosaic_moe_combine": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int32, c_int64, c_void_p, c_int64, c_void_p],
    ),
    "mosaic_ffn_gemm": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int32, c_void_p,
         c_int64, c_void_p],
    ),
    "mosaic_ffn_gemm_ex": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int32, c_void_p,
         c_int64, c_void_p],
    ),
    "mosaic_ffn_gemm_sched": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int32, c_void_p,
         c_int64, c_void_p, c_void_p],
    ),
    "mosaic_arena_reserve": (c_int, [c_int32, c_uint64, POINTER(c_void_p)]),
    "mosaic_arena_commit": (c_int, [c_void_p, c_uint64]),
    "mosaic_arena_info": (c_int, [c_void_p, _u64p, _u64p, _u64p, _u64p]),
    "mosaic_arena_release": (c_int, [c_void_p]),
    "mosaic_pool_bind": (c_int, [c_int32, c_void_p, c_uint64]),
    "mosaic_pool_select": (c_int, [c_int32, c_void_p]),
    "mosaic_pool_unbind": (c_int, [c_int32, c_void_p]),
    "mosaic_pool_alloc": (c_void_p, [ctypes.c_ssize_t, c_int, c_void_p]),
    "mosaic_pool_free": (None, [c_void_p, ctypes.c_ssize_t, c_int, c_void_p]),
    "mosaic_pool_stats": (c_int, [c_int32, c_void_p, _u64p, _u64p, _u64p, _u64p]),
    "mosaic_tag_fill": (c_int, [c_void_p, c_int64, c_uint64, c_void_p]),
    "mosaic_tag_check": (c_int, [c_void_p, c_int64, c_uint64, c_void_p, c_void_p]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load (once) and type the native library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2601_06562_b200._build` "
                    "(there is no CPU fallback for the hot path)"
                )
            lib = ctypes.CDLL(os.fspath(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise the mapped exception."""
    lib = load()
    status = getattr(lib, name)(*args)
    if status != 0:
        msg = lib.mosaic_last_error()
        raise_for_status(int(status), msg.decode() if msg else "", name)


def value(name: str, *args):
    return getattr(load(), name)(*args)
