"""ctypes binding of libepk.so (include/epk/epk.h).

There is no fallback: if the CUDA library is missing or no sm_100 GPU is
present, every entry point raises.  Importing this module does not need a GPU
(the CPU test suite checks that the library loads and exports every symbol).
"""
from __future__ import annotations

import ctypes as C
import os
import re

from .errors import raise_for_status

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "libepk.so")
HEADER = os.path.join(ROOT, "include", "epk", "epk.h")

EPK_OK = 0
EPK_F32, EPK_BF16, EPK_F64 = 0, 1, 2
EPK_AGG_AVG, EPK_AGG_MAX = 0, 1
EPK_SCORE_EXACT_F32, EPK_SCORE_TC_BF16 = 0, 1

i32, i64, u64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p


class CacheDesc(C.Structure):
    _fields_ = [
        ("layers", i32),
        ("kv_heads", i32),
        ("head_dim", i32),
        ("dtype", i32),
        ("k", vp),
        ("v", vp),
        ("pos", vp),
        ("head_off", vp),
        ("head_len", vp),
        ("layer_base", vp),
    ]


_SIGS = {
    "epk_ctx_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    "epk_ctx_destroy": (C.c_int, [vp]),
    "epk_ctx_set_stream": (C.c_int, [vp, vp]),
    "epk_ctx_reserve": (C.c_int, [vp, i64]),
    "epk_ctx_synchronize": (C.c_int, [vp]),
    "epk_ctx_poll_error": (C.c_int, [vp]),
    "epk_last_error": (C.c_char_p, []),
    "epk_status_string": (C.c_char_p, [C.c_int]),
    "epk_version": (C.c_int, []),
    "epk_ctx_launch_count": (i64, [vp]),
    "epk_ctx_profile": (C.c_int, [vp, i32]),
    "epk_ctx_set_option": (C.c_int, [vp, i32, i64]),
    "epk_ctx_profile_read": (i64, [vp, i64, C.c_char_p, C.POINTER(C.c_float)]),
    "epk_ctx_profile_timeline": (C.c_int, [vp, i64, C.c_char_p, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                           C.POINTER(C.c_int32)]),
    "epk_score": (C.c_int, [vp, C.POINTER(CacheDesc), vp, vp, i32, i32, i32, i32, i64, vp]),
    "epk_score_grids": (C.c_int, [vp, i32, i32, i32, vp, vp, i32, vp]),
    "epk_select_pooled": (C.c_int, [vp, C.POINTER(CacheDesc), vp, i32, vp, vp, i32, vp, vp, i32]),
    "epk_select_per_head": (C.c_int, [vp, C.POINTER(CacheDesc), vp, i32, vp, vp]),
    "epk_compact": (C.c_int, [vp, C.POINTER(CacheDesc), C.POINTER(CacheDesc), vp, i32]),
    "epk_append": (C.c_int, [vp, C.POINTER(CacheDesc), vp, vp, vp, i32, i32]),
    "epk_evict_step": (C.c_int, [vp, C.POINTER(CacheDesc), C.POINTER(CacheDesc), vp, vp, i32, i32, vp, vp, i32,
                                 i32, i32, i64, i32, vp, vp]),
    "epk_kmeans_assign": (C.c_int, [vp, vp, i64, i64, vp, i64, vp, vp]),
    "epk_kmeans_partial_sums": (C.c_int, [vp, vp, i64, i64, vp, i64, vp, vp, i32]),
    "epk_kmeans_finalize": (C.c_int, [vp, vp, vp, i64, i64, vp]),
    "epk_kmeans_sq_dist": (C.c_int, [vp, vp, i64, i64, vp, vp, vp]),
    "epk_kmeans": (C.c_int, [vp, vp, i64, i64, i64, u64, i64, vp, vp, vp, vp]),
    "epk_pool_scores": (C.c_int, [vp, C.POINTER(CacheDesc), vp, vp, i32]),
    "epk_epkv_scan": (C.c_int, [vp, i64, vp, vp, vp]),
    "epk_load_epkv": (C.c_int, [vp, vp, i64, vp, C.POINTER(CacheDesc)]),
    "epk_kmeans_sharded": (C.c_int, [vp, i32, vp, vp, i64, i64, u64, i64, vp, vp, vp, vp]),
    "epk_key_cosine_sigma": (C.c_int, [vp, vp, vp, i32, i32, i32, i64, i32, vp, vp]),
    "epk_score_keydiff": (C.c_int, [vp, vp, vp]),
    "epk_serialize_epkv": (C.c_int, [vp, vp, C.c_uint64, C.c_char_p, C.c_uint64, vp, i32, vp, i64, vp, vp]),
    "epk_debug_expf": (C.c_int, [vp, vp, vp, i64]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function declared in include/epk/epk.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(epk_[a-z_0-9]+)\s*\(", text, re.M)))


def load(build_if_missing: bool = True):
    """Loads libepk.so, building it with nvcc first if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise RuntimeError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        from ._build import build
        build()
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != EPK_OK:
        msg = load().epk_last_error()
        raise_for_status(rc, msg.decode() if msg else "")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
