"""ctypes binding of libstrata (include/strata.h, include/strata_baseline.h).

Argument marshalling only: every step of the I/O path runs in libstrata's sm_100a kernels.  The
binding fails loudly if the shared library is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import List

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STRATA_LIB_PATH") or os.path.join(_HERE, "libstrata.so")   # env: A/B builds
INCLUDE_DIR = os.path.join(os.path.dirname(_HERE), "include")

STRATA_OK = 0
STRATA_ERR_INVALID_ARG = -1
STRATA_ERR_ALIGNMENT = -2
STRATA_ERR_INDEX_RANGE = -3
STRATA_ERR_DUPLICATE = -4
STRATA_ERR_CUDA = -5
STRATA_ERR_OOM = -6
STRATA_ERR_UNSUPPORTED = -7
STRATA_ERR_STALE_TICKET = -8
STRATA_ERR_TIMEOUT = -9
STRATA_ERR_IO = -10

STRATA_HOST_HUGEPAGES = 1
STRATA_HOST_WRITECOMBINED = 2
STRATA_VALIDATE = 4
STRATA_HOST_NO_NUMA_BIND = 8
STRATA_HOST_CUDA_ALLOC = 16
STRATA_POOL_SINGLE_KV = 32
STRATA_HOST_HEAD_MAJOR = 64

STRATA_ENGINE_DEFAULT = 0
STRATA_ENGINE_LDG = 1
STRATA_ENGINE_TMA = 2
STRATA_ENGINE_TMA_BULK = 3
STRATA_ENGINE_DMA = 4

STRATA_H2D = 0
STRATA_D2H = 1

ERROR_NAMES = {
    0: "STRATA_OK", -1: "STRATA_ERR_INVALID_ARG", -2: "STRATA_ERR_ALIGNMENT",
    -3: "STRATA_ERR_INDEX_RANGE", -4: "STRATA_ERR_DUPLICATE", -5: "STRATA_ERR_CUDA",
    -6: "STRATA_ERR_OOM", -7: "STRATA_ERR_UNSUPPORTED", -8: "STRATA_ERR_STALE_TICKET",
    -9: "STRATA_ERR_TIMEOUT", -10: "STRATA_ERR_IO",
}


class StrataError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn} -> {ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


class PoolDesc(ctypes.Structure):
    """strata_pool_desc"""
    _fields_ = [
        ("device", ctypes.c_int32), ("num_layers", ctypes.c_int32), ("num_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("elem_bytes", ctypes.c_int32), ("page_size", ctypes.c_int32),
        ("chunk_tokens", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("k_ptrs", ctypes.POINTER(ctypes.c_void_p)), ("v_ptrs", ctypes.POINTER(ctypes.c_void_p)),
        ("page_stride", ctypes.c_int64), ("token_stride", ctypes.c_int64), ("head_stride", ctypes.c_int64),
        ("num_pages", ctypes.c_int64), ("host_base", ctypes.c_void_p), ("num_chunks", ctypes.c_int64),
        ("host_heads", ctypes.c_int32), ("head_begin", ctypes.c_int32),
    ]


class Xfer(ctypes.Structure):
    """strata_xfer"""
    _fields_ = [
        ("num_reqs", ctypes.c_int32), ("layer_begin", ctypes.c_int32), ("layer_end", ctypes.c_int32),
        ("engine", ctypes.c_int32), ("num_ctas", ctypes.c_int32), ("threads", ctypes.c_int32),
        ("num_tokens", ctypes.c_void_p), ("host_chunks", ctypes.c_void_p), ("chunk_start", ctypes.c_void_p),
        ("dev_pages", ctypes.c_void_p), ("page_start", ctypes.c_void_p), ("chunk_offset", ctypes.c_void_p),
        ("page_offset", ctypes.c_void_p), ("host_chunks_len", ctypes.c_int64), ("dev_pages_len", ctypes.c_int64),
        ("host_chunks_host", ctypes.c_void_p), ("layer_group", ctypes.c_int32), ("inflight_kib", ctypes.c_int32),
    ]


class Counters(ctypes.Structure):
    """strata_counters"""
    _fields_ = [("operations", ctypes.c_int64), ("kernel_launches", ctypes.c_int64), ("dma_copies", ctypes.c_int64),
                ("bytes", ctypes.c_int64), ("last_engine", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None

_SIGS = {
    "strata_get_counters": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Counters)]),
    "strata_wait_layer": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p]),
    "strata_set_load_quota": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "strata_layer_elapsed_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32,
                                               ctypes.POINTER(ctypes.c_float)]),
    "strata_register_host_pool": (ctypes.c_int, [ctypes.POINTER(PoolDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "strata_unregister_host_pool": (ctypes.c_int, [ctypes.c_void_p]),
    "strata_host_pool_ptr": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.POINTER(ctypes.c_size_t)]),
    "strata_load": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Xfer), ctypes.c_void_p,
                                   ctypes.POINTER(ctypes.c_uint64)]),
    "strata_offload": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Xfer), ctypes.c_void_p,
                                      ctypes.POINTER(ctypes.c_uint64)]),
    "strata_layer_event": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_void_p)]),
    "strata_last_error": (ctypes.c_char_p, []),
    "strata_version": (ctypes.c_int, []),
    "strata_baseline_memcpy_pages": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Xfer), ctypes.c_int32,
                                                    ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "strata_baseline_contiguous": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                                  ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]),
    "strata_test_ring_geometry": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.POINTER(ctypes.c_int32)]),
}


def lib() -> ctypes.CDLL:
    """Load libstrata.so (built in-tree by __graft_entry__.build()).  Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libstrata.so not built ({LIB_PATH}); run __graft_entry__.build()")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(code: int, fn: str) -> None:
    if code != STRATA_OK:
        raise StrataError(code, fn, lib().strata_last_error().decode(errors="replace"))


def declared_symbols() -> List[str]:
    """Every function declared in include/*.h (for the ABI export test)."""
    names = []
    for h in sorted(os.listdir(INCLUDE_DIR)):
        if h.endswith(".h"):
            text = open(os.path.join(INCLUDE_DIR, h)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
            names += re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(strata_\w+)\s*\(", text, flags=re.M)
    return names
