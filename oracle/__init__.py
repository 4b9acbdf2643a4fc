"""CPU oracle for the Strata KV-cache I/O path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product (``paper_2508_18572_b200``) never
imports it, and it imports nothing from the product.

Two independent implementations of the same plain definition:
  * ``oracle.c`` (built to ``liboracle.so`` by :func:`build`): plain nested loops, one memcpy of D*e
    bytes per (token, layer, kv, head), own index math.  Wrapped by :func:`load` / :func:`offload`.
  * ``oracle_np`` : numpy fancy indexing on reshaped views (tiny pools only).

Both are pinned by tests/test_oracle.py against closed forms, brute force, round-trip identity,
tagged-coordinate decoding, conservation and the TP-union invariant.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

from . import oracle_np  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib: Optional[ctypes.CDLL] = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-fopenmp for the timing build)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-Wall", "-o", _SO, src])
    return _SO


class _Geom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("L", "H", "D", "e", "P", "C", "page_stride", "token_stride", "head_stride",
                 "num_pages", "num_chunks", "KV", "Ht", "h0", "head_major")]


class _Reqs(ctypes.Structure):
    _fields_ = [("R", ctypes.c_int64),
                ("num_tokens", ctypes.c_void_p), ("host_chunks", ctypes.c_void_p),
                ("chunk_start", ctypes.c_void_p), ("dev_pages", ctypes.c_void_p),
                ("page_start", ctypes.c_void_p), ("chunk_offset", ctypes.c_void_p),
                ("page_offset", ctypes.c_void_p),
                ("layer_begin", ctypes.c_int64), ("layer_end", ctypes.c_int64)]


def _get() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        for fn in (_lib.oracle_load, _lib.oracle_offload):
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.POINTER(_Geom), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.POINTER(_Reqs), ctypes.c_int]
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def max_threads() -> int:
    return int(_get().oracle_max_threads())


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _prep(g, host, k_imgs, v_imgs, q, l0, l1, strides):
    tok = g.H * g.D * g.e
    ps, ts, hs = strides or (g.P * tok, tok, g.D * g.e)
    geom = _Geom(g.L, g.H, g.D, g.e, g.P, g.C, ps, ts, hs, g.num_pages, g.num_chunks, getattr(g, "kv", 2),
                 getattr(g, "Ht", 0) or g.H, getattr(g, "h0", 0), int(getattr(g, "head_major", False)))
    keep = [np.ascontiguousarray(q.num_tokens, np.int64), np.ascontiguousarray(q.host_chunks, np.int32),
            np.ascontiguousarray(q.chunk_start, np.int64), np.ascontiguousarray(q.dev_pages, np.int32),
            np.ascontiguousarray(q.page_start, np.int64), np.ascontiguousarray(q.chunk_offset, np.int32),
            np.ascontiguousarray(q.page_offset, np.int32)]
    # a zero-length list still needs a valid pointer
    keep = [k if k.size else np.zeros(1, k.dtype) for k in keep]
    reqs = _Reqs(q.R, *[_ptr(k) for k in keep], l0, l1)
    kp = (ctypes.c_void_p * g.L)(*[_ptr(a) if a is not None else 0 for a in k_imgs])
    vp = (ctypes.c_void_p * g.L)(*[_ptr(a) if a is not None else 0 for a in v_imgs])
    return geom, reqs, kp, vp, keep


def load(g, host: np.ndarray, k_imgs: Sequence[np.ndarray], v_imgs: Sequence[np.ndarray], q,
         layer_begin: int, layer_end: int, strides=None, nthreads: int = 1) -> None:
    """C oracle LOAD into host images of the device pool (k_imgs[l], v_imgs[l]: uint8 arrays).
    Layers outside [layer_begin, layer_end) may be None."""
    geom, reqs, kp, vp, keep = _prep(g, host, k_imgs, v_imgs, q, layer_begin, layer_end, strides)
    rc = _get().oracle_load(ctypes.byref(geom), _ptr(host), kp, vp, ctypes.byref(reqs), nthreads)
    if rc != 0:
        raise IndexError("oracle_load: index out of range")


def offload(g, host: np.ndarray, k_imgs: Sequence[np.ndarray], v_imgs: Sequence[np.ndarray], q,
            layer_begin: int, layer_end: int, strides=None, nthreads: int = 1) -> None:
    """C oracle OFFLOAD from the device images into the host pool image ``host``."""
    geom, reqs, kp, vp, keep = _prep(g, host, k_imgs, v_imgs, q, layer_begin, layer_end, strides)
    rc = _get().oracle_offload(ctypes.byref(geom), _ptr(host), kp, vp, ctypes.byref(reqs), nthreads)
    if rc != 0:
        raise IndexError("oracle_offload: index out of range")
