"""Binding of the disk tier (include/strata_disk.h): argument marshalling only.

    strata_disk_open / strata_disk_close / strata_disk_prefetch / strata_disk_writeback /
    strata_disk_cancel / strata_disk_wait
plus :class:`DiskTier`.  No CUDA is involved: prefetches land in a host tier (``HostPool.host`` or
any 4096-byte aligned numpy buffer of whole chunks).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import check

STRATA_DISK_PAGE_FIRST = 0
STRATA_DISK_LAYER_FIRST = 1
STRATA_DISK_O_DIRECT = 1
STRATA_DISK_CREATE = 2
STRATA_DISK_PENDING, STRATA_DISK_DONE, STRATA_DISK_CANCELLED, STRATA_DISK_FAILED = 0, 1, 2, 3


class DiskDesc(ctypes.Structure):
    """strata_disk_desc"""
    _fields_ = [("path", ctypes.c_char_p), ("chunk_bytes", ctypes.c_int64), ("num_layers", ctypes.c_int32),
                ("layout", ctypes.c_int32), ("num_chunks", ctypes.c_int64), ("flags", ctypes.c_int32),
                ("io_threads", ctypes.c_int32)]


_bound = False


def _l():
    global _bound
    lib = _lib.lib()
    if not _bound:
        vp, i32p, i64, u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)
        sigs = {
            "strata_disk_open": [ctypes.POINTER(DiskDesc), ctypes.POINTER(vp)],
            "strata_disk_close": [vp],
            "strata_disk_prefetch": [vp, vp, vp, vp, i64, u64p],
            "strata_disk_writeback": [vp, vp, vp, vp, i64, u64p],
            "strata_disk_cancel": [vp, ctypes.c_uint64],
            "strata_disk_wait": [vp, ctypes.c_uint64, i64, ctypes.POINTER(i64), i32p],
        }
        for name, args in sigs.items():
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = args
        _bound = True
    return lib


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def strata_disk_open(desc: DiskDesc) -> int:
    h = ctypes.c_void_p()
    check(_l().strata_disk_open(ctypes.byref(desc), ctypes.byref(h)), "strata_disk_open")
    return int(h.value)


def strata_disk_close(disk: int) -> None:
    check(_l().strata_disk_close(ctypes.c_void_p(disk)), "strata_disk_close")


def strata_disk_prefetch(disk: int, host_base: int, disk_chunks, host_chunks) -> int:
    dc, hc = _i32(disk_chunks), _i32(host_chunks)
    job = ctypes.c_uint64()
    check(_l().strata_disk_prefetch(ctypes.c_void_p(disk), ctypes.c_void_p(host_base), dc.ctypes.data, hc.ctypes.data,
                                    dc.size, ctypes.byref(job)), "strata_disk_prefetch")
    return int(job.value)


def strata_disk_writeback(disk: int, host_base: int, host_chunks, disk_chunks) -> int:
    hc, dc = _i32(host_chunks), _i32(disk_chunks)
    job = ctypes.c_uint64()
    check(_l().strata_disk_writeback(ctypes.c_void_p(disk), ctypes.c_void_p(host_base), hc.ctypes.data, dc.ctypes.data,
                                     dc.size, ctypes.byref(job)), "strata_disk_writeback")
    return int(job.value)


def strata_disk_cancel(disk: int, job: int) -> None:
    check(_l().strata_disk_cancel(ctypes.c_void_p(disk), job), "strata_disk_cancel")


def strata_disk_wait(disk: int, job: int, n: int, timeout_ms: int = -1) -> Tuple[int, int, np.ndarray]:
    """Returns (status code, chunks done, per-chunk status array); does not raise on TIMEOUT / IO."""
    nd = ctypes.c_int64()
    st = np.zeros(max(n, 1), np.int32)
    rc = _l().strata_disk_wait(ctypes.c_void_p(disk), job, timeout_ms, ctypes.byref(nd),
                               st.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    if rc not in (_lib.STRATA_OK, _lib.STRATA_ERR_TIMEOUT, _lib.STRATA_ERR_IO):
        check(rc, "strata_disk_wait")
    return rc, int(nd.value), st[:n]


class DiskTier:
    """A disk tier file bound to a host-tier geometry (chunk_bytes, L)."""

    def __init__(self, path: str, chunk_bytes: int, num_layers: int, num_chunks: int,
                 layout: int = STRATA_DISK_PAGE_FIRST, o_direct: bool = False, create: bool = True,
                 io_threads: int = 0):
        self.path = path.encode()
        flags = (STRATA_DISK_O_DIRECT if o_direct else 0) | (STRATA_DISK_CREATE if create else 0)
        self.desc = DiskDesc(path=self.path, chunk_bytes=chunk_bytes, num_layers=num_layers, layout=layout,
                             num_chunks=num_chunks, flags=flags, io_threads=io_threads)
        self.handle = strata_disk_open(self.desc)
        self._pending = {}

    def prefetch(self, host: np.ndarray, disk_chunks: Sequence[int], host_chunks: Sequence[int]) -> int:
        job = strata_disk_prefetch(self.handle, host.ctypes.data, disk_chunks, host_chunks)
        self._pending[job] = (host, len(disk_chunks))
        return job

    def writeback(self, host: np.ndarray, host_chunks: Sequence[int], disk_chunks: Sequence[int]) -> int:
        job = strata_disk_writeback(self.handle, host.ctypes.data, host_chunks, disk_chunks)
        self._pending[job] = (host, len(disk_chunks))
        return job

    def cancel(self, job: int) -> None:
        strata_disk_cancel(self.handle, job)

    def wait(self, job: int, timeout_ms: int = -1):
        n = self._pending[job][1]
        rc, done, st = strata_disk_wait(self.handle, job, n, timeout_ms)
        if rc != _lib.STRATA_ERR_TIMEOUT:
            self._pending.pop(job, None)
        return rc, done, st

    def close(self) -> None:
        if getattr(self, "handle", None):
            strata_disk_close(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def aligned_empty(nbytes: int, align: int = 4096) -> np.ndarray:
    """A uint8 buffer whose data pointer is `align`-byte aligned (for O_DIRECT)."""
    raw = np.empty(nbytes + align, np.uint8)
    off = (-raw.ctypes.data) % align
    return raw[off: off + nbytes]
