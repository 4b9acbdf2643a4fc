"""paper_2508_18572_b200 — B200-native GPU-assisted KV-cache I/O (Strata, arXiv 2508.18572).

Thin Python binding over libstrata's C ABI (include/strata.h).  The functions below carry the C
names and only marshal arguments; every byte moves in libstrata's sm_100a kernels.  PyTorch is used
by callers for device memory and streams only.

    strata_register_host_pool / strata_unregister_host_pool / strata_host_pool_ptr
    strata_load / strata_offload            -> ticket
    strata_layer_event / strata_wait_layer / strata_layer_elapsed_ms
    strata_baseline_memcpy_pages / strata_baseline_contiguous

Plus two conveniences: :class:`HostPool` (owns a registered pool, exposes the host tier as a numpy
array) and :class:`Requests` (request tables with device-resident index lists).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (STRATA_D2H, STRATA_ENGINE_DEFAULT, STRATA_ENGINE_LDG, STRATA_ENGINE_TMA,  # noqa: F401
                   STRATA_ENGINE_TMA_BULK, STRATA_ENGINE_DMA,
                   STRATA_H2D, STRATA_HOST_HUGEPAGES, STRATA_HOST_NO_NUMA_BIND, STRATA_POOL_SINGLE_KV,
                   STRATA_HOST_HEAD_MAJOR,
                   STRATA_HOST_WRITECOMBINED, STRATA_VALIDATE, STRATA_ERR_UNSUPPORTED, PoolDesc, StrataError,
                   Xfer, check)

__all__ = [
    "strata_register_host_pool", "strata_unregister_host_pool", "strata_host_pool_ptr", "strata_load",
    "strata_offload", "strata_layer_event", "strata_wait_layer", "strata_layer_elapsed_ms", "strata_set_load_quota",
    "strata_baseline_memcpy_pages", "strata_baseline_contiguous", "strata_test_ring_geometry",
    "strata_version", "strata_get_counters", "HostPool", "Requests", "StrataError",
]


def _stream_handle(stream) -> int:
    """Raw cudaStream_t from a torch.cuda.Stream, an int, or None (torch's current stream)."""
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


# ------------------------------------------------------------------------------------------------
# C-named entry points (argument marshalling only)
def strata_version() -> int:
    return int(_lib.lib().strata_version())


def strata_register_host_pool(desc: PoolDesc) -> int:
    h = ctypes.c_void_p()
    check(_lib.lib().strata_register_host_pool(ctypes.byref(desc), ctypes.byref(h)), "strata_register_host_pool")
    return int(h.value)


def strata_unregister_host_pool(pool: int) -> None:
    check(_lib.lib().strata_unregister_host_pool(ctypes.c_void_p(pool)), "strata_unregister_host_pool")


def strata_host_pool_ptr(pool: int):
    a, n = ctypes.c_void_p(), ctypes.c_size_t()
    check(_lib.lib().strata_host_pool_ptr(ctypes.c_void_p(pool), ctypes.byref(a), ctypes.byref(n)),
          "strata_host_pool_ptr")
    return int(a.value or 0), int(n.value)


def strata_load(pool: int, xfer: Xfer, stream=None) -> int:
    t = ctypes.c_uint64()
    check(_lib.lib().strata_load(ctypes.c_void_p(pool), ctypes.byref(xfer), ctypes.c_void_p(_stream_handle(stream)),
                                 ctypes.byref(t)), "strata_load")
    return int(t.value)


def strata_offload(pool: int, xfer: Xfer, stream=None) -> int:
    t = ctypes.c_uint64()
    check(_lib.lib().strata_offload(ctypes.c_void_p(pool), ctypes.byref(xfer),
                                    ctypes.c_void_p(_stream_handle(stream)), ctypes.byref(t)), "strata_offload")
    return int(t.value)


def strata_layer_event(pool: int, ticket: int, layer: int) -> int:
    ev = ctypes.c_void_p()
    check(_lib.lib().strata_layer_event(ctypes.c_void_p(pool), ticket, layer, ctypes.byref(ev)),
          "strata_layer_event")
    return int(ev.value)


def strata_set_load_quota(pool: int, max_ctas: int, stream=None) -> None:
    check(_lib.lib().strata_set_load_quota(ctypes.c_void_p(pool), max_ctas, ctypes.c_void_p(_stream_handle(stream))),
          "strata_set_load_quota")


def strata_wait_layer(pool: int, ticket: int, layer: int, consumer=None) -> None:
    check(_lib.lib().strata_wait_layer(ctypes.c_void_p(pool), ticket, layer,
                                       ctypes.c_void_p(_stream_handle(consumer))), "strata_wait_layer")


def strata_layer_elapsed_ms(pool: int, ticket: int, layer: int) -> float:
    ms = ctypes.c_float()
    check(_lib.lib().strata_layer_elapsed_ms(ctypes.c_void_p(pool), ticket, layer, ctypes.byref(ms)),
          "strata_layer_elapsed_ms")
    return float(ms.value)


def strata_get_counters(pool: int) -> dict:
    c = _lib.Counters()
    check(_lib.lib().strata_get_counters(ctypes.c_void_p(pool), ctypes.byref(c)), "strata_get_counters")
    return {f: int(getattr(c, f)) for f, _ in c._fields_ if f != "reserved"}


def strata_baseline_memcpy_pages(pool: int, xfer: Xfer, direction: int, stream=None) -> int:
    n = ctypes.c_int64()
    check(_lib.lib().strata_baseline_memcpy_pages(ctypes.c_void_p(pool), ctypes.byref(xfer), direction,
                                                  ctypes.c_void_p(_stream_handle(stream)), ctypes.byref(n)),
          "strata_baseline_memcpy_pages")
    return int(n.value)


def strata_test_ring_geometry(tok_bytes: int, chunk_tokens: int, gran: int, smem_budget: int, inflight_bytes: int,
                              ctas: int, warps: int, stage_target: int):
    """The ring engine's per-CTA geometry (include/strata_test.h): (rows per piece, stages, warps,
    stage bytes), or None when no 2-stage ring fits."""
    out = (ctypes.c_int32 * 4)()
    rc = _lib.lib().strata_test_ring_geometry(tok_bytes, chunk_tokens, gran, smem_budget, inflight_bytes, ctas, warps,
                                              stage_target, out)
    if rc == STRATA_ERR_UNSUPPORTED:
        return None
    check(rc, "strata_test_ring_geometry")
    return tuple(out)


def strata_baseline_contiguous(pool: int, direction: int, dev_ptr: int, host_offset: int, nbytes: int,
                               stream=None) -> None:
    check(_lib.lib().strata_baseline_contiguous(ctypes.c_void_p(pool), direction, ctypes.c_void_p(dev_ptr),
                                                host_offset, nbytes, ctypes.c_void_p(_stream_handle(stream))),
          "strata_baseline_contiguous")


# ------------------------------------------------------------------------------------------------
class Requests:
    """Request tables for one strata_xfer: host numpy metadata + device int32 index lists.

    ``host_chunks`` / ``dev_pages`` are uploaded to ``device`` once (torch int32 tensors) and must
    stay alive while an operation using them is in flight.  ``host_lists=True`` keeps host copies
    for the copy-engine baselines.
    """

    def __init__(self, num_tokens, host_chunks, chunk_start, dev_pages, page_start, chunk_offset=None,
                 page_offset=None, device: int = 0):
        import torch
        self.num_tokens = np.ascontiguousarray(num_tokens, np.int64)
        self.chunk_start = np.ascontiguousarray(chunk_start, np.int64)
        self.page_start = np.ascontiguousarray(page_start, np.int64)
        R = self.num_tokens.shape[0]
        self.chunk_offset = np.ascontiguousarray(np.zeros(R) if chunk_offset is None else chunk_offset, np.int32)
        self.page_offset = np.ascontiguousarray(np.zeros(R) if page_offset is None else page_offset, np.int32)
        self.host_chunks_h = np.ascontiguousarray(host_chunks, np.int32)
        self.dev_pages_h = np.ascontiguousarray(dev_pages, np.int32)
        dev = torch.device("cuda", device)
        self.host_chunks_d = torch.from_numpy(self.host_chunks_h.copy()).to(dev)
        self.dev_pages_d = torch.from_numpy(self.dev_pages_h.copy()).to(dev)
        self._xcache = {}

    @classmethod
    def from_kvgen(cls, q, device: int = 0) -> "Requests":
        return cls(q.num_tokens, q.host_chunks, q.chunk_start, q.dev_pages, q.page_start, q.chunk_offset,
                   q.page_offset, device=device)

    @property
    def R(self) -> int:
        return int(self.num_tokens.shape[0])

    @property
    def total_tokens(self) -> int:
        return int(self.num_tokens.sum())

    def xfer(self, layer_begin: int, layer_end: int, engine: int = 0, num_ctas: int = 0, threads: int = 0,
             host_lists: bool = False, layer_group: int = 0, inflight_kib: int = 0) -> Xfer:
        """strata_xfer pointing at these tables (device lists, or host lists for the baselines)."""
        hc = self.host_chunks_h.ctypes.data if host_lists else self.host_chunks_d.data_ptr()
        dp = self.dev_pages_h.ctypes.data if host_lists else self.dev_pages_d.data_ptr()
        return Xfer(num_reqs=self.R, layer_begin=layer_begin, layer_end=layer_end, engine=engine,
                    num_ctas=num_ctas, threads=threads, num_tokens=self.num_tokens.ctypes.data,
                    host_chunks=hc, chunk_start=self.chunk_start.ctypes.data, dev_pages=dp,
                    page_start=self.page_start.ctypes.data, chunk_offset=self.chunk_offset.ctypes.data,
                    page_offset=self.page_offset.ctypes.data, host_chunks_len=self.host_chunks_h.size,
                    dev_pages_len=self.dev_pages_h.size, host_chunks_host=self.host_chunks_h.ctypes.data,
                    layer_group=layer_group, inflight_kib=inflight_kib)


class HostPool:
    """A registered host tier bound to a paged device pool (one K and one V buffer per layer).

    k_ptrs / v_ptrs: device addresses (ints) or tensors (their data_ptr() is used).  The device
    buffers stay owned by the caller.  ``host``: optional caller array to register, else the
    library allocates the tier.  ``.host`` is a numpy uint8 view of the tier either way.
    """

    def __init__(self, *, num_layers: int, num_heads: int, head_dim: int, elem_bytes: int, page_size: int,
                 chunk_tokens: int, k_ptrs: Sequence, v_ptrs: Optional[Sequence], num_pages: int, num_chunks: int,
                 device: int = 0, flags: int = 0, host: Optional[np.ndarray] = None,
                 strides=(0, 0, 0), host_heads: int = 0, head_begin: int = 0, head_major: bool = False):
        def ptr(x):
            return int(x) if isinstance(x, int) else int(x.data_ptr())
        if head_major:
            flags |= STRATA_HOST_HEAD_MAJOR
        # v_ptrs=None: one buffer per layer (MLA latent cache, STRATA_POOL_SINGLE_KV)
        if v_ptrs is None:
            flags |= STRATA_POOL_SINGLE_KV
            v_ptrs = k_ptrs
        self._k = (ctypes.c_void_p * num_layers)(*[ptr(x) for x in k_ptrs])
        self._v = (ctypes.c_void_p * num_layers)(*[ptr(x) for x in v_ptrs])
        self._host_owner = host
        desc = PoolDesc(device=device, num_layers=num_layers, num_heads=num_heads, head_dim=head_dim,
                        elem_bytes=elem_bytes, page_size=page_size, chunk_tokens=chunk_tokens, flags=flags,
                        k_ptrs=ctypes.cast(self._k, ctypes.POINTER(ctypes.c_void_p)),
                        v_ptrs=ctypes.cast(self._v, ctypes.POINTER(ctypes.c_void_p)),
                        page_stride=strides[0], token_stride=strides[1], head_stride=strides[2],
                        num_pages=num_pages, host_base=(host.ctypes.data if host is not None else None),
                        num_chunks=num_chunks, host_heads=host_heads, head_begin=head_begin)
        self.handle = strata_register_host_pool(desc)
        self._hptr = ctypes.c_void_p(self.handle)
        self._ticket = ctypes.c_uint64()
        addr, nbytes = strata_host_pool_ptr(self.handle)
        self.nbytes = nbytes
        buf = (ctypes.c_uint8 * nbytes).from_address(addr)
        self.host = np.frombuffer(buf, dtype=np.uint8, count=nbytes)
        self.host_addr = addr
        self.num_layers = num_layers

    def close(self) -> None:
        if getattr(self, "handle", None):
            strata_unregister_host_pool(self.handle)
            self.handle = None
            self.host = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _op(self, fn, name: str, reqs: Requests, layer_begin: int, layer_end: Optional[int], stream, engine: int,
            num_ctas: int, threads: int, layer_group: int, inflight_kib: int = 0) -> int:
        # The strata_xfer of a (Requests, layer range, options) tuple is built once and reused: its
        # pointers are those of the Requests' arrays, which stay put, while the C call re-reads the
        # values behind them (num_tokens, offsets) every time.  Saves ~15 us of ctypes marshalling
        # per call, which is most of a small load's host cost.
        key = (layer_begin, self.num_layers if layer_end is None else layer_end, engine, num_ctas, threads,
               layer_group, inflight_kib)
        x = reqs._xcache.get(key)
        if x is None:
            x = reqs._xcache[key] = reqs.xfer(key[0], key[1], engine, num_ctas, threads, layer_group=layer_group,
                                              inflight_kib=inflight_kib)
        check(fn(self._hptr, ctypes.byref(x), ctypes.c_void_p(_stream_handle(stream)), self._ticket), name)
        if stream is not None and hasattr(stream, "cuda_stream"):
            # the kernels read the device index lists on `stream`: keep torch's caching allocator
            # from handing their memory out again before that stream passes this operation
            reqs.host_chunks_d.record_stream(stream)
            reqs.dev_pages_d.record_stream(stream)
        return self._ticket.value

    def load(self, reqs: Requests, layer_begin: int = 0, layer_end: Optional[int] = None, stream=None,
             engine: int = 0, num_ctas: int = 0, threads: int = 0, layer_group: int = 0, inflight_kib: int = 0) -> int:
        return self._op(_lib.lib().strata_load, "strata_load", reqs, layer_begin, layer_end, stream, engine,
                        num_ctas, threads, layer_group, inflight_kib)

    def offload(self, reqs: Requests, layer_begin: int = 0, layer_end: Optional[int] = None, stream=None,
                engine: int = 0, num_ctas: int = 0, threads: int = 0, layer_group: int = 0,
                inflight_kib: int = 0) -> int:
        return self._op(_lib.lib().strata_offload, "strata_offload", reqs, layer_begin, layer_end, stream, engine,
                        num_ctas, threads, layer_group, inflight_kib)

    def layer_event(self, ticket: int, layer: int) -> int:
        return strata_layer_event(self.handle, ticket, layer)

    def set_load_quota(self, max_ctas: int, stream=None) -> None:
        strata_set_load_quota(self.handle, max_ctas, stream)

    def wait_layer(self, ticket: int, layer: int, consumer=None) -> None:
        strata_wait_layer(self.handle, ticket, layer, consumer)

    def layer_elapsed_ms(self, ticket: int, layer: int) -> float:
        return strata_layer_elapsed_ms(self.handle, ticket, layer)

    def counters(self) -> dict:
        return strata_get_counters(self.handle)
