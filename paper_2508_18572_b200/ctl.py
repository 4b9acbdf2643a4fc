"""Binding of the control plane (include/strata_ctl.h): argument marshalling only.

    strata_ctl_create / _destroy / _insert / _match / _submit / _schedule / _ids / _plan_get /
    _req_slots / _complete / _abort / _get_stats / _dump / strata_ctl_bubble_steps

:class:`Ctl` owns one handle.  Every decision (HiRadixTree, deferral, Algorithm 1, allocation,
eviction, plans) is made in libstrata's C++; this module only converts arrays.
:meth:`Ctl.xfer` turns a plan into the :class:`paper_2508_18572_b200.Requests` that drive
``strata_load`` / ``strata_offload``.
"""
from __future__ import annotations

import ctypes
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check

STRATA_CTL_NO_DEFER, STRATA_CTL_NO_BALANCE, STRATA_CTL_NO_BUNDLE = 1, 2, 4
DEVICE, HOST = 0, 1
BATCH, DEFERRED, FORMED, QUEUE = 0, 1, 2, 3
LOAD, WRITEBACK = 0, 1


class CtlDesc(ctypes.Structure):
    """strata_ctl_desc"""
    _fields_ = [("page_size", ctypes.c_int32), ("chunk_tokens", ctypes.c_int32),
                ("num_pages", ctypes.c_int64), ("num_chunks", ctypes.c_int64),
                ("deferral_threshold", ctypes.c_int64), ("loading_bound_ratio", ctypes.c_double),
                ("max_batch_tokens", ctypes.c_int64), ("max_batch_reqs", ctypes.c_int32),
                ("flags", ctypes.c_int32)]


class Match(ctypes.Structure):
    """strata_ctl_match_t"""
    _fields_ = [(n, ctypes.c_int64) for n in ("total", "device", "host", "transient")]


class Round(ctypes.Structure):
    """strata_ctl_round"""
    _fields_ = [(n, ctypes.c_int64) for n in ("num_batch", "num_deferred", "num_formed", "formed_load",
                                              "formed_compute", "new_tokens", "load_tokens",
                                              "writeback_tokens")]


class Plan(ctypes.Structure):
    """strata_ctl_plan"""
    _fields_ = [("num_reqs", ctypes.c_int64), ("num_tokens", ctypes.POINTER(ctypes.c_int64)),
                ("chunk_start", ctypes.POINTER(ctypes.c_int64)), ("chunk_offset", ctypes.POINTER(ctypes.c_int32)),
                ("host_chunks", ctypes.POINTER(ctypes.c_int32)), ("host_chunks_len", ctypes.c_int64),
                ("page_start", ctypes.POINTER(ctypes.c_int64)), ("page_offset", ctypes.POINTER(ctypes.c_int32)),
                ("dev_pages", ctypes.POINTER(ctypes.c_int32)), ("dev_pages_len", ctypes.c_int64)]


class Stats(ctypes.Structure):
    """strata_ctl_stats"""
    _fields_ = [(n, ctypes.c_int64) for n in ("nodes", "transient_nodes", "free_pages", "free_chunks",
                                              "device_tokens", "host_tokens", "queued", "dispatched")]


_bound = False


def _l():
    global _bound
    lib = _lib.lib()
    if not _bound:
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        p64 = ctypes.POINTER(ctypes.c_int64)
        sigs = {
            "strata_ctl_create": (ctypes.c_int, [ctypes.POINTER(CtlDesc), ctypes.POINTER(vp)]),
            "strata_ctl_destroy": (ctypes.c_int, [vp]),
            "strata_ctl_insert": (ctypes.c_int, [vp, vp, i64, i32, dbl, vp]),
            "strata_ctl_match": (ctypes.c_int, [vp, vp, i64, ctypes.POINTER(Match)]),
            "strata_ctl_submit": (ctypes.c_int, [vp, i64, vp, i64]),
            "strata_ctl_schedule": (ctypes.c_int, [vp, dbl, ctypes.POINTER(Round)]),
            "strata_ctl_ids": (ctypes.c_int, [vp, i32, vp, p64]),
            "strata_ctl_plan_get": (ctypes.c_int, [vp, i32, ctypes.POINTER(Plan)]),
            "strata_ctl_req_slots": (ctypes.c_int, [vp, i64, vp, p64]),
            "strata_ctl_complete": (ctypes.c_int, [vp, i64, dbl]),
            "strata_ctl_abort": (ctypes.c_int, [vp, i64]),
            "strata_ctl_get_stats": (ctypes.c_int, [vp, ctypes.POINTER(Stats)]),
            "strata_ctl_dump": (ctypes.c_char_p, [vp]),
            "strata_ctl_bubble_steps": (ctypes.c_int64, [dbl, dbl, dbl, i64]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _bound = True
    return lib


def _tok(tokens) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))


def _arr(ptr, n: int, dtype) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def bubble_steps(t_load_ms: float, t_comp_ms: float, decode_step_ms: float, decode_reqs: int) -> int:
    return int(_l().strata_ctl_bubble_steps(t_load_ms, t_comp_ms, decode_step_ms, decode_reqs))


class Ctl:
    """One control plane (HiRadixTree + scheduler + allocators) for one KV pool and host tier."""

    def __init__(self, page_size: int, chunk_tokens: int, num_pages: int, num_chunks: int,
                 threshold: int = 100, ratio: float = 100.0, max_batch_tokens: int = 0,
                 max_batch_reqs: int = 0, defer: bool = True, balance: bool = True, bundle: bool = True):
        flags = ((0 if defer else STRATA_CTL_NO_DEFER) | (0 if balance else STRATA_CTL_NO_BALANCE)
                 | (0 if bundle else STRATA_CTL_NO_BUNDLE))
        d = CtlDesc(page_size, chunk_tokens, num_pages, num_chunks, threshold, ratio,
                    max_batch_tokens, max_batch_reqs, flags)
        h = ctypes.c_void_p()
        check(_l().strata_ctl_create(ctypes.byref(d), ctypes.byref(h)), "strata_ctl_create")
        self.h = h
        self.P, self.C = page_size, chunk_tokens

    def close(self) -> None:
        if self.h:
            _l().strata_ctl_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def insert(self, tokens, tier: int, now: float) -> List[int]:
        t = _tok(tokens)
        out = np.zeros(len(t), np.int64)
        check(_l().strata_ctl_insert(self.h, t.ctypes.data, len(t), tier, now, out.ctypes.data),
              "strata_ctl_insert")
        return out.tolist()

    def match(self, tokens) -> Dict[str, int]:
        t = _tok(tokens)
        m = Match()
        check(_l().strata_ctl_match(self.h, t.ctypes.data, len(t), ctypes.byref(m)), "strata_ctl_match")
        return {"total": m.total, "device": m.device, "host": m.host, "transient": m.transient}

    def submit(self, rid: int, tokens) -> None:
        t = _tok(tokens)
        check(_l().strata_ctl_submit(self.h, rid, t.ctypes.data, len(t)), "strata_ctl_submit")

    def ids(self, which: int) -> List[int]:
        n = ctypes.c_int64()
        check(_l().strata_ctl_ids(self.h, which, None, ctypes.byref(n)), "strata_ctl_ids")
        out = np.zeros(n.value, np.int64)
        check(_l().strata_ctl_ids(self.h, which, out.ctypes.data, ctypes.byref(n)), "strata_ctl_ids")
        return out.tolist()

    @property
    def queue(self) -> List[int]:
        return self.ids(QUEUE)

    def schedule(self, now: float) -> Dict:
        r = Round()
        check(_l().strata_ctl_schedule(self.h, now, ctypes.byref(r)), "strata_ctl_schedule")
        return {"batch": self.ids(BATCH), "deferred": self.ids(DEFERRED), "formed": self.ids(FORMED),
                "formed_load": r.formed_load, "formed_compute": r.formed_compute,
                "new_tokens": r.new_tokens, "load_tokens": r.load_tokens,
                "writeback_tokens": r.writeback_tokens}

    def plan(self, which) -> Dict[str, np.ndarray]:
        which = {"load": LOAD, "offload": WRITEBACK, "writeback": WRITEBACK}.get(which, which)
        p = Plan()
        check(_l().strata_ctl_plan_get(self.h, which, ctypes.byref(p)), "strata_ctl_plan_get")
        R = p.num_reqs
        return {"num_tokens": _arr(p.num_tokens, R, np.int64), "chunk_start": _arr(p.chunk_start, R, np.int64),
                "chunk_offset": _arr(p.chunk_offset, R, np.int32),
                "host_chunks": _arr(p.host_chunks, p.host_chunks_len, np.int32),
                "page_start": _arr(p.page_start, R, np.int64), "page_offset": _arr(p.page_offset, R, np.int32),
                "dev_pages": _arr(p.dev_pages, p.dev_pages_len, np.int32)}

    def req_slots(self, rid: int) -> np.ndarray:
        n = ctypes.c_int64()
        check(_l().strata_ctl_req_slots(self.h, rid, None, ctypes.byref(n)), "strata_ctl_req_slots")
        out = np.zeros(n.value, np.int64)
        check(_l().strata_ctl_req_slots(self.h, rid, out.ctypes.data, ctypes.byref(n)), "strata_ctl_req_slots")
        return out

    def complete(self, rid: int, now: float) -> None:
        check(_l().strata_ctl_complete(self.h, rid, now), "strata_ctl_complete")

    def abort(self, rid: int) -> None:
        check(_l().strata_ctl_abort(self.h, rid), "strata_ctl_abort")

    def stats(self) -> Dict[str, int]:
        s = Stats()
        check(_l().strata_ctl_get_stats(self.h, ctypes.byref(s)), "strata_ctl_get_stats")
        return {n: getattr(s, n) for n, _ in Stats._fields_}

    def dump(self):
        """[(path, dev, host, mark, tref, ref, last_access)] sorted by path."""
        rows = []
        for line in _l().strata_ctl_dump(self.h).decode().splitlines():
            p, d, h, mark, tref, ref, la = line.split(";")
            ints = lambda s: tuple(int(x) for x in s.split(",")) if s else ()
            rows.append((ints(p), ints(d), ints(h), int(mark), int(tref), int(ref), float(la)))
        return rows

    def xfer(self, which, device: int = 0):
        """The plan as a :class:`Requests` (index lists on `device`, host mirror kept) or None."""
        from . import Requests
        p = self.plan(which)
        if len(p["num_tokens"]) == 0:
            return None
        return Requests(p["num_tokens"], p["host_chunks"], p["chunk_start"], p["dev_pages"],
                        p["page_start"], p["chunk_offset"], p["page_offset"], device=device)
