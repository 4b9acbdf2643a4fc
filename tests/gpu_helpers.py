"""Helpers for the GPU parity tests: build a pool + device buffers through the C ABI binding, run
the CUDA path, and compute the expected images with the CPU oracle from the same seeded inputs."""
from __future__ import annotations

from typing import List, Optional

import numpy as np

import kvgen
import oracle
from tests.helpers import CANARY


def default_engine(g, strides=None, direction: str = "load", op_bytes: int = 0) -> int:
    """The engine strata_load/offload pick with STRATA_ENGINE_DEFAULT (transfer.cpp): loads of
    16-byte-granular rows of >= 16 MiB take the LDG engine (the paper's configuration, NEXT-1);
    otherwise the ring engine (STRATA_ENGINE_TMA) when the tier has whole host rows in 16-byte units — or, for
    loads, narrow rows (R29) of 8- or 4-byte granularity whose host rows of a chunk form one run and
    whose device rows are head-contiguous; else LDG (a head-major tier with several heads per GPU,
    narrow offloads, 2- / 1-byte granularity).  Assumes a library-allocated (aligned) host tier."""
    import paper_2508_18572_b200 as st
    if getattr(g, "head_major", False) and g.H > 1:
        return st.STRATA_ENGINE_LDG
    vals = [g.H * g.D * g.e, g.D * g.e] + list(strides or ())
    gran = 16
    for v in vals:
        while gran > 1 and v % gran:
            gran //= 2
    if gran == 16 and direction == "load" and op_bytes >= 16 << 20:
        return st.STRATA_ENGINE_LDG
    if gran == 16:
        return st.STRATA_ENGINE_TMA
    Ht = getattr(g, "Ht", 0) or g.H
    head_contig = strides is None or strides[2] == g.D * g.e or g.H == 1
    if direction == "load" and gran in (8, 4) and Ht == g.H and head_contig:
        return st.STRATA_ENGINE_TMA
    return st.STRATA_ENGINE_LDG


def nhd(g):
    tok = g.H * g.D * g.e
    return (g.P * tok, tok, g.D * g.e)


class GpuCase:
    """Device pool (one K and one V uint8 buffer per layer) + registered host tier + request tables."""

    def __init__(self, g, q, strides=None, flags: int = 0, host_fill: str = "random", seed: int = 0,
                 dev_fill: str = "canary"):
        import torch

        import paper_2508_18572_b200 as st
        self.g, self.q = g, q
        self.strides = strides or nhd(g)
        ps, ts, hs = self.strides
        self.layer_bytes = g.num_pages * ps
        rng = kvgen.rng_for(seed)
        if dev_fill == "canary":
            self.k = [torch.full((self.layer_bytes,), CANARY, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
            self.v = [torch.full((self.layer_bytes,), CANARY, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        else:
            gen = torch.Generator(device="cuda")
            gen.manual_seed(seed)
            self.k = [torch.randint(0, 256, (self.layer_bytes,), dtype=torch.uint8, device="cuda", generator=gen)
                      for _ in range(g.L)]
            self.v = [torch.randint(0, 256, (self.layer_bytes,), dtype=torch.uint8, device="cuda", generator=gen)
                      for _ in range(g.L)]
        self.pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P,
                                chunk_tokens=g.C, k_ptrs=self.k,
                                # KV = 1 (MLA latent): one buffer per layer; self.v stays canary
                                v_ptrs=None if getattr(g, "kv", 2) == 1 else self.v, num_pages=g.num_pages,
                                num_chunks=g.num_chunks, flags=flags,
                                strides=(0, 0, 0) if strides is None else strides,
                                host_heads=getattr(g, "Ht", 0), head_begin=getattr(g, "h0", 0),
                                head_major=getattr(g, "head_major", False))
        if host_fill == "random":
            if g.host_bytes <= (64 << 20):
                self.pool.host[:] = kvgen.random_bytes(rng, g.host_bytes)
            else:
                kvgen.fill_random(self.pool.host[: g.host_bytes], seed)
        self.reqs = st.Requests.from_kvgen(q)

    def close(self):
        self.pool.close()

    # -- expected images ------------------------------------------------------------------------
    def expected_load_layer(self, l: int, pre_k: Optional[np.ndarray] = None, pre_v: Optional[np.ndarray] = None):
        """Oracle LOAD of layer l from the host tier into canary (or given) pre-state images."""
        g = self.g
        ek: List[Optional[np.ndarray]] = [None] * g.L
        ev: List[Optional[np.ndarray]] = [None] * g.L
        ek[l] = np.full(self.layer_bytes, CANARY, np.uint8) if pre_k is None else pre_k.copy()
        ev[l] = np.full(self.layer_bytes, CANARY, np.uint8) if pre_v is None else pre_v.copy()
        oracle.load(g, self.pool.host[: g.host_bytes], ek, ev, self.q, l, l + 1, strides=self.strides)
        return ek[l], ev[l]

    def check_load(self, l0: int, l1: int, layers=None):
        """Every byte of every layer's K/V equals the oracle image (untouched layers: canary)."""
        g = self.g
        layers = range(g.L) if layers is None else layers
        for l in layers:
            got_k = self.k[l].cpu().numpy()
            got_v = self.v[l].cpu().numpy()
            if l0 <= l < l1:
                ek, ev = self.expected_load_layer(l)
            else:
                ek = ev = np.full(self.layer_bytes, CANARY, np.uint8)
            _assert_same(got_k, ek, f"K layer {l}")
            _assert_same(got_v, ev, f"V layer {l}")

    def expected_offload(self, host_before: np.ndarray, l0: int, l1: int) -> np.ndarray:
        g = self.g
        ks = [t.cpu().numpy() if l0 <= l < l1 else None for l, t in enumerate(self.k)]
        vs = [t.cpu().numpy() if l0 <= l < l1 else None for l, t in enumerate(self.v)]
        out = host_before.copy()
        oracle.offload(g, out, ks, vs, self.q, l0, l1, strides=self.strides)
        return out


def _assert_same(got: np.ndarray, exp: np.ndarray, what: str):
    if not np.array_equal(got, exp):
        bad = np.flatnonzero(got != exp)
        raise AssertionError(f"{what}: {bad.size} bytes differ, first at {bad[0]} "
                             f"(got {got[bad[0]]:#x}, expected {exp[bad[0]]:#x})")
