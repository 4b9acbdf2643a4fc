"""Pins for host tiers holding more heads than one GPU moves, and for the head-major chunk layout
(reading R28; SURVEY.md §8f "head-major host chunk for TP-degree-independent host tiers").

A host tier may hold Ht >= H KV heads per token (e.g. every KV head of the model, shared by all
tensor-parallel ranks, or written by a deployment with another TP degree); a GPU moves its heads
[h0, h0+H).  Token-major chunks keep R1's [L][KV][C][Ht][D]; head-major chunks keep
[Ht][L][KV][C][D], so each head's part of a chunk is a one-head page-first chunk.  Pinned by:
  * layout equivalence — a head-major tier built by numpy.transpose of a token-major tier loads to
    the same device bytes (ties head-major to the pinned token-major definition),
  * slicing        — a slice load equals the load from the compact per-rank tier cut out by numpy
    slicing (ties Ht > H to the per-GPU tier of R13, pinned in test_oracle.py),
  * TP union       — the T rank slices loaded from ONE shared tier concatenate to the full load,
  * tagged coordinates — each vector lands at page_table[token] with its GLOBAL head h0 + h,
  * Ht = H = 1     — both layouts are the same bytes,
  * brute force    — the C and numpy oracles agree on a grid of layouts, Ht, h0, H, KV.
"""
import dataclasses
import itertools

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.helpers import CANARY, dev_images, slots_of


def _geom(H=2, Ht=4, h0=1, head_major=False, L=2, D=16, e=2, P=2, C=4, kv=2, num_pages=40, num_chunks=16):
    return Geometry(L=L, H=H, D=D, e=e, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks, kv=kv, Ht=Ht,
                    h0=h0, head_major=head_major)


def _to_head_major(host, g):
    v = host.reshape(g.num_chunks, g.L, g.kv, g.C, g.host_heads, g.D * g.e)
    return np.ascontiguousarray(v.transpose(0, 4, 1, 2, 3, 5)).reshape(-1)


def _load(oracle_mod, impl, g, host, q, l0=0, l1=None):
    k, v = dev_images(g)
    fn = oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load
    fn(g, host, k, v, q, l0, g.L if l1 is None else l1)
    return k, v


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("H,Ht,h0,kv", [(2, 4, 1, 2), (1, 8, 7, 2), (4, 4, 0, 2), (2, 4, 2, 1)])
def test_head_major_equals_transposed_token_major(oracle_mod, impl, H, Ht, h0, kv):
    g_tok = _geom(H=H, Ht=Ht, h0=h0, kv=kv)
    g_hm = dataclasses.replace(g_tok, head_major=True)
    rng = kvgen.rng_for(61)
    host = kvgen.random_bytes(rng, g_tok.host_bytes)
    q = kvgen.make_requests(rng, [13, 22, 3], g_tok.P, g_tok.C, g_tok.num_pages, g_tok.num_chunks, offsets=True)
    a = _load(oracle_mod, impl, g_tok, host, q)
    b = _load(oracle_mod, impl, g_hm, _to_head_major(host, g_tok), q)
    for x, y in zip(a[0] + a[1], b[0] + b[1]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("head_major", [False, True])
def test_slice_equals_compact_rank_tier(oracle_mod, impl, head_major):
    g = _geom(H=2, Ht=6, h0=3, head_major=head_major)
    rng = kvgen.rng_for(62)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [9, 17], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    # the compact per-rank tier (Ht = H, h0 = 0, token-major) cut out with numpy slicing
    if head_major:
        v = host.reshape(g.num_chunks, g.host_heads, g.L, g.kv, g.C, g.D * g.e)
        part = v[:, g.h0:g.h0 + g.H].transpose(0, 2, 3, 4, 1, 5)
    else:
        v = host.reshape(g.num_chunks, g.L, g.kv, g.C, g.host_heads, g.D * g.e)
        part = v[:, :, :, :, g.h0:g.h0 + g.H]
    compact = np.ascontiguousarray(part).reshape(-1)
    g_rank = dataclasses.replace(g, Ht=0, h0=0, head_major=False)
    a = _load(oracle_mod, impl, g, host, q)
    b = _load(oracle_mod, impl, g_rank, compact, q)
    for x, y in zip(a[0] + a[1], b[0] + b[1]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("head_major", [False, True])
@pytest.mark.parametrize("T", [2, 4])
def test_tp_union_from_one_shared_tier(oracle_mod, head_major, T):
    Htot = 4
    g_full = _geom(H=Htot, Ht=Htot, h0=0, head_major=head_major)
    rng = kvgen.rng_for(63)
    host = kvgen.random_bytes(rng, g_full.host_bytes)
    q = kvgen.make_requests(rng, [11, 6], g_full.P, g_full.C, g_full.num_pages, g_full.num_chunks, offsets=True)
    full = _load(oracle_mod, "c", g_full, host, q)
    slots = g_full.num_pages * g_full.P
    for side in (0, 1):
        for l in range(g_full.L):
            parts = []
            for r in range(T):
                hs = kvgen.head_slice(r, T, Htot)
                g_r = dataclasses.replace(g_full, H=len(hs), h0=hs.start)
                parts.append(_load(oracle_mod, "c", g_r, host, q)[side][l].reshape(slots, len(hs), -1))
            np.testing.assert_array_equal(np.concatenate(parts, axis=1).reshape(-1), full[side][l])


def _tagged(g):
    vph = g.D * g.e // 16
    Ht = g.host_heads
    if g.head_major:
        order = (g.num_chunks, Ht, g.L, g.kv, g.C, vph)
        c, h, l, kv, t, vec = np.meshgrid(*[np.arange(s, dtype=np.uint32) for s in order], indexing="ij")
    else:
        order = (g.num_chunks, g.L, g.kv, g.C, Ht, vph)
        c, l, kv, t, h, vec = np.meshgrid(*[np.arange(s, dtype=np.uint32) for s in order], indexing="ij")
    tags = np.stack([c, (l << 1) | kv, t, (h << 16) | vec], axis=-1)
    return np.ascontiguousarray(tags).view(np.uint8).reshape(-1)


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("head_major", [False, True])
def test_tagged_global_heads(oracle_mod, impl, head_major):
    g = _geom(H=2, Ht=5, h0=2, head_major=head_major, L=3, D=16, P=4, C=4)
    host = _tagged(g)
    assert host.size == g.host_bytes
    rng = kvgen.rng_for(64)
    q = kvgen.make_requests(rng, [5, 9], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    k, v = _load(oracle_mod, impl, g, host, q, 1, 3)
    vph = g.D * g.e // 16
    written = set()
    for r in range(q.R):
        for pg, po, hc, ho in slots_of(q, r, g):
            slot = pg * g.P + po
            written.add(slot)
            for l in range(1, 3):
                for kvi, imgs in ((0, k), (1, v)):
                    row = imgs[l].reshape(-1, g.H, vph, 16)[slot].copy().view(np.uint32).reshape(g.H, vph, 4)
                    for h in range(g.H):
                        for vec in range(vph):
                            assert tuple(row[h, vec]) == (hc, (l << 1) | kvi, ho, ((g.h0 + h) << 16) | vec)
    for l in range(g.L):
        for imgs in (k, v):
            rows = imgs[l].reshape(-1, g.token_bytes)
            for s in range(rows.shape[0]):
                if l == 0 or s not in written:
                    assert (rows[s] == CANARY).all()


def test_single_head_layouts_coincide(oracle_mod):
    g = _geom(H=1, Ht=1, h0=0, head_major=False)
    rng = kvgen.rng_for(65)
    host = kvgen.random_bytes(rng, g.host_bytes)
    np.testing.assert_array_equal(_to_head_major(host, g), host)
    q = kvgen.make_requests(rng, [20], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    a = _load(oracle_mod, "c", g, host, q)
    b = _load(oracle_mod, "c", dataclasses.replace(g, head_major=True), host, q)
    for x, y in zip(a[0] + a[1], b[0] + b[1]):
        np.testing.assert_array_equal(x, y)


GRID = list(itertools.product([False, True], [(1, 1, 0), (2, 4, 2), (1, 8, 5), (3, 3, 0)], [1, 2], [1, 4], [4, 16]))


@pytest.mark.parametrize("head_major,heads,kv,P,C", GRID)
def test_two_oracles_agree_heads(oracle_mod, head_major, heads, kv, P, C):
    H, Ht, h0 = heads
    rng = kvgen.rng_for(hash(("heads", head_major, heads, kv, P, C)) % 2**31)
    ns = [int(x) for x in rng.integers(0, 2 * C + 3, size=3)]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + 3
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + 2
    g = _geom(H=H, Ht=Ht, h0=h0, head_major=head_major, kv=kv, L=2, D=16, P=P, C=C, num_pages=num_pages,
              num_chunks=num_chunks)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True)
    a = _load(oracle_mod, "c", g, host, q, 1, 2)
    b = _load(oracle_mod, "np", g, host, q, 1, 2)
    for x, y in zip(a[0] + a[1], b[0] + b[1]):
        np.testing.assert_array_equal(x, y)
    k, v = dev_images(g, rng=rng)
    h1, h2 = host.copy(), host.copy()
    oracle_mod.offload(g, h1, k, v, q, 0, g.L)
    oracle_mod.oracle_np.offload(g, h2, k, v, q, 0, g.L)
    np.testing.assert_array_equal(h1, h2)
