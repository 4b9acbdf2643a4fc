"""Pins for the CPU oracle (``-m "not gpu"``): nothing here compares the oracle with itself.

Each test ties the oracle to something the paper or the mathematics fixes:
  * closed form  — identity tables reduce LOAD to a numpy slice,
  * brute force  — the C loop oracle and the numpy fancy-index oracle agree on a grid and on every
                   page-table permutation of a tiny pool,
  * tagged coordinates — every valid token's bytes land exactly at page_table[token] (north_star),
  * conservation — nothing outside the destination rows changes,
  * round trip   — OFFLOAD then LOAD is the page-table permutation; LOAD then OFFLOAD restores host,
  * TP union     — head-slice loads concatenate to the full-head load,
  * geometry / partial-page values printed in PAPER.md / SPEC.md (tests/golden/geometry.json).
"""
import itertools
import json
import os

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.helpers import (CANARY, dev_images, hnd_strides, nhd_strides, slots_of, tagged_host)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _geom(L=2, H=2, D=8, e=2, P=4, C=4, num_pages=16, num_chunks=8):
    return Geometry(L=L, H=H, D=D, e=e, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks)


def _run_both(oracle_mod, g, host, q, l0, l1, strides=None, seed=0):
    """LOAD with both oracles from identical random pre-states; return both post-states."""
    rng = kvgen.rng_for(seed)
    k1, v1 = dev_images(g, rng=rng, strides=strides)
    k2, v2 = [a.copy() for a in k1], [a.copy() for a in v1]
    oracle_mod.load(g, host, k1, v1, q, l0, l1, strides=strides)
    oracle_mod.oracle_np.load(g, host, k2, v2, q, l0, l1, strides=strides)
    return (k1, v1), (k2, v2)


# ----------------------------------------------------------------------------------------------
# Closed form: identity tables reduce LOAD to a slice of the page-first host view.
@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("P,C,n", [(1, 64, 64), (4, 64, 48), (16, 32, 32), (2, 8, 8)])
def test_closed_form_identity_slice(oracle_mod, impl, P, C, n):
    g = _geom(L=3, H=2, D=8, e=2, P=P, C=C, num_pages=64 // P + 2, num_chunks=2)
    rng = kvgen.rng_for(1)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [n], P, C, g.num_pages, g.num_chunks, frag="identity",
                            chunk_frag="identity")
    k, v = dev_images(g)
    fn = oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load
    fn(g, host, k, v, q, 0, g.L)
    hv = host.reshape(g.num_chunks, g.L, 2, g.C, g.token_bytes)
    for l in range(g.L):
        for kv, imgs in ((0, k), (1, v)):
            rows = imgs[l].reshape(-1, g.token_bytes)
            np.testing.assert_array_equal(rows[:n], hv[0, l, kv, :n])
            assert (rows[n:] == CANARY).all()


@pytest.mark.parametrize("impl", ["c", "np"])
def test_closed_form_chunks_equal_pages(oracle_mod, impl):
    """C == P, identity pages, chunk list = permutation: device rows = host chunks in list order."""
    P = C = 4
    g = _geom(L=2, H=1, D=16, e=1, P=P, C=C, num_pages=8, num_chunks=8)
    rng = kvgen.rng_for(2)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [32], P, C, g.num_pages, g.num_chunks, frag="identity")
    k, v = dev_images(g)
    (oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load)(g, host, k, v, q, 0, g.L)
    hv = host.reshape(g.num_chunks, g.L, 2, C * g.token_bytes)
    for l in range(g.L):
        for kv, imgs in ((0, k), (1, v)):
            expect = np.concatenate([hv[c, l, kv] for c in q.host_chunks])
            np.testing.assert_array_equal(imgs[l], expect)


# ----------------------------------------------------------------------------------------------
# Brute force: two independent oracles agree byte for byte.
GRID = list(itertools.product([1, 3], [1, 2], [8, 64], [1, 2], [1, 2, 4, 16], [1, 4, 16, 64]))


@pytest.mark.parametrize("L,H,D,e,P,C", GRID)
def test_two_oracles_agree_grid(oracle_mod, L, H, D, e, P, C):
    # the oracles are byte-granular: rows of 8 bytes (D*e % 16 != 0) are pinned here too (R29)
    rng = kvgen.rng_for(hash((L, H, D, e, P, C)) % 2**31)
    ns = [0, 1, max(P - 1, 1), P, P + 1, C + 1][: int(rng.integers(1, 4))]
    g0 = _geom(L=L, H=H, D=D, e=e, P=P, C=C, num_pages=1, num_chunks=1)
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + 3
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + 2
    g = Geometry(L, H, D, e, P, C, num_pages, num_chunks)
    del g0
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True)
    l0 = int(rng.integers(0, L))
    l1 = int(rng.integers(l0, L + 1))
    for strides in (None, hnd_strides(g)):
        (k1, v1), (k2, v2) = _run_both(oracle_mod, g, host, q, l0, l1, strides=strides)
        for a, b in zip(k1 + v1, k2 + v2):
            np.testing.assert_array_equal(a, b)
    # offload direction
    k, v = dev_images(g, rng=rng)
    h1, h2 = host.copy(), host.copy()
    oracle_mod.offload(g, h1, k, v, q, l0, l1)
    oracle_mod.oracle_np.offload(g, h2, k, v, q, l0, l1)
    np.testing.assert_array_equal(h1, h2)


@pytest.mark.parametrize("num_pages,P", [(4, 1), (5, 1), (4, 2), (5, 4)])
def test_two_oracles_agree_every_permutation(oracle_mod, num_pages, P):
    """Every page-table permutation of a 4-5 page pool (SURVEY.md §8c brute force)."""
    g = _geom(L=2, H=1, D=16, e=1, P=P, C=4, num_pages=num_pages, num_chunks=(num_pages * P + 3) // 4)
    rng = kvgen.rng_for(7)
    host = kvgen.random_bytes(rng, g.host_bytes)
    n = num_pages * P
    base = kvgen.make_requests(rng, [n], P, g.C, num_pages, g.num_chunks, frag="identity")
    for perm in itertools.permutations(range(num_pages)):
        base.dev_pages = np.asarray(perm, np.int32)
        (k1, v1), (k2, v2) = _run_both(oracle_mod, g, host, base, 0, g.L)
        for a, b in zip(k1 + v1, k2 + v2):
            np.testing.assert_array_equal(a, b)


# ----------------------------------------------------------------------------------------------
# Tagged coordinates: decode every valid vector; untouched slots keep their canary.
@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("P,C,offsets", [(1, 4, False), (4, 4, True), (2, 8, True), (16, 4, True)])
def test_tagged_coordinates(oracle_mod, impl, P, C, offsets):
    L, H, D, e = 3, 2, 16, 2
    rng = kvgen.rng_for(11)
    ns = [5, 9, 1]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + 4
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + 2
    g = Geometry(L, H, D, e, P, C, num_pages, num_chunks)
    host = tagged_host(g)
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=offsets)
    k, v = dev_images(g)
    (oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load)(g, host, k, v, q, 1, 3)
    vph = D * e // 16
    written = set()
    for r in range(q.R):
        for pg, po, hc, ho in slots_of(q, r, g):
            slot = pg * P + po
            written.add(slot)
            for l in range(1, 3):
                for kv, imgs in ((0, k), (1, v)):
                    row = imgs[l].reshape(-1, H, vph, 4 * 4)[slot].copy().view(np.uint32).reshape(H, vph, 4)
                    for h in range(H):
                        for vec in range(vph):
                            assert tuple(row[h, vec]) == (hc, (l << 1) | kv, ho, (h << 16) | vec)
    for l in range(L):
        for imgs in (k, v):
            rows = imgs[l].reshape(-1, g.token_bytes)
            for s in range(rows.shape[0]):
                if l == 0 or s not in written:
                    assert (rows[s] == CANARY).all(), (l, s)


# ----------------------------------------------------------------------------------------------
# Conservation: only destination rows change; the number of changed rows is bounded.
def test_conservation_mask(oracle_mod):
    g = _geom(L=2, H=2, D=8, e=2, P=4, C=4, num_pages=32, num_chunks=16)
    rng = kvgen.rng_for(5)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [7, 13, 2], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    k0, v0 = dev_images(g, rng=rng)
    k, v = [a.copy() for a in k0], [a.copy() for a in v0]
    oracle_mod.load(g, host, k, v, q, 0, 2)
    mask = np.zeros(g.num_pages * g.P, bool)
    for r in range(q.R):
        for pg, po, _, _ in slots_of(q, r, g):
            mask[pg * g.P + po] = True
    for a0, a in zip(k0 + v0, k + v):
        rows0, rows = a0.reshape(-1, g.token_bytes), a.reshape(-1, g.token_bytes)
        np.testing.assert_array_equal(rows0[~mask], rows[~mask])
        changed = np.count_nonzero((rows0 != rows).any(axis=1))
        assert changed <= int(q.num_tokens.sum())


# ----------------------------------------------------------------------------------------------
# Round trip identity.
@pytest.mark.parametrize("P,C", [(1, 16), (4, 4), (16, 64), (3, 5)])
def test_round_trip_offload_then_load(oracle_mod, P, C):
    g = Geometry(L=2, H=2, D=16, e=2, P=P, C=C, num_pages=64, num_chunks=32)
    rng = kvgen.rng_for(3)
    ns = [17, 40]
    A_k, A_v = dev_images(g, rng=rng)
    T1 = kvgen.make_requests(rng, ns, P, C, g.num_pages, g.num_chunks, offsets=True)
    T2 = kvgen.make_requests(rng, ns, P, C, g.num_pages, g.num_chunks, offsets=True)
    # T2 must reuse T1's host positions: same chunk lists and chunk offsets
    T2.host_chunks, T2.chunk_start, T2.chunk_offset = T1.host_chunks, T1.chunk_start, T1.chunk_offset
    host = np.zeros(g.host_bytes, np.uint8)
    oracle_mod.offload(g, host, A_k, A_v, T1, 0, g.L)
    B_k, B_v = dev_images(g)
    oracle_mod.load(g, host, B_k, B_v, T2, 0, g.L)
    for r in range(len(ns)):
        for (p1, o1, _, _), (p2, o2, _, _) in zip(slots_of(T1, r, g), slots_of(T2, r, g)):
            for A, B in ((A_k, B_k), (A_v, B_v)):
                for l in range(g.L):
                    a = A[l].reshape(-1, g.token_bytes)[p1 * P + o1]
                    b = B[l].reshape(-1, g.token_bytes)[p2 * P + o2]
                    np.testing.assert_array_equal(a, b)


def test_round_trip_load_then_offload(oracle_mod):
    g = Geometry(L=3, H=1, D=32, e=2, P=2, C=8, num_pages=40, num_chunks=12)
    rng = kvgen.rng_for(4)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [16, 24], g.P, g.C, g.num_pages, g.num_chunks)  # chunk aligned
    k, v = dev_images(g)
    oracle_mod.load(g, host, k, v, q, 0, g.L)
    fresh = kvgen.make_requests(rng, [16, 24], g.P, g.C, g.num_pages, g.num_chunks)
    fresh.dev_pages, fresh.page_start, fresh.page_offset = q.dev_pages, q.page_start, q.page_offset
    out = np.zeros_like(host)
    oracle_mod.offload(g, out, k, v, fresh, 0, g.L)
    hv, ov = host.reshape(g.num_chunks, -1), out.reshape(g.num_chunks, -1)
    for a, b in zip(q.host_chunks, fresh.host_chunks):
        np.testing.assert_array_equal(hv[a], ov[b])


# ----------------------------------------------------------------------------------------------
# TP union: per-rank head slices concatenate to the full-head load.
@pytest.mark.parametrize("T", [2, 4])
def test_tp_union(oracle_mod, T):
    H = 4
    g = Geometry(L=2, H=H, D=16, e=2, P=2, C=4, num_pages=24, num_chunks=12)
    rng = kvgen.rng_for(9)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [9, 14], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    kf, vf = dev_images(g)
    oracle_mod.load(g, host, kf, vf, q, 0, g.L)
    hv = host.reshape(g.num_chunks, g.L, 2, g.C, H, g.D * g.e)
    parts_k, parts_v = [], []
    for rank in range(T):
        hs = kvgen.head_slice(rank, T, H)
        gr = Geometry(g.L, len(hs), g.D, g.e, g.P, g.C, g.num_pages, g.num_chunks)
        host_r = np.ascontiguousarray(hv[:, :, :, :, hs.start:hs.stop]).reshape(-1)
        kr, vr = dev_images(gr)
        oracle_mod.load(gr, host_r, kr, vr, q, 0, g.L)
        parts_k.append(kr)
        parts_v.append(vr)
    for l in range(g.L):
        for full, parts in ((kf, parts_k), (vf, parts_v)):
            cat = np.concatenate([p[l].reshape(-1, len(kvgen.head_slice(0, T, H)), g.D * g.e)
                                  for p in parts], axis=1)
            np.testing.assert_array_equal(full[l].reshape(-1, H, g.D * g.e), cat)


# ----------------------------------------------------------------------------------------------
# Edge cases and errors.
def test_empty_and_empty_layer_range(oracle_mod):
    g = _geom()
    rng = kvgen.rng_for(0)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [0, 0], g.P, g.C, g.num_pages, g.num_chunks)
    k, v = dev_images(g)
    oracle_mod.load(g, host, k, v, q, 0, g.L)
    q2 = kvgen.make_requests(rng, [5], g.P, g.C, g.num_pages, g.num_chunks)
    oracle_mod.load(g, host, k, v, q2, 1, 1)
    assert all((a == CANARY).all() for a in k + v)


def test_out_of_range_index_raises(oracle_mod):
    g = _geom()
    rng = kvgen.rng_for(0)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [4], g.P, g.C, g.num_pages, g.num_chunks)
    q.dev_pages = np.array([g.num_pages], np.int32)
    k, v = dev_images(g)
    with pytest.raises(IndexError):
        oracle_mod.load(g, host, k, v, q, 0, g.L)
    with pytest.raises(IndexError):
        oracle_mod.oracle_np.load(g, host, k, v, q, 0, g.L)


def test_nan_and_negative_zero_payloads_preserved(oracle_mod):
    """Opaque bytes: fp16/bf16 NaN payloads and -0.0 survive bit-exactly (reading R9)."""
    g = _geom(L=1, H=1, D=8, e=2, P=1, C=8, num_pages=8, num_chunks=1)
    pats = np.array([0x7E01, 0xFE7F, 0x8000, 0x7FC1, 0xFFFF, 0x7C01, 0x0001, 0x8001], np.uint16)
    host = np.tile(pats, g.host_bytes // 16).view(np.uint8).copy()
    q = kvgen.make_requests(kvgen.rng_for(0), [8], 1, 8, 8, 1)
    k, v = dev_images(g)
    oracle_mod.load(g, host, k, v, q, 0, 1)
    hv = host.reshape(1, 1, 2, 8, 16)
    for kv, imgs in ((0, k), (1, v)):
        rows = imgs[0].reshape(8, 16)
        for i, slot in enumerate(q.dev_pages):
            np.testing.assert_array_equal(rows[slot], hv[0, 0, kv, i])


# ----------------------------------------------------------------------------------------------
# Values the paper / SPEC print.
def test_geometry_golden():
    gold = json.load(open(os.path.join(GOLDEN, "geometry.json")))
    g = kvgen.geometry("llama8b_32k")
    assert 2 * g.token_bytes == gold["llama8b_kv_bytes_per_token_per_layer"]["value"]
    g32 = Geometry(g.L, g.H, g.D, g.e, 32, 32, 1, 1)
    assert 2 * g32.C * g32.token_bytes == gold["llama8b_layer_chunk_bytes_page32"]["value"]
    assert g32.chunk_bytes == gold["llama8b_page_first_chunk_bytes_page32"]["value"]
    t = gold["llama8b_tokens_in_40GB"]
    per_token = g.L * 2 * g.token_bytes
    assert abs(t["hbm_bytes"] / per_token - t["value_approx"]) <= t["rel_tol"] * t["value_approx"]
    rng_ = gold["token_bytes_range_all_layers"]
    for name in ("llama8b_32k", "qwen14b_batch8"):
        gg = kvgen.geometry(name)
        assert rng_["min"] <= gg.L * 2 * gg.token_bytes <= rng_["max"]


def test_partial_pages_golden():
    gold = json.load(open(os.path.join(GOLDEN, "geometry.json")))["partial_pages_page32"]
    for n, pages in gold["cases"]:
        assert kvgen.pages_needed(0, n, gold["P"]) == pages


def test_generators_deterministic_and_duplicate_free():
    a = kvgen.make_requests(kvgen.rng_for(3), [100, 7], 4, 16, 64, 16, offsets=True)
    b = kvgen.make_requests(kvgen.rng_for(3), [100, 7], 4, 16, 64, 16, offsets=True)
    for f in ("num_tokens", "host_chunks", "dev_pages", "page_offset", "chunk_offset"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    assert len(set(a.dev_pages.tolist())) == a.dev_pages.size
    assert len(set(a.host_chunks.tolist())) == a.host_chunks.size
    churn = kvgen.churn_free_list(kvgen.rng_for(1), 4096, 16, rounds=200)
    assert sorted(churn.tolist()) == list(range(4096))


def test_fill_random_deterministic():
    a = np.empty(3 * (1 << 20) + 5, np.uint8)
    b = np.empty_like(a)
    kvgen.fill_random(a, 7, block=1 << 20)
    kvgen.fill_random(b, 7, block=1 << 20)
    np.testing.assert_array_equal(a, b)
    blocks = a[: 3 << 20].reshape(3, -1)
    assert not (blocks[0] == blocks[1]).all()
