"""Pins for the oracle's single-buffer (MLA latent) pools, KV = 1 (reading R27).

MLA (DeepSeek-V2/V3) caches one compressed latent per token and layer instead of a K and a V row;
SGLang keeps it in one buffer per layer.  The host chunk then holds [L][C][H][D] (the page-first
layout of R1 with one buffer instead of two).  Pinned, as for KV = 2, by things other than the
oracle itself:
  * closed form  — identity tables reduce LOAD to a slice of the [chunks][L][C][tok] view,
  * brute force  — the C loop oracle and the numpy oracle agree (grid, both directions),
  * tagged coordinates — every vector lands at page_table[token]; V images are never touched,
  * reduction to KV = 2 — a KV = 1 load equals the K half of a KV = 2 load from a host tier whose
    K blocks are the latent blocks (ties KV = 1 to the already pinned two-buffer definition),
  * round trip   — OFFLOAD then LOAD is the page-table permutation.
"""
import itertools

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.helpers import CANARY, dev_images, hnd_strides, slots_of, tagged_host


def _g(L=2, H=1, D=64, e=2, P=4, C=4, num_pages=24, num_chunks=12):
    return Geometry(L=L, H=H, D=D, e=e, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks, kv=1)


def test_geometry_of_deepseek_v3_latent():
    """kv_lora_rank 512 + qk_rope_head_dim 64 = 576 bf16 per token and layer: 1152 B; 61 layers."""
    g = kvgen.geometry("deepseek_v3_mla")
    assert (g.kv, g.token_bytes, g.L) == (1, 1152, 61)
    assert g.chunk_bytes == 61 * 64 * 1152          # one buffer: half a K,V chunk of the same rows


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("P,C,n", [(1, 64, 64), (4, 16, 48), (16, 32, 32)])
def test_closed_form_identity_slice_kv1(oracle_mod, impl, P, C, n):
    g = _g(L=3, H=1, D=72, e=2, P=P, C=C, num_pages=64 // P + 2, num_chunks=4)
    rng = kvgen.rng_for(31)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [n], P, C, g.num_pages, g.num_chunks, frag="identity",
                            chunk_frag="identity")
    k, v = dev_images(g)
    (oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load)(g, host, k, v, q, 0, g.L)
    hv = host.reshape(g.num_chunks, g.L, g.C, g.token_bytes)
    for l in range(g.L):
        rows = k[l].reshape(-1, g.token_bytes)
        expect = np.concatenate([hv[c, l] for c in range(-(-n // C))])[:n]
        np.testing.assert_array_equal(rows[:n], expect)
        assert (rows[n:] == CANARY).all()
        assert (v[l] == CANARY).all()


GRID = list(itertools.product([1, 3], [1, 2], [16, 72], [1, 4, 16], [1, 4, 64]))


@pytest.mark.parametrize("L,H,D,P,C", GRID)
def test_two_oracles_agree_kv1(oracle_mod, L, H, D, P, C):
    rng = kvgen.rng_for(hash(("kv1", L, H, D, P, C)) % 2**31)
    ns = [0, 1, max(P - 1, 1), P + 1, C + 1][: int(rng.integers(1, 5))]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + 3
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + 2
    g = _g(L=L, H=H, D=D, e=2, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True)
    l0 = int(rng.integers(0, L))
    l1 = int(rng.integers(l0, L + 1))
    for strides in (None, hnd_strides(g)):
        k1, v1 = dev_images(g, rng=kvgen.rng_for(1), strides=strides)
        k2, v2 = [a.copy() for a in k1], [a.copy() for a in v1]
        oracle_mod.load(g, host, k1, v1, q, l0, l1, strides=strides)
        oracle_mod.oracle_np.load(g, host, k2, v2, q, l0, l1, strides=strides)
        for a, b in zip(k1 + v1, k2 + v2):
            np.testing.assert_array_equal(a, b)
    k, v = dev_images(g, rng=rng)
    h1, h2 = host.copy(), host.copy()
    oracle_mod.offload(g, h1, k, v, q, l0, l1)
    oracle_mod.oracle_np.offload(g, h2, k, v, q, l0, l1)
    np.testing.assert_array_equal(h1, h2)


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("P,C", [(1, 4), (4, 4), (2, 8)])
def test_tagged_coordinates_kv1(oracle_mod, impl, P, C):
    L, H, D, e = 3, 2, 16, 2
    rng = kvgen.rng_for(12)
    ns = [5, 9, 1]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + 4
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + 2
    g = _g(L=L, H=H, D=D, e=e, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks)
    host = tagged_host(g)
    assert host.size == g.host_bytes
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True)
    k, v = dev_images(g)
    (oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load)(g, host, k, v, q, 1, 3)
    vph = D * e // 16
    written = set()
    for r in range(q.R):
        for pg, po, hc, ho in slots_of(q, r, g):
            slot = pg * P + po
            written.add(slot)
            for l in range(1, 3):
                row = k[l].reshape(-1, H, vph, 16)[slot].copy().view(np.uint32).reshape(H, vph, 4)
                for h in range(H):
                    for vec in range(vph):
                        assert tuple(row[h, vec]) == (hc, l << 1, ho, (h << 16) | vec)
    for l in range(L):
        assert (v[l] == CANARY).all()
        rows = k[l].reshape(-1, g.token_bytes)
        for s in range(rows.shape[0]):
            if l == 0 or s not in written:
                assert (rows[s] == CANARY).all(), (l, s)


@pytest.mark.parametrize("impl", ["c", "np"])
def test_kv1_is_k_half_of_kv2(oracle_mod, impl):
    """A KV = 1 load equals the K images of a KV = 2 load whose host K blocks hold the latents."""
    g1 = _g(L=3, H=2, D=32, e=2, P=2, C=8, num_pages=40, num_chunks=12)
    g2 = Geometry(g1.L, g1.H, g1.D, g1.e, g1.P, g1.C, g1.num_pages, g1.num_chunks, kv=2)
    rng = kvgen.rng_for(13)
    h1 = kvgen.random_bytes(rng, g1.host_bytes)
    h2 = kvgen.random_bytes(rng, g2.host_bytes)
    blk = g1.C * g1.token_bytes
    h2.reshape(g2.num_chunks, g2.L, 2, blk)[:, :, 0] = h1.reshape(g1.num_chunks, g1.L, blk)
    q = kvgen.make_requests(rng, [11, 30, 4], g1.P, g1.C, g1.num_pages, g1.num_chunks, offsets=True)
    fn = oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load
    k1, v1 = dev_images(g1)
    k2, v2 = dev_images(g2)
    fn(g1, h1, k1, v1, q, 0, g1.L)
    fn(g2, h2, k2, v2, q, 0, g2.L)
    for a, b in zip(k1, k2):
        np.testing.assert_array_equal(a, b)


def test_round_trip_offload_then_load_kv1(oracle_mod):
    g = _g(L=2, H=1, D=64, e=2, P=4, C=4, num_pages=64, num_chunks=32)
    rng = kvgen.rng_for(14)
    ns = [17, 40]
    A_k, A_v = dev_images(g, rng=rng)
    T1 = kvgen.make_requests(rng, ns, g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    T2 = kvgen.make_requests(rng, ns, g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    T2.host_chunks, T2.chunk_start, T2.chunk_offset = T1.host_chunks, T1.chunk_start, T1.chunk_offset
    host = np.zeros(g.host_bytes, np.uint8)
    oracle_mod.offload(g, host, A_k, A_v, T1, 0, g.L)
    B_k, B_v = dev_images(g)
    oracle_mod.load(g, host, B_k, B_v, T2, 0, g.L)
    for r in range(len(ns)):
        for (p1, o1, _, _), (p2, o2, _, _) in zip(slots_of(T1, r, g), slots_of(T2, r, g)):
            for l in range(g.L):
                a = A_k[l].reshape(-1, g.token_bytes)[p1 * g.P + o1]
                b = B_k[l].reshape(-1, g.token_bytes)[p2 * g.P + o2]
                np.testing.assert_array_equal(a, b)
    assert all((b == CANARY).all() for b in B_v)
