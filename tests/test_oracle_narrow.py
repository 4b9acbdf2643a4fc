"""Pins for rows that are not a multiple of 16 bytes (reading R29; SURVEY.md §8f "an fp8 KV
scalar fallback for S_tok % 16 != 0"): the oracles are byte-granular, so odd row sizes are pinned the
same way as the 16-byte ones — closed form (identity tables reduce LOAD to a slice), two-oracle
brute force over odd sizes and all layouts, and the offload -> load round trip."""
import itertools

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.helpers import CANARY, dev_images, hnd_strides, slots_of

SIZES = [(1, 1, 1), (3, 1, 1), (2, 3, 1), (1, 5, 2), (3, 4, 2), (1, 72, 1), (2, 60, 1)]   # (H, D, e)


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("H,D,e", SIZES)
def test_closed_form_identity_slice_narrow(oracle_mod, impl, H, D, e):
    P, C, n = 4, 8, 20
    g = Geometry(L=2, H=H, D=D, e=e, P=P, C=C, num_pages=8, num_chunks=3)
    rng = kvgen.rng_for(71)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, [n], P, C, g.num_pages, g.num_chunks, frag="identity", chunk_frag="identity")
    k, v = dev_images(g)
    (oracle_mod.load if impl == "c" else oracle_mod.oracle_np.load)(g, host, k, v, q, 0, g.L)
    hv = host.reshape(g.num_chunks, g.L, 2, g.C, g.token_bytes)
    for l in range(g.L):
        for kv, imgs in ((0, k), (1, v)):
            rows = imgs[l].reshape(-1, g.token_bytes)
            expect = np.concatenate([hv[c, l, kv] for c in range(g.num_chunks)])[:n]
            np.testing.assert_array_equal(rows[:n], expect)
            assert (rows[n:] == CANARY).all()


@pytest.mark.parametrize("H,D,e,kv,P,C", list(itertools.product([1, 3], [3, 5], [1, 2], [1, 2], [1, 4], [1, 8])))
def test_two_oracles_agree_narrow(oracle_mod, H, D, e, kv, P, C):
    rng = kvgen.rng_for(hash(("narrow", H, D, e, kv, P, C)) % 2**31)
    ns = [int(x) for x in rng.integers(0, 2 * C + 3, size=3)]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + 3
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + 2
    g = Geometry(L=2, H=H, D=D, e=e, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks, kv=kv)
    host = kvgen.random_bytes(rng, g.host_bytes)
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True)
    for strides in (None, hnd_strides(g)):
        k1, v1 = dev_images(g, rng=kvgen.rng_for(2), strides=strides)
        k2, v2 = [a.copy() for a in k1], [a.copy() for a in v1]
        oracle_mod.load(g, host, k1, v1, q, 0, g.L, strides=strides)
        oracle_mod.oracle_np.load(g, host, k2, v2, q, 0, g.L, strides=strides)
        for a, b in zip(k1 + v1, k2 + v2):
            np.testing.assert_array_equal(a, b)
    k, v = dev_images(g, rng=rng)
    h1, h2 = host.copy(), host.copy()
    oracle_mod.offload(g, h1, k, v, q, 0, g.L)
    oracle_mod.oracle_np.offload(g, h2, k, v, q, 0, g.L)
    np.testing.assert_array_equal(h1, h2)


@pytest.mark.parametrize("H,D,e", SIZES)
def test_round_trip_narrow(oracle_mod, H, D, e):
    g = Geometry(L=2, H=H, D=D, e=e, P=3, C=5, num_pages=60, num_chunks=30)
    rng = kvgen.rng_for(72)
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
            for A, B in ((A_k, B_k), (A_v, B_v)):
                for l in range(g.L):
                    np.testing.assert_array_equal(A[l].reshape(-1, g.token_bytes)[p1 * g.P + o1],
                                                  B[l].reshape(-1, g.token_bytes)[p2 * g.P + o2])
