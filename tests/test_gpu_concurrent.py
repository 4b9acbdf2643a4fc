"""Several operations of ONE pool in flight at once on different streams: a load and
an offload (both directions of the link at once), two loads, two offloads — every engine pairing,
each result bit-exact against the oracle.  The operations touch disjoint device slots and host
chunks, so each one's expected image is independent of the other's timing."""
import numpy as np
import pytest

import kvgen
import oracle
from kvgen import Geometry
from tests.helpers import CANARY

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

DMA, LDG, TMA = st.STRATA_ENGINE_DMA, st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA


def _setup(n=20000, L=4, seed=31):
    # two disjoint halves of the device pool and of the host tier
    g = Geometry(L, 8, 128, 2, 1, 64, 2 * 25000, 2 * 400)
    rng = kvgen.rng_for(seed)
    half_p, half_c = g.num_pages // 2, g.num_chunks // 2
    qa = kvgen.make_requests(rng, [n, 777], g.P, g.C, half_p, half_c, offsets=True)
    qb = kvgen.make_requests(rng, [n - 5000, 1500], g.P, g.C, half_p, half_c, offsets=True)
    qb.dev_pages = (qb.dev_pages + half_p).astype(np.int32)
    qb.host_chunks = (qb.host_chunks + half_c).astype(np.int32)
    nb = g.num_pages * g.P * g.token_bytes
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    k = [torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda", generator=gen) for _ in range(g.L)]
    v = [torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda", generator=gen) for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    pool.host[:] = kvgen.random_bytes(rng, g.host_bytes)
    return g, qa, qb, k, v, pool


@pytest.mark.parametrize("ea,eb", [(DMA, DMA), (DMA, LDG), (LDG, DMA), (LDG, LDG), (TMA, DMA)])
@pytest.mark.parametrize("kinds", [("load", "offload"), ("load", "load"), ("offload", "offload")])
def test_two_operations_in_flight(kinds, ea, eb):
    g, qa, qb, k, v, pool = _setup()
    try:
        host0 = pool.host.copy()
        dev0k = [t.cpu().numpy() for t in k]
        dev0v = [t.cpu().numpy() for t in v]
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        # the device index lists must outlive the operations (include/strata.h): keep both alive
        reqs = [st.Requests.from_kvgen(qa), st.Requests.from_kvgen(qb)]
        torch.cuda.synchronize()
        for kind, r, eng, s in ((kinds[0], reqs[0], ea, sa), (kinds[1], reqs[1], eb, sb)):
            op = pool.load if kind == "load" else pool.offload
            op(r, stream=s, engine=eng)
        torch.cuda.synchronize()
        # expected: apply both (disjoint) operations to the pre-states with the oracle
        ek, ev_ = [a.copy() for a in dev0k], [a.copy() for a in dev0v]
        eh = host0.copy()
        for kind, q in ((kinds[0], qa), (kinds[1], qb)):
            if kind == "load":
                oracle.load(g, host0, ek, ev_, q, 0, g.L)
            else:
                oracle.offload(g, eh, dev0k, dev0v, q, 0, g.L)
        for l in range(g.L):
            assert np.array_equal(k[l].cpu().numpy(), ek[l]), f"K layer {l}"
            assert np.array_equal(v[l].cpu().numpy(), ev_[l]), f"V layer {l}"
        assert np.array_equal(pool.host, eh), "host tier"
    finally:
        pool.close()


@pytest.mark.slow
@pytest.mark.parametrize("load_engine", [TMA, LDG])
def test_load_keeps_the_link_beside_a_running_offload(load_engine):
    """A load and an offload of one pool in flight together (a serving engine loads the next batch's
    prefixes while it backs up finished ones): the offload paces itself while the load
    runs (the backup is the non-critical path), so the load keeps >= 85 % of its
    solo rate; both results stay bit-exact.  Without pacing the load fell to ~15 GB/s
    (profiles/r02/bidir/).  Both zero-copy load engines (the ring and the fused LDG kernel, the
    default for large loads) count themselves in the device-wide running-load counter the offload paces against."""
    L, n = 16, 32768
    g = Geometry(L, 8, 128, 2, 1, 64, 2 * 41000, 2 * 520)
    rng = kvgen.rng_for(41)
    half_p, half_c = g.num_pages // 2, g.num_chunks // 2
    qa = kvgen.make_requests(rng, [n], g.P, g.C, half_p, half_c)
    qb = kvgen.make_requests(rng, [n], g.P, g.C, half_p, half_c)
    qb.dev_pages = (qb.dev_pages + half_p).astype(np.int32)
    qb.host_chunks = (qb.host_chunks + half_c).astype(np.int32)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda") for _ in range(L)]
    v = [torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda") for _ in range(L)]
    pool = st.HostPool(num_layers=L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    try:
        kvgen.fill_random(pool.host, 5)
        ra, rb = st.Requests.from_kvgen(qa), st.Requests.from_kvgen(qb)
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        nbytes = 2 * L * n * g.token_bytes

        def timed(ops):
            torch.cuda.synchronize()
            evs = {}
            for name, fn, s in ops:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn(s)
                b.record(s)
                evs[name] = (a, b)
            torch.cuda.synchronize()
            return {name: nbytes / (a.elapsed_time(b) / 1e3) / 1e9 for name, (a, b) in evs.items()}

        load = ("load", lambda s: pool.load(ra, stream=s, engine=load_engine), sa)
        off = ("offload", lambda s: pool.offload(rb, stream=sb), sb)
        timed([load])
        solo = sorted(timed([load])["load"] for _ in range(3))[1]
        host_before = pool.host.copy()
        pre_k = [t.cpu().numpy() for t in k]
        pre_v = [t.cpu().numpy() for t in v]
        both = timed([load, off])
        print(f"load alone {solo:.1f} GB/s, beside the offload {both['load']:.1f}; offload {both['offload']:.1f}")
        assert both["load"] >= 0.85 * solo, both
        # bit-exact: the load's pages from host set A, the offload's chunks of host set B
        exp_host = host_before.copy()
        oracle.offload(g, exp_host, pre_k, pre_v, qb, 0, L)
        assert np.array_equal(pool.host, exp_host)
        for l in (0, L // 2, L - 1):
            ek, ev = pre_k[l].copy(), pre_v[l].copy()
            ek_l, ev_l = [None] * L, [None] * L
            ek_l[l], ev_l[l] = ek, ev
            oracle.load(g, host_before, ek_l, ev_l, qa, l, l + 1)
            assert np.array_equal(k[l].cpu().numpy(), ek) and np.array_equal(v[l].cpu().numpy(), ev)
    finally:
        pool.close()
