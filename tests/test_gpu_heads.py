"""GPU parity of host tiers read in a head slice and of head-major host chunks (R28):
every engine (TMA rings and the copy-engine path fall back to LDG where the layout leaves them no
long runs), both directions, bit-exact against the CPU oracle over whole buffers."""
import dataclasses

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.gpu_helpers import GpuCase, default_engine

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

ENGINES = [st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_TMA_BULK, st.STRATA_ENGINE_DMA,
           st.STRATA_ENGINE_DEFAULT]
SLICES = [(1, 8, 3), (2, 8, 4), (8, 8, 0), (2, 2, 0)]


def _run(g, q, engine, seed, l0=0, l1=None):
    l1 = g.L if l1 is None else l1
    c = GpuCase(g, q, seed=seed)
    try:
        c.pool.load(c.reqs, l0, l1, engine=engine)
        torch.cuda.synchronize()
        c.check_load(l0, l1)
        before = c.pool.host.copy()
        for t in c.k + c.v:
            t.copy_(torch.randint(0, 256, t.shape, dtype=torch.uint8, device="cuda"))
        c.pool.offload(c.reqs, l0, l1, engine=engine)
        torch.cuda.synchronize()
        assert np.array_equal(c.pool.host, c.expected_offload(before, l0, l1)), (engine, g)
        return c.pool.counters()["last_engine"]
    finally:
        c.close()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("head_major", [False, True])
@pytest.mark.parametrize("H,Ht,h0", SLICES)
def test_head_slice_small(engine, head_major, H, Ht, h0):
    g = Geometry(L=3, H=H, D=128, e=2, P=4, C=16, num_pages=200, num_chunks=48, Ht=Ht, h0=h0,
                 head_major=head_major)
    q = kvgen.make_requests(kvgen.rng_for(70 + h0), [300, 211, 7], g.P, g.C, g.num_pages, g.num_chunks,
                            offsets=True)
    _run(g, q, engine, seed=h0)


@pytest.mark.parametrize("head_major", [False, True])
@pytest.mark.parametrize("H,Ht,h0", [(1, 8, 5), (8, 8, 0)])
def test_head_slice_layer_sized_default_engine(head_major, H, Ht, h0):
    """>= 4 MiB per layer: the default engine is zero-copy: the ring engine where the tier has whole
    host rows (token-major, or one head per GPU), LDG for a head-major tier with several heads."""
    n = 9000 if H == 1 else 1200
    g = Geometry(L=2, H=H, D=128, e=2, P=1, C=64, num_pages=n + 2000, num_chunks=n // 64 + 20, Ht=Ht, h0=h0,
                 head_major=head_major)
    q = kvgen.make_requests(kvgen.rng_for(80), [n - 100, 90], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    assert 2 * sum(q.num_tokens) * g.token_bytes >= 4 << 20
    used = _run(g, q, st.STRATA_ENGINE_DEFAULT, seed=3)
    assert used == default_engine(g), used


@pytest.mark.parametrize("i", range(40))
def test_fuzz_head_slices(i):
    rng = kvgen.rng_for(7000 + i)
    Ht = int(rng.choice([2, 4, 8]))
    H = int(rng.choice([h for h in (1, 2, 4, 8) if h <= Ht]))
    h0 = int(rng.integers(0, Ht - H + 1))
    D = int(rng.choice([64, 128]))
    P = int(rng.choice([1, 4, 16]))
    C = int(rng.choice([1, 16, 64]))
    kv = int(rng.choice([1, 2]))
    ns = [int(rng.integers(0, 3 * C + 8)) for _ in range(int(rng.choice([1, 3])))]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + 4
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + 2
    g = Geometry(L=int(rng.choice([1, 3])), H=H, D=D, e=2, P=P, C=C, num_pages=num_pages, num_chunks=num_chunks,
                 kv=kv, Ht=Ht, h0=h0, head_major=bool(rng.integers(0, 2)))
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True)
    l0 = int(rng.integers(0, g.L))
    _run(g, q, ENGINES[i % len(ENGINES)], seed=i, l0=l0, l1=int(rng.integers(l0, g.L + 1)))


def test_tp_ranks_from_one_shared_tier():
    """Eight 'ranks' (one pool each, same device) register the SAME caller-owned head-major tier
    and load their own head: concatenated along heads they equal the full-head oracle load."""
    g_full = Geometry(L=2, H=8, D=128, e=2, P=1, C=64, num_pages=3000, num_chunks=50, Ht=8, head_major=True)
    q = kvgen.make_requests(kvgen.rng_for(90), [2500], g_full.P, g_full.C, g_full.num_pages, g_full.num_chunks)
    host = np.empty(g_full.host_bytes, np.uint8)
    host[:] = kvgen.random_bytes(kvgen.rng_for(91), g_full.host_bytes)
    import oracle
    from tests.helpers import CANARY
    ek = [np.full(g_full.layer_buffer_bytes, CANARY, np.uint8) for _ in range(g_full.L)]
    ev = [np.full(g_full.layer_buffer_bytes, CANARY, np.uint8) for _ in range(g_full.L)]
    oracle.load(g_full, host, ek, ev, q, 0, g_full.L)
    slots = g_full.num_pages * g_full.P
    got = {side: [[] for _ in range(g_full.L)] for side in (0, 1)}
    for r in range(8):
        g = dataclasses.replace(g_full, H=1, h0=r)
        nb = g.layer_buffer_bytes
        k = [torch.full((nb,), CANARY, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        v = [torch.full((nb,), CANARY, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        with st.HostPool(num_layers=g.L, num_heads=1, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                         k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks, host=host,
                         host_heads=8, head_begin=r, head_major=True) as pool:
            pool.load(st.Requests.from_kvgen(q))
            torch.cuda.synchronize()
        for l in range(g.L):
            got[0][l].append(k[l].cpu().numpy().reshape(slots, 1, -1))
            got[1][l].append(v[l].cpu().numpy().reshape(slots, 1, -1))
    for l in range(g_full.L):
        assert np.array_equal(np.concatenate(got[0][l], axis=1).reshape(-1), ek[l])
        assert np.array_equal(np.concatenate(got[1][l], axis=1).reshape(-1), ev[l])


@pytest.mark.slow
def test_llama70b_tp8_shared_tier_bench_config():
    """bench.py --config llama70b_tp8_shared in its launch configuration (default engine), rank 5's
    head: sampled layers byte for byte."""
    g = dataclasses.replace(kvgen.geometry("llama70b_tp8_shared"), h0=5)
    q = kvgen.make_requests(kvgen.rng_for(0), kvgen.CONFIGS["llama70b_tp8_shared"]["n"], g.P, g.C,
                            g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        c.pool.load(c.reqs)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == st.STRATA_ENGINE_LDG   # default for >= 16 MiB loads
        c.check_load(0, g.L, layers=[0, 41, 79])
        c.pool.load(c.reqs, engine=st.STRATA_ENGINE_TMA)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == st.STRATA_ENGINE_TMA
        c.check_load(0, g.L, layers=[5, 79])
    finally:
        c.close()


@pytest.mark.parametrize("group", [1, 2])
@pytest.mark.parametrize("H,Ht,h0", [(1, 8, 6), (2, 4, 1), (4, 4, 0)])
def test_head_major_strided_runs_dma(H, Ht, h0, group):
    """Consecutive host chunks of a head-major tier move as one strided copy per head and run
    (copy engines), with partial first / last chunks and a permuted tail; both directions."""
    g = Geometry(L=3, H=H, D=128, e=2, P=1, C=64, num_pages=12000, num_chunks=200, Ht=Ht, h0=h0,
                 head_major=True)
    rng = kvgen.rng_for(95)
    q = kvgen.make_requests(rng, [7000, 3000], g.P, g.C, g.num_pages, g.num_chunks, offsets=True,
                            chunk_frag="identity")
    hc = q.host_chunks.copy()
    hc[-20:] = rng.permutation(hc[-20:])
    q.host_chunks = hc
    c = GpuCase(g, q, seed=5)
    try:
        c.pool.load(c.reqs, engine=st.STRATA_ENGINE_DMA, layer_group=group)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == st.STRATA_ENGINE_DMA
        c.check_load(0, g.L)
        before = c.pool.host.copy()
        for t in c.k + c.v:
            t.copy_(torch.randint(0, 256, t.shape, dtype=torch.uint8, device="cuda"))
        c.pool.offload(c.reqs, engine=st.STRATA_ENGINE_DMA, layer_group=group)
        torch.cuda.synchronize()
        assert np.array_equal(c.pool.host, c.expected_offload(before, 0, g.L))
    finally:
        c.close()


def test_shared_tier_outlives_first_pool():
    """Two pools over ONE caller tier alive at once (round-1 advice): closing the pool that
    registered it first must not unregister it under the second, whose loads keep matching the
    oracle; a third pool whose range only partly overlaps the shared registration is refused."""
    g_full = Geometry(L=2, H=2, D=128, e=2, P=1, C=64, num_pages=3000, num_chunks=50, Ht=2, head_major=True)
    q = kvgen.make_requests(kvgen.rng_for(92), [2500], g_full.P, g_full.C, g_full.num_pages, g_full.num_chunks)
    host = np.empty(g_full.host_bytes + 4096, np.uint8)
    tier = host[:g_full.host_bytes]
    tier[:] = kvgen.random_bytes(kvgen.rng_for(93), g_full.host_bytes)
    import oracle
    from tests.helpers import CANARY
    ek = [np.full(g_full.layer_buffer_bytes, CANARY, np.uint8) for _ in range(g_full.L)]
    ev = [np.full(g_full.layer_buffer_bytes, CANARY, np.uint8) for _ in range(g_full.L)]
    oracle.load(g_full, tier, ek, ev, q, 0, g_full.L)
    slots = g_full.num_pages * g_full.P
    pools, bufs = [], []
    for r in range(2):
        g = dataclasses.replace(g_full, H=1, h0=r)
        nb = g.layer_buffer_bytes
        k = [torch.full((nb,), CANARY, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        v = [torch.full((nb,), CANARY, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        pools.append(st.HostPool(num_layers=g.L, num_heads=1, head_dim=g.D, elem_bytes=g.e, page_size=g.P,
                                 chunk_tokens=g.C, k_ptrs=k, v_ptrs=v, num_pages=g.num_pages,
                                 num_chunks=g.num_chunks, host=tier, host_heads=2, head_begin=r, head_major=True))
        bufs.append((k, v))
    try:
        # a range that straddles the shared registration's end cannot share it
        with pytest.raises(st.StrataError):
            k, v = bufs[0]
            st.HostPool(num_layers=g_full.L, num_heads=1, head_dim=g_full.D, elem_bytes=g_full.e, page_size=1,
                        chunk_tokens=g_full.C, k_ptrs=k, v_ptrs=v, num_pages=g_full.num_pages,
                        num_chunks=g_full.num_chunks, host=host[4096:4096 + g_full.host_bytes], host_heads=2,
                        head_begin=0, head_major=True)
        pools[0].close()
        for _ in range(3):   # loads through the second pool after the first closed
            pools[1].load(st.Requests.from_kvgen(q))
        torch.cuda.synchronize()
        k, v = bufs[1]
        for l in range(g_full.L):
            want_k = ek[l].reshape(slots, 2, -1)[:, 1].reshape(-1)
            want_v = ev[l].reshape(slots, 2, -1)[:, 1].reshape(-1)
            assert np.array_equal(k[l].cpu().numpy(), want_k)
            assert np.array_equal(v[l].cpu().numpy(), want_v)
    finally:
        for p in pools:
            p.close()
