"""GPU parity: strata_load / strata_offload through the C ABI, bit-exact against the CPU oracle on
the same seeded inputs.  Every comparison covers the WHOLE destination buffer, so it
checks both "every valid byte landed at page_table[token]" and "nothing else was touched"."""
import itertools

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.gpu_helpers import GpuCase, nhd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

ENGINES = [st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_TMA_BULK, st.STRATA_ENGINE_DMA]


def _sync():
    torch.cuda.synchronize()


# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("engine", ENGINES + [st.STRATA_ENGINE_DEFAULT])
def test_tiny_load_offload(engine):
    g = kvgen.geometry("tiny")
    q = kvgen.make_requests(kvgen.rng_for(0), kvgen.CONFIGS["tiny"]["n"], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        stream = torch.cuda.Stream()
        c.pool.load(c.reqs, stream=stream, engine=engine)
        _sync()
        c.check_load(0, g.L)
        before = c.pool.host.copy()
        # offload the (now loaded) pages into the same chunks: host tier must be unchanged
        c.pool.offload(c.reqs, stream=stream, engine=engine)
        _sync()
        assert np.array_equal(c.pool.host, before)
    finally:
        c.close()


def _fuzz_params(i):
    rng = kvgen.rng_for(1000 + i)
    L = int(rng.choice([1, 2, 3, 5]))
    H = int(rng.choice([1, 2, 8]))
    D = int(rng.choice([64, 128, 256]))
    e = int(rng.choice([1, 2]))
    P = int(rng.choice([1, 2, 4, 8, 16, 32, 64]))
    C = int(rng.choice([1, 16, 64, 256]))
    R = int(rng.choice([1, 2, 8]))
    ns = [int(rng.integers(0, 3 * C + 8)) for _ in range(R)]
    l0 = int(rng.integers(0, L))
    l1 = int(rng.integers(l0, L + 1))
    if rng.random() < 0.2:
        l0, l1 = 0, L
    ctas = int(rng.choice([0, 1, 2, 4, 16, 148]))
    engine = ENGINES[i % len(ENGINES)]
    frag = "churn" if rng.random() < 0.3 else "perm"
    layout = rng.choice(["nhd", "hnd", "padded"])
    group = int(rng.choice([0, 1, 2, 3])) if engine == st.STRATA_ENGINE_DMA else 0
    return dict(rng=rng, L=L, H=H, D=D, e=e, P=P, C=C, ns=ns, l0=l0, l1=l1, ctas=ctas, engine=engine,
                frag=frag, layout=str(layout), group=group)


def _fuzz_case(i):
    f = _fuzz_params(i)
    rng, P, C, ns = f["rng"], f["P"], f["C"], f["ns"]
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + int(rng.integers(1, 9))
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + int(rng.integers(1, 4))
    if f["frag"] == "churn":
        num_pages = max(num_pages, 64)
    g = Geometry(f["L"], f["H"], f["D"], f["e"], P, C, num_pages, num_chunks)
    tok = g.H * g.D * g.e
    if f["layout"] == "hnd":
        strides = (g.H * P * g.D * g.e, g.D * g.e, P * g.D * g.e)
    elif f["layout"] == "padded":
        strides = (P * (tok + 32) + 48, tok + 32, g.D * g.e)
    else:
        strides = None
    kw = dict(frag=f["frag"]) if f["frag"] != "churn" else dict(frag="perm")
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True, **kw)
    if f["frag"] == "churn":
        pages = kvgen.churn_free_list(rng, num_pages, P, rounds=50, lo=1, hi=4 * P)[: q.dev_pages.size]
        q.dev_pages = pages.astype(np.int32)
    return f, g, q, strides


@pytest.mark.parametrize("i", range(150))
def test_fuzz_load(i):
    f, g, q, strides = _fuzz_case(i)
    c = GpuCase(g, q, strides=strides, seed=i)
    try:
        c.pool.load(c.reqs, f["l0"], f["l1"], engine=f["engine"], num_ctas=f["ctas"], layer_group=f["group"])
        _sync()
        c.check_load(f["l0"], f["l1"])
    finally:
        c.close()


@pytest.mark.parametrize("i", range(150, 300))
def test_fuzz_offload(i):
    f, g, q, strides = _fuzz_case(i)
    c = GpuCase(g, q, strides=strides, seed=i, dev_fill="random")
    try:
        before = c.pool.host.copy()
        c.pool.offload(c.reqs, f["l0"], f["l1"], engine=f["engine"], num_ctas=f["ctas"], layer_group=f["group"])
        _sync()
        exp = c.expected_offload(before, f["l0"], f["l1"])
        got = c.pool.host
        if not np.array_equal(got, exp):
            bad = np.flatnonzero(got != exp)
            raise AssertionError(f"{bad.size} host bytes differ, first at {bad[0]}; case {f}")
    finally:
        c.close()


@pytest.mark.parametrize("engine", ENGINES)
def test_many_requests_split_launches(engine):
    """> 128 requests per call: the planner splits them across launches per layer."""
    rng = kvgen.rng_for(77)
    ns = [int(x) for x in rng.integers(0, 40, size=300)]
    g = Geometry(2, 2, 64, 2, 4, 16, sum(kvgen.pages_needed(3, n, 4) for n in ns) + 4,
                 sum(kvgen.chunks_needed(15, n, 16) for n in ns) + 2)
    q = kvgen.make_requests(rng, ns, g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    c = GpuCase(g, q)
    try:
        c.pool.load(c.reqs, engine=engine)
        _sync()
        c.check_load(0, g.L)
    finally:
        c.close()


@pytest.mark.parametrize("engine", ENGINES)
def test_special_float_payloads(engine):
    """fp16/bf16 NaN payloads, infinities and -0.0 move bit-exactly (R9)."""
    g = Geometry(2, 2, 64, 2, 1, 16, 64, 4)
    q = kvgen.make_requests(kvgen.rng_for(5), [48], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q, host_fill="none")
    try:
        pats = np.array([0x7E01, 0xFE7F, 0x8000, 0x7FC1, 0xFFFF, 0x7C01, 0x0001, 0x8001,
                         0x7C00, 0xFC00, 0x7F80, 0xFF80, 0x7FBF, 0x0000, 0x3C00, 0xBC00], np.uint16)
        c.pool.host[:] = np.tile(pats, g.host_bytes // 32).view(np.uint8)
        c.pool.load(c.reqs, engine=engine)
        _sync()
        c.check_load(0, g.L)
    finally:
        c.close()


@pytest.mark.parametrize("engine", [st.STRATA_ENGINE_DEFAULT, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_LDG])
@pytest.mark.parametrize("H,D,e,P", [(3, 16, 2, 1), (5, 16, 2, 4), (1, 40, 2, 1), (3, 64, 2, 16), (7, 16, 2, 1),
                                     (1, 24, 2, 2), (9, 16, 2, 1), (3, 32, 1, 8)])
@pytest.mark.parametrize("strides", ["nhd", "hnd"])
def test_rows_with_odd_vector_counts(engine, H, D, e, P, strides):
    """Rows of 3, 5, 6, 7, 9, 10 ... 16-byte vectors (not a power of two, fewer than 32): the ring
    engine moves 32 / vpt rows per warp instruction, and with 64-row pieces a group straddles row 32
    (two address slots per lane).  Partial chunks and pages, several requests, both directions."""
    g = Geometry(3, H, D, e, P, 64, -(-1400 // P) + 8, 40)
    tok = g.token_bytes
    st_ = (g.H * P * g.D * g.e, g.D * g.e, P * g.D * g.e) if strides == "hnd" else None
    q = kvgen.make_requests(kvgen.rng_for(13 + H + D), [700, 129, 64, 1], g.P, g.C, g.num_pages, g.num_chunks,
                            offsets=True)
    c = GpuCase(g, q, strides=st_, seed=H * D)
    try:
        c.pool.load(c.reqs, engine=engine)
        _sync()
        c.check_load(0, g.L)
        before = c.pool.host.copy()
        for t in c.k + c.v:
            t.copy_(torch.randint(0, 256, t.shape, dtype=torch.uint8, device="cuda"))
        c.pool.offload(c.reqs, 1, 3, engine=engine)
        _sync()
        assert np.array_equal(c.pool.host, c.expected_offload(before, 1, 3)), (tok, engine)
    finally:
        c.close()


@pytest.mark.parametrize("direction", ["load", "offload"])
@pytest.mark.parametrize("group", [1, 2, 4])
def test_dma_engine_multi_piece(direction, group):
    """STRATA_ENGINE_DMA with layers larger than one 64 MiB staging slot: several pieces per layer
    alternate between the two slots, within and across layers; partial first/last chunks; layer
    groups (G layers of a chunk per copy, ragged last group)."""
    g = Geometry(6, 8, 128, 2, 1, 64, 40960, 560)
    rng = kvgen.rng_for(21)
    q = kvgen.make_requests(rng, [20000, 13000, 77], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    c = GpuCase(g, q, dev_fill="canary" if direction == "load" else "random")
    try:
        if direction == "load":
            t = c.pool.load(c.reqs, 1, 6, engine=st.STRATA_ENGINE_DMA, layer_group=group)
            _sync()
            c.check_load(1, 6)
            done = [c.pool.layer_elapsed_ms(t, l) for l in range(1, 6)]
            assert all(b >= a for a, b in zip(done, done[1:])), done
        else:
            before = c.pool.host.copy()
            c.pool.offload(c.reqs, 0, 5, engine=st.STRATA_ENGINE_DMA, layer_group=group)
            _sync()
            assert np.array_equal(c.pool.host, c.expected_offload(before, 0, 5))
    finally:
        c.close()


@pytest.mark.parametrize("edge,ordered,streams", [("1", "0", "4"), ("1", "1", "4"), ("4", "1", "4"), ("16", "0", "3"),
                                                  ("4", "1", "1"), ("4", "0", "8")])
@pytest.mark.parametrize("direction", ["load", "offload"])
def test_dma_engine_piece_schedule(direction, edge, ordered, streams, monkeypatch):
    """The DMA engine's piece schedule (edge pieces of the first / last layer, the per-piece copy
    barrier, the number of copy streams) changes only timing: the result stays the oracle's and
    layer events stay ordered."""
    monkeypatch.setenv("STRATA_DMA_EDGE_SPLIT", edge)
    monkeypatch.setenv("STRATA_DMA_ORDERED", ordered)
    monkeypatch.setenv("STRATA_COPY_STREAMS", streams)
    g = Geometry(4, 8, 128, 2, 1, 64, 40960, 560)
    rng = kvgen.rng_for(22)
    q = kvgen.make_requests(rng, [21000, 12000, 300], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    c = GpuCase(g, q, dev_fill="canary" if direction == "load" else "random")
    try:
        if direction == "load":
            t = c.pool.load(c.reqs, 0, 4, engine=st.STRATA_ENGINE_DMA)
            _sync()
            c.check_load(0, 4)
            done = [c.pool.layer_elapsed_ms(t, l) for l in range(0, 4)]
            assert all(b >= a for a, b in zip(done, done[1:])), done
        else:
            before = c.pool.host.copy()
            c.pool.offload(c.reqs, 0, 4, engine=st.STRATA_ENGINE_DMA)
            _sync()
            assert np.array_equal(c.pool.host, c.expected_offload(before, 0, 4))
    finally:
        c.close()


@pytest.mark.parametrize("kv", [2, 1])
@pytest.mark.parametrize("strided", ["1", "0"])
@pytest.mark.parametrize("group", [1, 3])
@pytest.mark.parametrize("direction", ["load", "offload"])
def test_dma_strided_chunk_runs(direction, group, strided, kv, monkeypatch):
    """Consecutive host chunk ids become one strided copy per run (cudaMemcpy2DAsync): requests
    with partial first / last chunks, runs broken by the request boundary and by a permuted tail,
    layer groups; the result stays the oracle's."""
    monkeypatch.setenv("STRATA_DMA_STRIDED", strided)
    g = Geometry(5, 8, 128, 2, 1, 64, 40960, 700, kv=kv)
    rng = kvgen.rng_for(23)
    q = kvgen.make_requests(rng, [20000, 9000, 130], g.P, g.C, g.num_pages, g.num_chunks, offsets=True,
                            chunk_frag="identity")
    hc = q.host_chunks.copy()
    hc[-40:] = rng.permutation(hc[-40:])          # a permuted tail: short runs and singles
    q.host_chunks = hc
    c = GpuCase(g, q, dev_fill="canary" if direction == "load" else "random")
    try:
        if direction == "load":
            c.pool.load(c.reqs, 0, 5, engine=st.STRATA_ENGINE_DMA, layer_group=group)
            _sync()
            c.check_load(0, 5)
        else:
            before = c.pool.host.copy()
            c.pool.offload(c.reqs, 0, 5, engine=st.STRATA_ENGINE_DMA, layer_group=group)
            _sync()
            assert np.array_equal(c.pool.host, c.expected_offload(before, 0, 5))
    finally:
        c.close()


def test_dma_engine_needs_host_list():
    g = kvgen.geometry("tiny")
    q = kvgen.make_requests(kvgen.rng_for(0), [64], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        x = c.reqs.xfer(0, g.L, engine=st.STRATA_ENGINE_DMA)
        x.host_chunks_host = None
        with pytest.raises(st.StrataError) as e:
            st.strata_load(c.pool.handle, x)
        assert e.value.code == st._lib.STRATA_ERR_INVALID_ARG
    finally:
        c.close()


@pytest.mark.parametrize("variant", ["gqa", "mla", "head_major_slice", "token_major_slice", "narrow"])
def test_baselines_match_oracle(variant):
    """The copy-engine baselines produce the same bytes (a library-routine pin on hardware), on the
    paper's GQA pools and on every pool variant (R27-R29)."""
    g = {"gqa": Geometry(3, 2, 64, 2, 4, 16, 96, 24),
         "mla": Geometry(3, 1, 576, 2, 4, 16, 96, 24, kv=1),
         "head_major_slice": Geometry(3, 2, 64, 2, 4, 16, 96, 24, Ht=6, h0=3, head_major=True),
         "token_major_slice": Geometry(3, 2, 64, 2, 4, 16, 96, 24, Ht=4, h0=1),
         "narrow": Geometry(3, 3, 10, 2, 4, 16, 96, 24)}[variant]
    rng = kvgen.rng_for(8)
    q = kvgen.make_requests(rng, [37, 100, 5], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    for fn in (st.strata_baseline_memcpy_pages,):
        c = GpuCase(g, q)
        try:
            s = torch.cuda.Stream()
            n = fn(c.pool.handle, c.reqs.xfer(0, g.L, host_lists=True), st.STRATA_H2D, s)
            assert n > 0
            _sync()
            c.check_load(0, g.L)
            before = c.pool.host.copy()
            for t in c.k + c.v:
                t.random_(0, 256)
            fn(c.pool.handle, c.reqs.xfer(1, 3, host_lists=True), st.STRATA_D2H, s)
            _sync()
            assert np.array_equal(c.pool.host, c.expected_offload(before, 1, 3))
        finally:
            c.close()


# ------------------------------------------------------------------------------------------------
# Per-layer completion events: a consumer that waits on ev[l] and immediately checksums layer l
# must see the final bytes (an early signal would expose canaries).
@pytest.mark.parametrize("engine", ENGINES)
def test_layer_events_order_consumer(engine):
    g = Geometry(8, 8, 128, 2, 1, 64, 8192 + 64, 140)
    q = kvgen.make_requests(kvgen.rng_for(3), [8192], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        io = torch.cuda.Stream()
        consumer = torch.cuda.Stream()
        sums = []
        ticket = c.pool.load(c.reqs, stream=io, engine=engine, num_ctas=2)
        with torch.cuda.stream(consumer):
            for l in range(g.L):
                c.pool.wait_layer(ticket, l, consumer)
                sums.append((c.k[l].view(torch.int64).sum(), c.v[l].view(torch.int64).sum()))
        _sync()
        for l in range(g.L):
            ek, ev = c.expected_load_layer(l)
            assert int(sums[l][0]) == int(ek.view(np.int64).sum()), f"layer {l} K consumed early"
            assert int(sums[l][1]) == int(ev.view(np.int64).sum()), f"layer {l} V consumed early"
        t = [c.pool.layer_elapsed_ms(ticket, l) for l in range(g.L)]
        assert all(b >= a for a, b in zip(t, t[1:])), t   # layers complete in order
        assert t[0] > 0
    finally:
        c.close()


def test_event_api_errors():
    g = kvgen.geometry("tiny")
    q = kvgen.make_requests(kvgen.rng_for(0), [64], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        with pytest.raises(st.StrataError) as e:
            c.pool.layer_event(0, 0)           # nothing issued yet
        assert e.value.code == st._lib.STRATA_ERR_STALE_TICKET
        t1 = c.pool.load(c.reqs, 1, 2)
        with pytest.raises(st.StrataError) as e:
            c.pool.layer_event(t1, 0)          # layer outside [1,2)
        assert e.value.code == st._lib.STRATA_ERR_INVALID_ARG
        assert c.pool.layer_event(t1, 1) != 0
        for _ in range(8):
            c.pool.load(c.reqs, 0, 1)
        with pytest.raises(st.StrataError) as e:
            c.pool.layer_event(t1, 1)          # ring of 8 overwritten
        assert e.value.code == st._lib.STRATA_ERR_STALE_TICKET
        t_empty = c.pool.load(c.reqs, 1, 1)    # empty layer range: successful no-op
        assert t_empty > t1
        _sync()
    finally:
        c.close()


# ------------------------------------------------------------------------------------------------
# Negative cases (DESIGN.md §2 error behaviour).
def test_validate_rejects_bad_indices_and_duplicates():
    g = kvgen.geometry("tiny")
    rng = kvgen.rng_for(1)
    q = kvgen.make_requests(rng, [100, 60], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q, flags=st.STRATA_VALIDATE)
    try:
        c.pool.load(c.reqs)   # valid tables pass validation
        _sync()
        c.check_load(0, g.L)
        bad = kvgen.make_requests(rng, [100, 60], g.P, g.C, g.num_pages, g.num_chunks)
        bad.dev_pages[3] = g.num_pages          # out of range
        with pytest.raises(st.StrataError) as e:
            c.pool.load(st.Requests.from_kvgen(bad))
        assert e.value.code == st._lib.STRATA_ERR_INDEX_RANGE
        dup = kvgen.make_requests(rng, [100, 60], g.P, g.C, g.num_pages, g.num_chunks)
        dup.dev_pages[-1] = dup.dev_pages[0]    # two tokens -> one slot
        with pytest.raises(st.StrataError) as e:
            c.pool.load(st.Requests.from_kvgen(dup))
        assert e.value.code == st._lib.STRATA_ERR_DUPLICATE
        dupc = kvgen.make_requests(rng, [100, 60], g.P, g.C, g.num_pages, g.num_chunks)
        dupc.host_chunks[-1] = dupc.host_chunks[0]
        c.pool.load(st.Requests.from_kvgen(dupc))   # duplicate SOURCES are legal for a load
        with pytest.raises(st.StrataError) as e:
            c.pool.offload(st.Requests.from_kvgen(dupc))   # ... but not for an offload
        assert e.value.code == st._lib.STRATA_ERR_DUPLICATE
        _sync()
    finally:
        c.close()


def test_host_side_argument_errors():
    g = kvgen.geometry("tiny")
    q = kvgen.make_requests(kvgen.rng_for(2), [64], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        x = c.reqs.xfer(0, g.L + 1)
        with pytest.raises(st.StrataError) as e:
            st.strata_load(c.pool.handle, x)
        assert e.value.code == st._lib.STRATA_ERR_INVALID_ARG
        x = c.reqs.xfer(0, g.L)
        x.dev_pages_len = 1                     # list too short for 64 tokens at P=16
        with pytest.raises(st.StrataError) as e:
            st.strata_load(c.pool.handle, x)
        assert e.value.code == st._lib.STRATA_ERR_INDEX_RANGE
        c.reqs.page_offset[0] = g.P             # offset outside [0, P)
        with pytest.raises(st.StrataError) as e:
            c.pool.load(c.reqs)
        assert e.value.code == st._lib.STRATA_ERR_INVALID_ARG
        c.reqs.page_offset[0] = 0
        x = c.reqs.xfer(0, g.L)
        x.dev_pages = None
        with pytest.raises(st.StrataError) as e:
            st.strata_load(c.pool.handle, x)
        assert e.value.code == st._lib.STRATA_ERR_INVALID_ARG
    finally:
        c.close()


def test_caller_owned_host_memory():
    """host_base != NULL: the library registers caller memory (and leaves it allocated)."""
    g = kvgen.geometry("tiny")
    q = kvgen.make_requests(kvgen.rng_for(4), [333], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    host = np.empty(g.host_bytes + 64, np.uint8)
    off = (-host.ctypes.data) % 64
    mine = host[off: off + g.host_bytes]
    mine[:] = kvgen.random_bytes(kvgen.rng_for(9), g.host_bytes)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.full((nb,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.full((nb,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    import oracle
    with st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                     k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks, host=mine) as pool:
        assert pool.host_addr == mine.ctypes.data
        pool.load(st.Requests.from_kvgen(q))
        _sync()
        ek = [np.full(nb, 0xA5, np.uint8) for _ in range(g.L)]
        ev = [np.full(nb, 0xA5, np.uint8) for _ in range(g.L)]
        oracle.load(g, mine, ek, ev, q, 0, g.L)
        for l in range(g.L):
            assert np.array_equal(k[l].cpu().numpy(), ek[l])
            assert np.array_equal(v[l].cpu().numpy(), ev[l])
    assert mine.sum() >= 0   # still allocated and readable after unregister


# ------------------------------------------------------------------------------------------------
# Full-size configs (BASELINE.json), in the launch configuration bench.py times.
@pytest.mark.slow
@pytest.mark.parametrize("P,engine", [(1, st.STRATA_ENGINE_DEFAULT), (16, st.STRATA_ENGINE_DEFAULT),
                                      (1, st.STRATA_ENGINE_TMA), (16, st.STRATA_ENGINE_TMA)])
def test_llama8b_32k_full(P, engine):
    """Every byte of all 32 layers, in bench.py's launch configuration (default engine and quota:
    the zero-copy LDG engine, 2 CTAs x 1024 threads, one fused launch) and with the zero-copy ring
    engine at its default 2-CTA quota."""
    g = kvgen.geometry("llama8b_32k", P=P)
    q = kvgen.make_requests(kvgen.rng_for(0), [32768], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        c.pool.load(c.reqs, engine=engine)
        _sync()
        c.check_load(0, g.L)
        used = c.pool.counters()["last_engine"]
        assert used == (st.STRATA_ENGINE_LDG if engine == st.STRATA_ENGINE_DEFAULT else engine)
    finally:
        c.close()


@pytest.mark.slow
def test_llama70b_tp8_rank_slice_load_offload():
    g = kvgen.geometry("llama70b_tp8")
    q = kvgen.make_requests(kvgen.rng_for(0), [131072], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        c.pool.load(c.reqs)
        _sync()
        c.check_load(0, g.L, layers=[0, 1, 39, 78, 79])
        # offload back into fresh chunks and compare sampled chunks with the oracle
        q2 = kvgen.make_requests(kvgen.rng_for(1), [131072], g.P, g.C, g.num_pages, g.num_chunks)
        q2.dev_pages, q2.page_start, q2.page_offset = q.dev_pages, q.page_start, q.page_offset
        c2_reqs = st.Requests.from_kvgen(q2)
        before = c.pool.host.copy()
        c.pool.offload(c2_reqs)
        _sync()
        c.q = q2
        exp = c.expected_offload(before, 0, g.L)
        assert np.array_equal(c.pool.host, exp)
    finally:
        c.close()


@pytest.mark.slow
def test_qwen14b_batch8_sampled_layers():
    g = kvgen.geometry("qwen14b_batch8")
    q = kvgen.make_requests(kvgen.rng_for(0), kvgen.CONFIGS["qwen14b_batch8"]["n"], g.P, g.C, g.num_pages,
                            g.num_chunks)
    c = GpuCase(g, q)
    try:
        c.pool.load(c.reqs)
        _sync()
        c.check_load(0, g.L, layers=[0, 23, 47])
    finally:
        c.close()
