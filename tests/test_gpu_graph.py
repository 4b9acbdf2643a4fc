"""strata_load inside CUDA graph capture (torch.cuda.graph): request tables travel in kernel
parameters and no call synchronises, so a load is capturable and replays bit-exactly, reading the
host tier as it is at replay time."""
import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.gpu_helpers import GpuCase

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402


VARIANTS = {
    "gqa": Geometry(4, 8, 128, 2, 1, 64, 12000, 200),                      # 8K tokens: 32 MiB per layer
    "mla": Geometry(4, 1, 576, 2, 1, 64, 12000, 200, kv=1),                # R27
    "head_major_slice": Geometry(4, 1, 128, 2, 1, 64, 12000, 200, Ht=8, h0=5, head_major=True),   # R28
    "narrow": Geometry(4, 1, 72, 1, 1, 256, 12000, 60),                     # R29
}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("engine", [st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_DMA])
def test_load_replays_from_cuda_graph(engine, variant):
    g = VARIANTS[variant]
    q = kvgen.make_requests(kvgen.rng_for(6), [8000, 1500], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    c = GpuCase(g, q)
    try:
        s = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            c.pool.load(c.reqs, engine=engine, stream=s)      # warm-up outside capture
        torch.cuda.synchronize()
        for t in c.k + c.v:
            t.fill_(0xA5)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            c.pool.load(c.reqs, engine=engine, stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert all(bool((t == 0xA5).all()) for t in c.k + c.v), "capture must not execute"
        graph.replay()
        torch.cuda.synchronize()
        c.check_load(0, g.L)
        # the graph reads the host tier at replay time
        c.pool.host[: g.host_bytes] = kvgen.random_bytes(kvgen.rng_for(99), g.host_bytes)
        graph.replay()
        torch.cuda.synchronize()
        c.check_load(0, g.L)
    finally:
        c.close()


@pytest.mark.parametrize("engine", [st.STRATA_ENGINE_DEFAULT, st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_DMA])
def test_captured_load_layer_events_signal_every_replay(engine):
    """A captured load's per-layer events (round-1 advice): every replay signals them (external event
    nodes), so a consumer OUTSIDE the graph waits on layer l of the latest replay; a consumer captured
    INTO the same graph on a forked stream waits through a graph edge; the captured ticket outlives
    the 8-slot event ring; strata_layer_elapsed_ms times the latest replay."""
    g = VARIANTS["gqa"]
    q = kvgen.make_requests(kvgen.rng_for(7), [8000, 1500], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    c = GpuCase(g, q)
    try:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c.pool.load(c.reqs, engine=engine, stream=s)
        torch.cuda.synchronize()
        snap_in = torch.empty_like(c.v[2])
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        with torch.cuda.graph(graph, stream=s):
            cur = torch.cuda.current_stream()
            side.wait_stream(cur)                       # fork BEFORE the load: side depends only on layer 2
            ticket = c.pool.load(c.reqs, engine=engine, stream=cur)
            c.pool.wait_layer(ticket, 2, side)
            with torch.cuda.stream(side):
                snap_in.copy_(c.v[2])
            cur.wait_stream(side)
        torch.cuda.synchronize()
        # ring slots reused by 9 live loads: the captured ticket stays valid
        for _ in range(9):
            c.pool.load(c.reqs, engine=engine, stream=s)
        torch.cuda.synchronize()
        consumer = torch.cuda.Stream()
        snaps = [torch.empty_like(c.k[l]) for l in range(g.L)]
        for rep in range(2):
            for t in c.k + c.v:
                t.fill_(0xA5)
            snap_in.fill_(0)
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                graph.replay()
            for l in range(g.L):
                c.pool.wait_layer(ticket, l, consumer)
                with torch.cuda.stream(consumer):
                    snaps[l].copy_(c.k[l])
            torch.cuda.synchronize()
            ms = [c.pool.layer_elapsed_ms(ticket, l) for l in range(g.L)]
            assert all(b >= a for a, b in zip(ms, ms[1:])) and ms[0] > 0, ms
            for l in range(g.L):
                ek, ev = c.expected_load_layer(l)
                assert np.array_equal(snaps[l].cpu().numpy(), ek), f"replay {rep}: outside consumer, layer {l}"
            assert np.array_equal(snap_in.cpu().numpy(), c.expected_load_layer(2)[1]), f"replay {rep}: in-graph consumer"
    finally:
        c.close()
