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
