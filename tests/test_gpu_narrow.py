"""GPU parity of pools whose rows, strides or bases are not 16-byte multiples (reading R29;
SURVEY.md §8f "an fp8 KV scalar fallback for S_tok % 16 != 0"): the narrow LDG kernel (8 / 4 / 2 /
1-byte words) and the copy-engine path over it, every engine request (TMA falls back), both
directions, bit-exact against the byte-granular oracle over whole buffers."""
import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.gpu_helpers import GpuCase

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

ENGINES = [st.STRATA_ENGINE_DEFAULT, st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_TMA_BULK,
           st.STRATA_ENGINE_DMA]
SHAPES = [(1, 72, 1), (3, 10, 2), (1, 25, 2), (3, 3, 1), (2, 100, 1)]   # (H, D, e): 72 / 60 / 50 / 9 / 200 B


def _run(g, q, engine, strides=None, seed=0):
    c = GpuCase(g, q, strides=strides, seed=seed)
    try:
        c.pool.load(c.reqs, engine=engine)
        torch.cuda.synchronize()
        c.check_load(0, g.L)
        before = c.pool.host.copy()
        for t in c.k + c.v:
            t.copy_(torch.randint(0, 256, t.shape, dtype=torch.uint8, device="cuda"))
        c.pool.offload(c.reqs, engine=engine)
        torch.cuda.synchronize()
        assert np.array_equal(c.pool.host, c.expected_offload(before, 0, g.L)), (engine, g)
    finally:
        c.close()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("kv", [2, 1])
@pytest.mark.parametrize("H,D,e", SHAPES)
def test_narrow_rows(engine, kv, H, D, e):
    g = Geometry(L=3, H=H, D=D, e=e, P=4, C=16, num_pages=200, num_chunks=48, kv=kv)
    q = kvgen.make_requests(kvgen.rng_for(101 + D), [300, 211, 7], g.P, g.C, g.num_pages, g.num_chunks,
                            offsets=True)
    _run(g, q, engine, seed=D)


@pytest.mark.parametrize("engine", [st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_DMA])
@pytest.mark.parametrize("layout", ["hnd", "padded", "head_major_slice"])
def test_narrow_layouts(engine, layout):
    H, D, e, P = 3, 10, 2, 4
    if layout == "head_major_slice":
        g = Geometry(L=2, H=2, D=D, e=e, P=P, C=16, num_pages=200, num_chunks=48, Ht=5, h0=2, head_major=True)
        strides = None
    else:
        g = Geometry(L=2, H=H, D=D, e=e, P=P, C=16, num_pages=200, num_chunks=48)
        tok = g.token_bytes
        strides = (H * P * D * e, D * e, P * D * e) if layout == "hnd" else (P * (tok + 6) + 10, tok + 6, D * e)
    q = kvgen.make_requests(kvgen.rng_for(111), [400, 33], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    _run(g, q, engine, strides=strides, seed=3)


@pytest.mark.parametrize("C", [64, 256])
def test_narrow_layer_sized_default_engine(C):
    """>= 4 MiB per layer of 72-byte fp8 rows: the default engine is zero-copy in both directions —
    the ring engine's narrow-word path for loads, the narrow LDG kernel for offloads (the copy
    engines run only when a caller asks for STRATA_ENGINE_DMA)."""
    g = Geometry(L=2, H=1, D=72, e=1, P=1, C=C, num_pages=40000, num_chunks=38400 // C)
    q = kvgen.make_requests(kvgen.rng_for(121), [32000], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q, seed=4)
    try:
        c.pool.load(c.reqs)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == st.STRATA_ENGINE_TMA
        c.check_load(0, g.L)
        before = c.pool.host.copy()
        for t in c.k + c.v:
            t.copy_(torch.randint(0, 256, t.shape, dtype=torch.uint8, device="cuda"))
        c.pool.offload(c.reqs)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == st.STRATA_ENGINE_LDG
        assert np.array_equal(c.pool.host, c.expected_offload(before, 0, g.L))
    finally:
        c.close()
