"""GPU parity of single-buffer (MLA latent) pools, STRATA_POOL_SINGLE_KV (reading R27):
every engine, both directions, bit-exact against the CPU oracle with KV = 1 over whole buffers
(the V buffers the library never sees must keep their canary)."""
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

ENGINES = [st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_TMA_BULK, st.STRATA_ENGINE_DMA]


def _g(L, H, D, P, C, num_pages, num_chunks, e=2):
    return Geometry(L, H, D, e, P, C, num_pages, num_chunks, kv=1)


@pytest.mark.parametrize("engine", ENGINES + [st.STRATA_ENGINE_DEFAULT])
@pytest.mark.parametrize("P", [1, 16, 64])
def test_deepseek_latent_small(engine, P):
    """DeepSeek-V3 latent rows (1 x 576 bf16 = 1152 B: 72 vectors, not a power of two)."""
    g = _g(L=3, H=1, D=576, P=P, C=64, num_pages=-(-2000 // P) + 4, num_chunks=40)
    q = kvgen.make_requests(kvgen.rng_for(40 + P), [700, 1100, 33], g.P, g.C, g.num_pages, g.num_chunks,
                            offsets=True)
    c = GpuCase(g, q, seed=P)
    try:
        c.pool.load(c.reqs, engine=engine)
        torch.cuda.synchronize()
        c.check_load(0, g.L)
        before = c.pool.host.copy()
        for t in c.k:   # new device content, offloaded into the same host positions
            t.copy_(torch.randint(0, 256, t.shape, dtype=torch.uint8, device="cuda"))
        c.pool.offload(c.reqs, 1, 3, engine=engine)
        torch.cuda.synchronize()
        assert np.array_equal(c.pool.host, c.expected_offload(before, 1, 3))
    finally:
        c.close()


@pytest.mark.parametrize("engine", ENGINES)
def test_deepseek_fp8_latent_rows(engine):
    """FP8 MLA cache rows as FlashMLA stores them: 512 fp8 latent + 4 fp32 scales + 64 bf16 rope
    = 656 B per token and layer (41 vectors: neither a power of two nor a multiple of 32)."""
    g = _g(L=2, H=1, D=656, P=64, C=64, num_pages=40, num_chunks=40, e=1)
    q = kvgen.make_requests(kvgen.rng_for(47), [1500, 301], g.P, g.C, g.num_pages, g.num_chunks, offsets=True)
    c = GpuCase(g, q, seed=9)
    try:
        c.pool.load(c.reqs, engine=engine)
        torch.cuda.synchronize()
        c.check_load(0, g.L)
        before = c.pool.host.copy()
        c.pool.offload(c.reqs, engine=engine)
        torch.cuda.synchronize()
        assert np.array_equal(c.pool.host, c.expected_offload(before, 0, g.L))
    finally:
        c.close()


@pytest.mark.parametrize("i", range(60))
def test_fuzz_single_kv(i):
    rng = kvgen.rng_for(5000 + i)
    L = int(rng.choice([1, 2, 4]))
    H = int(rng.choice([1, 2]))
    D = int(rng.choice([64, 512, 576]))
    P = int(rng.choice([1, 4, 16, 64]))
    C = int(rng.choice([1, 16, 64]))
    ns = [int(rng.integers(0, 3 * C + 8)) for _ in range(int(rng.choice([1, 3])))]
    l0 = int(rng.integers(0, L))
    l1 = int(rng.integers(l0, L + 1))
    engine = ENGINES[i % len(ENGINES)]
    ctas = int(rng.choice([0, 1, 2, 8]))
    num_pages = sum(kvgen.pages_needed(P - 1, n, P) for n in ns) + int(rng.integers(1, 9))
    num_chunks = sum(kvgen.chunks_needed(C - 1, n, C) for n in ns) + int(rng.integers(1, 4))
    g = _g(L, H, D, P, C, num_pages, num_chunks)
    tok = g.token_bytes
    strides = (P * (tok + 32) + 48, tok + 32, g.D * g.e) if rng.random() < 0.3 else None
    q = kvgen.make_requests(rng, ns, P, C, num_pages, num_chunks, offsets=True)
    offload = i % 2 == 1
    c = GpuCase(g, q, strides=strides, seed=i, dev_fill="random" if offload else "canary")
    try:
        if offload:
            before = c.pool.host.copy()
            c.pool.offload(c.reqs, l0, l1, engine=engine, num_ctas=ctas)
            torch.cuda.synchronize()
            assert np.array_equal(c.pool.host, c.expected_offload(before, l0, l1)), (engine, g, ns)
        else:
            c.pool.load(c.reqs, l0, l1, engine=engine, num_ctas=ctas)
            torch.cuda.synchronize()
            c.check_load(l0, l1)
    finally:
        c.close()


@pytest.mark.slow
def test_deepseek_v3_mla_32k_full():
    """The bench workload (deepseek_v3_mla, 32K tokens, P = 1) in bench.py's launch configuration
    (default engine), sampled layers compared byte for byte."""
    g = kvgen.geometry("deepseek_v3_mla")
    q = kvgen.make_requests(kvgen.rng_for(0), kvgen.CONFIGS["deepseek_v3_mla"]["n"], g.P, g.C,
                            g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        t = c.pool.load(c.reqs)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == st.STRATA_ENGINE_LDG   # default for >= 16 MiB loads
        for l in (0, 1, 30, 60):
            assert c.pool.layer_elapsed_ms(t, l) > 0
        c.check_load(0, g.L, layers=[0, 1, 30, 59, 60])
    finally:
        c.close()
