"""Full-size parity (SURVEY §8c "the 5 configs: full-size configs once, layer by layer"): the
BASELINE.json workloads at their real sizes, in the launch configuration bench.py times (each
engine's default SM quota), EVERY layer compared byte for byte with the CPU oracle, streamed one
layer at a time (one layer's device buffers and its oracle image in host memory at once).

Engines: the ring engine (STRATA_ENGINE_TMA; the default for offloads) and the LDG engine (the
default for loads of >= 16 MiB of 16-byte rows), both zero-copy
kernels reading / writing the host tier through its UVA mapping.  Loads start from a
canary-filled pool, so "nothing else was touched" is part of every layer's comparison.  Offloads
write into a canary-filled tier through a FRESH chunk list; each layer's blocks of the touched
chunks are compared with the oracle's offload of that layer into a compact one-layer image, and
every untouched chunk must still be canary."""
import dataclasses
import os

import numpy as np
import pytest

import kvgen
import oracle
from tests.gpu_helpers import GpuCase, _assert_same

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

TMA, LDG = st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_LDG
HOST_CANARY = 0x5A
NT = max(1, min(16, os.cpu_count() or 1))   # oracle threads (the oracle's OpenMP loops, oracle.c)


def _load_every_layer(name, P, engine):
    g = kvgen.geometry(name, P=P)
    q = kvgen.make_requests(kvgen.rng_for(0), kvgen.CONFIGS[name]["n"], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        t = c.pool.load(c.reqs, engine=engine)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == engine
        for l in range(g.L):
            assert c.pool.layer_elapsed_ms(t, l) > 0
            ek = [None] * g.L
            ev = [None] * g.L
            ek[l] = np.full(c.layer_bytes, 0xA5, np.uint8)
            ev[l] = np.full(c.layer_bytes, 0xA5, np.uint8) if g.kv == 2 else None
            oracle.load(g, c.pool.host[: g.host_bytes], ek, ev if g.kv == 2 else ek, q, l, l + 1, nthreads=NT)
            _assert_same(c.k[l].cpu().numpy(), ek[l], f"{name} P={P} engine={engine} K layer {l}")
            if g.kv == 2:
                _assert_same(c.v[l].cpu().numpy(), ev[l], f"{name} P={P} engine={engine} V layer {l}")
    finally:
        c.close()


@pytest.mark.parametrize("name,P,engine", [
    ("llama8b_32k", 1, TMA), ("llama8b_32k", 1, LDG), ("llama8b_32k", 16, TMA), ("llama8b_32k", 16, LDG),
    ("llama70b_tp8", 1, TMA), ("llama70b_tp8", 1, LDG), ("qwen14b_batch8", 1, TMA), ("qwen14b_batch8", 1, LDG),
])
def test_fullsize_load_every_layer(name, P, engine):
    _load_every_layer(name, P, engine)


def _used_chunks(q, C):
    out = []
    for r in range(q.R):
        n = int(q.num_tokens[r])
        nc = kvgen.chunks_needed(int(q.chunk_offset[r]), n, C)
        out.append(q.host_chunks[int(q.chunk_start[r]): int(q.chunk_start[r]) + nc])
    return out


def _offload_every_layer(name, P, engine):
    g = kvgen.geometry(name, P=P)
    assert not g.head_major and g.host_heads == g.H   # token-major per-GPU tier: a layer block is contiguous
    q = kvgen.make_requests(kvgen.rng_for(0), kvgen.CONFIGS[name]["n"], g.P, g.C, g.num_pages, g.num_chunks)
    # a fresh host chunk list (another permutation of the tier) for the write-back
    q2 = kvgen.make_requests(kvgen.rng_for(1), kvgen.CONFIGS[name]["n"], g.P, g.C, g.num_pages, g.num_chunks)
    q2 = dataclasses.replace(q2, dev_pages=q.dev_pages, page_start=q.page_start, page_offset=q.page_offset)
    c = GpuCase(g, q2, host_fill="none", dev_fill="random", seed=7)
    try:
        c.pool.host[: g.host_bytes].fill(HOST_CANARY)
        c.pool.offload(c.reqs, engine=engine)
        torch.cuda.synchronize()
        assert c.pool.counters()["last_engine"] == engine
        used = _used_chunks(q2, g.C)
        touched = np.unique(np.concatenate(used))
        # the write-back through a compact one-layer tier of the touched chunks (same order as `touched`)
        hc1 = np.zeros_like(q2.host_chunks)
        for r in range(q2.R):
            cs = int(q2.chunk_start[r])
            hc1[cs: cs + used[r].size] = np.searchsorted(touched, used[r])
        q1 = dataclasses.replace(q2, host_chunks=hc1.astype(np.int32))
        g1 = dataclasses.replace(g, L=1, num_chunks=int(touched.size))
        blk = g.kv * g.C * g.token_bytes
        tier = c.pool.host[: g.host_bytes].reshape(g.num_chunks, g.L, blk)
        for l in range(g.L):
            img = np.full(g1.host_bytes, HOST_CANARY, np.uint8)
            dk = c.k[l].cpu().numpy()
            dv = c.v[l].cpu().numpy() if g.kv == 2 else dk
            oracle.offload(g1, img, [dk], [dv], q1, 0, 1, nthreads=NT)
            _assert_same(np.ascontiguousarray(tier[touched, l, :]).reshape(-1), img,
                         f"{name} P={P} engine={engine} offload layer {l}")
        untouched = np.setdiff1d(np.arange(g.num_chunks), touched)
        for i in range(0, untouched.size, 256):
            sl = tier[untouched[i: i + 256]]
            assert np.all(sl == HOST_CANARY), f"{name}: an untouched host chunk was written"
    finally:
        c.close()


@pytest.mark.parametrize("name,P,engine", [
    ("llama8b_32k", 1, TMA), ("llama8b_32k", 1, LDG), ("llama8b_32k", 16, TMA),
    ("llama70b_tp8", 1, TMA), ("llama70b_tp8", 1, LDG), ("qwen14b_batch8", 1, TMA),
])
def test_fullsize_offload_every_layer(name, P, engine):
    _offload_every_layer(name, P, engine)
