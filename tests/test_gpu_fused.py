"""The fused LDG path (one launch for every layer, per-layer device flags -> layer events; SURVEY §8
a5's persistent variant) against the oracle, against the per-layer path, and under concurrency."""
import json
import os
import subprocess
import sys

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

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case(seed=4, L=6, n=3000, P=4):
    g = Geometry(L, 4, 128, 2, P, 64, 4096, 400)
    q = kvgen.make_requests(kvgen.rng_for(seed), [n, n // 3, 17], g.P, g.C, g.num_pages, g.num_chunks)
    return g, q


def _launches_and_check(ctas):
    g, q = _case()
    c = GpuCase(g, q)
    try:
        before = c.pool.counters()["kernel_launches"]
        c.pool.load(c.reqs, stream=torch.cuda.current_stream().cuda_stream, engine=st.STRATA_ENGINE_LDG,
                    num_ctas=ctas)
        torch.cuda.synchronize()
        launches = c.pool.counters()["kernel_launches"] - before
        c.check_load(0, g.L)
        return launches, g.L
    finally:
        c.close()


@pytest.mark.parametrize("ctas", [1, 2, 5])
def test_fused_single_launch_parity(ctas):
    launches, L = _launches_and_check(ctas)
    if os.environ.get("STRATA_LDG_FUSED", "1") != "0" and ctas >= 2:
        assert launches == 1, launches          # one launch for all L layers
    else:
        assert launches == L                    # 1-CTA grids keep per-layer launches


def test_per_layer_path_still_exact():
    """STRATA_LDG_FUSED=0 (read once per process): the one-launch-per-layer path, in a subprocess."""
    code = ("import json, sys; sys.path.insert(0, %r); from tests.test_gpu_fused import _launches_and_check;"
            "print(json.dumps(_launches_and_check(2)))" % ROOT)
    env = dict(os.environ, STRATA_LDG_FUSED="0")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    launches, L = json.loads(out.stdout.strip().splitlines()[-1])
    assert launches == L


def test_fused_offload_parity():
    g, q = _case(seed=9)
    c = GpuCase(g, q, dev_fill="random")
    try:
        before = c.pool.host.copy()
        c.pool.offload(c.reqs, 1, g.L - 1, stream=torch.cuda.current_stream().cuda_stream,
                       engine=st.STRATA_ENGINE_LDG, num_ctas=3)
        torch.cuda.synchronize()
        exp = c.expected_offload(before, 1, g.L - 1)
        assert np.array_equal(c.pool.host, exp)
    finally:
        c.close()


def test_concurrent_ops_cross_waits():
    """Two fused loads in flight on two streams, op A held back behind a spin kernel; the consumer
    waits on B's and A's layer events.  Slots have their own flags and side streams: B's events do
    not wait for A, A's do not fire early (the consumer's sums equal the final bytes), no hang."""
    g = Geometry(8, 8, 128, 2, 1, 64, 8192 + 64, 140)
    qa = kvgen.make_requests(kvgen.rng_for(21), [4096], g.P, g.C, 4096, g.num_chunks)   # pages < 4096
    c = GpuCase(g, qa)
    try:
        rb = st.Requests(qa.num_tokens, qa.host_chunks, qa.chunk_start, (qa.dev_pages + 4096).astype(np.int32),
                         qa.page_start, qa.chunk_offset, qa.page_offset)      # same rows, pages + 4096
        s1, s2, cons = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        with torch.cuda.stream(s1):
            torch.cuda._sleep(2_000_000)      # op A starts late
        ta = c.pool.load(c.reqs, stream=s1.cuda_stream, engine=st.STRATA_ENGINE_LDG)
        tb = c.pool.load(rb, stream=s2.cuda_stream, engine=st.STRATA_ENGINE_LDG)
        sums = []
        with torch.cuda.stream(cons):
            for l in range(g.L):
                c.pool.wait_layer(tb, l, cons)
                c.pool.wait_layer(ta, l, cons)
                sums.append((c.k[l].view(torch.int64).sum(), c.v[l].view(torch.int64).sum()))
        torch.cuda.synchronize()
        half = 4096 * g.P * g.token_bytes
        for l in range(g.L):
            ka, va = c.expected_load_layer(l)
            got_k, got_v = c.k[l].cpu().numpy(), c.v[l].cpu().numpy()
            for got, exp in ((got_k, ka), (got_v, va)):
                np.testing.assert_array_equal(got[:half], exp[:half])
                np.testing.assert_array_equal(got[half:2 * half], exp[:half])
                np.testing.assert_array_equal(got[2 * half:], exp[2 * half:])
            assert int(sums[l][0]) == int(got_k.view(np.int64).sum())
            assert int(sums[l][1]) == int(got_v.view(np.int64).sum())
        assert c.pool.layer_elapsed_ms(tb, g.L - 1) > 0
    finally:
        c.close()


@pytest.mark.parametrize("engine", [st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_LDG])
def test_event_ring_slot_reuse_never_fires_early(engine):
    """Nine fused loads on two streams, the first held back behind a spin kernel: op 1 and op 9 share
    an event-ring slot (kEventRing = 8) and so its arrival counters and layer flags.  Op 9 must be
    ordered after op 1 (transfer.cpp order_after_slot), so no layer event of op 1 fires before its
    bytes land: a consumer that waits on op 1's layer events checksums exactly the final (oracle)
    bytes of op 1's pages, and nothing hangs (the executor waits per layer)."""
    g = Geometry(4, 8, 128, 2, 1, 64, 17000, 300)
    ns = [8192] + [1024] * 8      # >= 1024 tokens: the LDG engine fuses (>= 2 CTAs) as well
    q = kvgen.make_requests(kvgen.rng_for(33), ns, g.P, g.C, g.num_pages, g.num_chunks)   # disjoint pages
    c = GpuCase(g, q)
    try:
        def one(r):
            cs, ps = int(q.chunk_start[r]), int(q.page_start[r])
            nc, npg = kvgen.chunks_needed(0, ns[r], g.C), kvgen.pages_needed(0, ns[r], g.P)
            return st.Requests([ns[r]], q.host_chunks[cs: cs + nc], [0], q.dev_pages[ps: ps + npg], [0])
        reqs = [one(r) for r in range(len(ns))]
        s1, s2, cons = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        with torch.cuda.stream(s1):
            torch.cuda._sleep(50_000_000)     # ~25 ms: op 1 starts long after ops 2..9 could
        t1 = c.pool.load(reqs[0], stream=s1, engine=engine)
        tickets = [c.pool.load(r, stream=s2, engine=engine) for r in reqs[1:8]]
        pages1 = torch.from_numpy(q.dev_pages[: ns[0]].astype(np.int64)).cuda()
        sums = []
        with torch.cuda.stream(cons):   # the consumer's waits are enqueued while op 1's ticket is live
            for l in range(g.L):
                c.pool.wait_layer(t1, l, cons)
                rows_k = c.k[l].view(g.num_pages, -1)[pages1].view(torch.int64).sum()
                rows_v = c.v[l].view(g.num_pages, -1)[pages1].view(torch.int64).sum()
                sums.append((rows_k, rows_v))
        t9 = c.pool.load(reqs[8], stream=s2, engine=engine)   # reuses op 1's ring slot
        assert t9 == t1 + 8 and tickets[-1] == t1 + 7
        torch.cuda.synchronize()
        c.check_load(0, g.L)
        p1 = q.dev_pages[: ns[0]]
        for l in range(g.L):
            ek = c.k[l].cpu().numpy().reshape(g.num_pages, -1)[p1].view(np.int64).sum()
            ev = c.v[l].cpu().numpy().reshape(g.num_pages, -1)[p1].view(np.int64).sum()
            assert int(sums[l][0]) == int(ek) and int(sums[l][1]) == int(ev), f"layer {l}: event fired early"
    finally:
        c.close()
