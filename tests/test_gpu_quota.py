"""Decode-aware SM quota (NEXT-1; strata_set_load_quota): a stream-ordered cap on the CTAs of
one-launch LDG loads that take new rows.  With the cap, the row groups of every layer are taken
dynamically, so the result must stay bit-exact against the oracle whatever the cap and whenever it
changes, every layer event must still fire in layer order, and a cap of 1 must actually confine the
host reads to one CTA (the load slows to the one-CTA rate) — the lever DESIGN.md §6.1 measured:
co-running decode slows with the number of SMs keeping host reads in flight."""
import statistics

import numpy as np
import pytest

import kvgen
from kvgen import Geometry
from tests.gpu_helpers import GpuCase
from tests.helpers import CANARY

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2508_18572_b200 as st  # noqa: E402

LDG = st.STRATA_ENGINE_LDG


def _case(seed=5, L=6, n=5000, P=4, H=4):
    tokens = n + n // 3 + 17
    g = Geometry(L, H, 128, 2, P, 64, tokens // P + 256, tokens // 64 + 64)
    q = kvgen.make_requests(kvgen.rng_for(seed), [n, n // 3, 17], g.P, g.C, g.num_pages, g.num_chunks)
    return g, q


@pytest.mark.parametrize("ctas,cap", [(2, 1), (4, 1), (4, 3), (3, 5), (2, 0)])
def test_capped_load_is_exact(ctas, cap):
    g, q = _case()
    c = GpuCase(g, q)
    try:
        io = torch.cuda.Stream()
        c.pool.set_load_quota(cap, stream=io)          # stream-ordered before the load
        t = c.pool.load(c.reqs, stream=io, engine=LDG, num_ctas=ctas)
        c.pool.set_load_quota(0, stream=io)
        torch.cuda.synchronize()
        assert c.pool.counters()["kernel_launches"] >= 1
        c.check_load(0, g.L)
        done = [c.pool.layer_elapsed_ms(t, l) for l in range(g.L)]
        assert all(b >= a for a, b in zip(done, done[1:])), done
    finally:
        c.close()


def test_cap_toggled_while_loads_run():
    """Caps written from another stream while several loads run back to back (as a serving engine
    brackets its decode steps): every load bit-exact, the slot's group counters reset for the next."""
    g, q = _case(seed=6, L=8, n=9000, P=1)
    c = GpuCase(g, q)
    try:
        io, dec = torch.cuda.Stream(), torch.cuda.Stream()
        c.pool.set_load_quota(0, stream=dec)
        torch.cuda.synchronize()
        spin = torch.empty(1 << 26, dtype=torch.uint8, device="cuda")
        for i in range(12):
            c.pool.load(c.reqs, stream=io, engine=LDG, num_ctas=2 + i % 3)
            with torch.cuda.stream(dec):
                c.pool.set_load_quota(1 + i % 2, stream=dec)
                spin.add_(1)                            # some decode-stream work between the writes
                c.pool.set_load_quota(0, stream=dec)
        torch.cuda.synchronize()
        c.check_load(0, g.L)
        # the loads after the toggling still use every CTA and stay exact
        for t in c.k + c.v:
            t.fill_(CANARY)
        c.pool.load(c.reqs, stream=io, engine=LDG, num_ctas=4)
        torch.cuda.synchronize()
        c.check_load(0, g.L)
    finally:
        c.close()


def test_cap_confines_the_host_reads_to_one_cta():
    """A Llama-8B-row load of 512 MiB at 2 CTAs: capped to 1 it runs at the one-CTA rate (well below
    the uncapped rate), uncapped again it is back at the two-CTA rate."""
    L, n = 4, 32768
    g = Geometry(L, 8, 128, 2, 1, 64, n + 1024, n // 64 + 16)
    q = kvgen.make_requests(kvgen.rng_for(9), [n], g.P, g.C, g.num_pages, g.num_chunks)
    c = GpuCase(g, q)
    try:
        io = torch.cuda.Stream()
        c.pool.set_load_quota(0, stream=io)
        nbytes = 2 * L * n * g.token_bytes

        def rate(cap):
            out = []
            for _ in range(5):
                c.pool.set_load_quota(cap, stream=io)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(io)
                c.pool.load(c.reqs, stream=io, engine=LDG, num_ctas=2)
                b.record(io)
                b.synchronize()
                out.append(nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
            return statistics.median(out[1:])
        free, capped, again = rate(0), rate(1), rate(0)
        print(f"uncapped {free:.1f} GB/s, capped to 1 CTA {capped:.1f}, uncapped again {again:.1f}")
        assert capped < 0.8 * free, (free, capped)
        assert again > 0.9 * free, (free, again)
        c.pool.set_load_quota(0, stream=io)
        torch.cuda.synchronize()
        c.check_load(0, g.L)
    finally:
        c.close()


def test_quota_writes_captured_in_a_graph():
    """A decode step captured into a CUDA graph with its quota bracket (serving engines replay decode
    from graphs): the writes replay with it, the load beside the replays stays exact."""
    g, q = _case(seed=8, L=6, n=6000, P=2)
    c = GpuCase(g, q)
    try:
        io, dec = torch.cuda.Stream(), torch.cuda.Stream()
        c.pool.set_load_quota(0, stream=dec)
        x = torch.zeros(1 << 24, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=dec):
            c.pool.set_load_quota(1, stream=torch.cuda.current_stream())
            x.add_(1.0)
            c.pool.set_load_quota(0, stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
        c.pool.load(c.reqs, stream=io, engine=LDG, num_ctas=4)
        with torch.cuda.stream(dec):
            for _ in range(20):
                gr.replay()
        torch.cuda.synchronize()
        c.check_load(0, g.L)
        assert float(x[0]) == 20.0
    finally:
        c.close()


def test_quota_argument_errors():
    g, q = _case()
    c = GpuCase(g, q)
    try:
        with pytest.raises(st.StrataError):
            c.pool.set_load_quota(-1)
        assert np.isfinite(c.pool.counters()["kernel_launches"])
    finally:
        c.close()
