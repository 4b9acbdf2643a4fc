"""Parity of the native control plane (csrc/ctl.cpp via include/strata_ctl.h) with the oracle.

CPU only (the control plane makes no CUDA call).  Random traces of submits, host / device inserts,
scheduling rounds, completions and aborts drive both sides in lock step; after every operation the
batches, deferrals, Algorithm 1 accounting, both plans (strata_xfer arrays), every dispatched
request's page table, the queue, match results and the whole tree (canonical dump: paths, slots,
marks, pins, access times) must be identical.  Small pools make eviction and write-back frequent.
"""
import numpy as np
import pytest

from kvgen import traces
from oracle import ctl_oracle as co

ctl_mod = pytest.importorskip("paper_2508_18572_b200.ctl")


def _pair(P, C, pages, chunks, **kw):
    return (co.Ctl(P, C, pages, chunks, **kw),
            ctl_mod.Ctl(P, C, pages, chunks, max_batch_tokens=kw.pop("max_batch_tokens", 0),
                        max_batch_reqs=kw.pop("max_batch_reqs", 0), **kw))


def _same_plans(o, n):
    for which in ("load", "offload"):
        po, pn = o.plan(which), n.plan(which)
        for k in po:
            assert list(pn[k]) == list(po[k]), (which, k)


def _same_state(o, n, rng):
    assert n.dump() == o.dump()
    assert n.queue == o.queue
    for rid, r in o.reqs.items():
        if r.state == "dispatched":
            assert n.req_slots(rid).tolist() == r.slots


def _run_trace(seed, P, C, pages, chunks, vocab, steps, **kw):
    rng = np.random.default_rng(seed)
    o, n = _pair(P, C, pages, chunks, **kw)
    fam = traces.random_prefix_family(rng, 400, 160, vocab=vocab, branch=0.8)
    rid, t = 0, 0.0
    cov = {"batch": 0, "deferred": 0, "load": 0, "writeback": 0}
    for step in range(steps):
        op = rng.random()
        if op < 0.35:
            toks = fam[int(rng.integers(0, len(fam)))] + rng.integers(0, vocab, int(rng.integers(1, 20))).tolist()
            o.submit(rid, toks)
            n.submit(rid, toks)
            rid += 1
        elif op < 0.45:
            toks = fam[int(rng.integers(0, len(fam)))]
            tier = int(rng.integers(0, 2))
            try:
                so = o.insert(toks, tier, t)
            except MemoryError:
                so = None
            if so is None:
                with pytest.raises(Exception):
                    n.insert(toks, tier, t)
            else:
                assert n.insert(toks, tier, t) == so
            _same_plans(o, n)
        elif op < 0.75:
            oo = o.schedule(t)
            on = n.schedule(t)
            for k in ("batch", "deferred", "formed", "formed_load", "formed_compute", "new_tokens"):
                assert on[k] == oo[k], (step, k)
            assert on["load_tokens"] == len(o.load_pairs)
            assert on["writeback_tokens"] == len(o.offload_pairs)
            _same_plans(o, n)
            cov["batch"] += len(oo["batch"])
            cov["deferred"] += len(oo["deferred"])
            cov["load"] += on["load_tokens"]
            cov["writeback"] += on["writeback_tokens"]
        else:
            live = [r for r, q in o.reqs.items() if q.state == "dispatched"]
            if live:
                r = live[int(rng.integers(0, len(live)))]
                if rng.random() < 0.85:
                    o.complete(r, t)
                    n.complete(r, t)
                else:
                    o.abort(r)
                    n.abort(r)
            elif o.queue and rng.random() < 0.2:
                r = o.queue[int(rng.integers(0, len(o.queue)))]
                o.abort(r)
                n.abort(r)
        for _ in range(2):
            q = fam[int(rng.integers(0, len(fam)))][: int(rng.integers(0, 200))]
            assert n.match(q) == o.match(q)
        _same_state(o, n, rng)
        t += float(rng.integers(0, 3))      # equal timestamps exercise the LRU path tie-break
    return cov


@pytest.mark.parametrize("seed,P,C,pages,chunks", [
    (0, 1, 16, 900, 120), (1, 4, 16, 200, 100), (2, 16, 4, 40, 400), (3, 3, 5, 300, 150),
    (4, 1, 1, 1000, 3000), (5, 8, 64, 120, 40)])
def test_random_trace_parity(seed, P, C, pages, chunks):
    cov = _run_trace(seed, P, C, pages, chunks, vocab=4, steps=150, threshold=20, ratio=4.0,
               max_batch_tokens=600, max_batch_reqs=5)
    assert all(v > 0 for v in cov.values()), cov      # deferrals, loads and write-backs all happened


@pytest.mark.parametrize("flags", [dict(defer=False), dict(balance=False), dict(bundle=False),
                                   dict(defer=False, balance=False, bundle=False)])
def test_random_trace_parity_ablations(flags):
    _run_trace(11, 4, 16, 300, 200, vocab=3, steps=120, threshold=10, ratio=2.0,
               max_batch_tokens=400, max_batch_reqs=4, **flags)


def test_fig7_native():
    """The paper's Fig. 7 scenario through the native scheduler (same golden as the oracle pin)."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig7_scheduling.json")))
    n = ctl_mod.Ctl(1, 16, 1 << 16, 1 << 14, threshold=g["threshold"], ratio=g["ratio"],
                    max_batch_reqs=g["max_batch_reqs"])
    ctx = {name: list(range(base, base + g["context_tokens"])) for name, base in g["contexts"].items()}
    for c in g["host_resident"].values():
        n.insert(ctx[c], ctl_mod.HOST, 0.0)
    names = {}
    for i, (name, c, q) in enumerate(g["queue"]):
        n.submit(i, (ctx[c] if c else []) + [100000 + 1000 * i + j for j in range(q)])
        names[i] = name
    for t, expect in enumerate(g["batches"]):
        out = n.schedule(float(t))
        assert [names[r] for r in out["batch"]] == expect
        for r in out["batch"]:
            n.complete(r, t + 0.5)


def test_errors_and_bubble():
    n = ctl_mod.Ctl(4, 8, 4, 4)
    n.submit(1, [1, 2, 3])
    with pytest.raises(Exception):
        n.submit(1, [4])
    with pytest.raises(Exception):
        n.submit(2, [])
    with pytest.raises(Exception):
        n.complete(1, 0.0)                    # not dispatched
    with pytest.raises(Exception):
        n.insert(list(range(100)), ctl_mod.DEVICE, 0.0)   # 25 pages > 4
    for args in ((20.0, 5.0, 3.0, 8), (5.0, 5.0, 3.0, 8), (20.0, 5.0, 3.0, 0), (7.5, 1.0, 0.5, 2)):
        assert ctl_mod.bubble_steps(*args) == co.bubble_steps(*args)
