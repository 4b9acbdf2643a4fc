"""Pins for the control-plane oracle (oracle/ctl_oracle.py).

Nothing here compares the oracle with itself.  It is tied to:
  * brute force       — longest-prefix match and per-tier counts against a plain prefix store,
  * the paper's worked example — Fig. 7 / PAPER.md:358-362: queue (C, D0, D1, F) forms (C, F) then
                        the bundle hit (D0, D1),
  * the paper's constants — delay-hit threshold 100 tokens, loading-bound ratio 100
                        (PAPER.md:366), strict comparisons at the boundary,
  * accounting        — with deferral, a shared uncached context is prefilled once
                        (PAPER.md:316-317): total prefill tokens = unique context + queries,
  * invariants        — radix property, slot conservation, the head of the queue always enters the
                        batch, plans decode back to exactly the planned pairs
                        through include/strata.h's token formula.
"""
import json
import os

import numpy as np
import pytest

from kvgen import traces
from oracle import ctl_oracle as co

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ helpers
def check_invariants(ctl: co.Ctl) -> None:
    """Radix property, transient nodes hold no slots, and every live slot has one owner."""
    dev_owner, host_owner = {}, {}
    for n in ctl._nodes():
        assert n.key, "empty edge"
        assert n.parent.children[n.key[0]] is n
        if n.mark:
            assert not n.dev and not n.host, "transient node holds slots"
        else:
            assert n.dev or n.host, "committed node without residency"
        for lst, own in ((n.dev, dev_owner), (n.host, host_owner)):
            assert len(lst) in (0, len(n.key))
            for s in lst:
                assert s not in own, "slot owned twice"
                own[s] = n
        assert n.ref >= 0 and n.tref >= 0
    for r in ctl.reqs.values():
        if r.state == "dispatched":
            for s in r.slots[r.k:]:
                if s in dev_owner:     # already attached? impossible before complete()
                    raise AssertionError("request slot owned by the tree before commit")
                dev_owner[s] = r
    for pool, own in ((ctl.dpool, dev_owner), (ctl.hpool, host_owner)):
        live = [0] * len(pool.live)
        for s in own:
            live[s // pool.unit] += 1
        assert live == pool.live
        assert sorted(pool.free) == [u for u in range(len(live)) if live[u] == 0]


def decode_plan(plan, C, P):
    """Per-token (host slot, device slot) through include/strata.h:25-27, written out."""
    pairs = []
    for r, n in enumerate(plan["num_tokens"]):
        for i in range(n):
            ci = plan["chunk_offset"][r] + i
            pi = plan["page_offset"][r] + i
            h = plan["host_chunks"][plan["chunk_start"][r] + ci // C] * C + ci % C
            d = plan["dev_pages"][plan["page_start"][r] + pi // P] * P + pi % P
            pairs.append((h, d))
    return pairs


# ------------------------------------------------------------------ match: brute force
@pytest.mark.parametrize("seed", range(6))
def test_match_brute_force(seed):
    rng = np.random.default_rng(seed)
    ctl = co.Ctl(page_size=4, chunk_tokens=8, num_pages=4096, num_chunks=4096)
    seqs = traces.random_prefix_family(rng, 60, 24, vocab=5)
    store = {}                                   # prefix tuple -> set of tiers holding it
    for j, s in enumerate(seqs):
        tier = int(rng.integers(0, 2))
        ctl.insert(s, tier, now=float(j))
        for i in range(1, len(s) + 1):
            store.setdefault(tuple(s[:i]), set()).add(tier)
    for q in traces.random_prefix_family(rng, 80, 30, vocab=5) + seqs:
        total = 0
        while total < len(q) and tuple(q[:total + 1]) in store:
            total += 1
        dev = sum(1 for i in range(total) if co.DEVICE in store[tuple(q[:i + 1])])
        m = ctl.match(q)
        assert m == {"total": total, "device": dev, "host": total - dev, "transient": 0}
    check_invariants(ctl)


def test_insert_returns_slots_and_is_idempotent():
    ctl = co.Ctl(page_size=4, chunk_tokens=8, num_pages=64, num_chunks=64)
    a = ctl.insert([1, 2, 3, 4, 5, 6], co.DEVICE, 0.0)
    assert a == [0, 1, 2, 3, 4, 5]               # pages 0, 1 (LIFO pops 0 first), P = 4
    b = ctl.insert([1, 2, 3, 9, 9], co.DEVICE, 1.0)
    assert b[:3] == a[:3] and b[3:] == [8, 9]    # the split keeps slots; new suffix gets page 2
    assert ctl.insert([1, 2, 3], co.DEVICE, 2.0) == a[:3]
    assert ctl.match([1, 2, 3, 4, 5, 6, 7]) == {"total": 6, "device": 6, "host": 0, "transient": 0}
    h = ctl.insert([1, 2, 3, 4], co.HOST, 3.0)   # now also host resident: counted as device
    assert h == [0, 1, 2, 8]                     # one run per node (R23): [1,2,3] chunk 0, [4] chunk 1
    assert ctl.match([1, 2, 3, 4])["device"] == 4
    check_invariants(ctl)


# ------------------------------------------------------------------ delay hits (§4.3.1)
def _ctl(**kw):
    args = dict(page_size=1, chunk_tokens=16, num_pages=1 << 16, num_chunks=1 << 14)
    args.update(kw)
    return co.Ctl(**args)


def test_delay_hit_defers_shared_miss_and_prefills_context_once():
    rng = np.random.default_rng(1)
    ctx = rng.integers(0, 1000, 5000).tolist()
    ctl = _ctl()
    for i in range(3):
        ctl.submit(i, ctx + [2000 + i] * 10)
    out = ctl.schedule(0.0)
    assert out["batch"] == [0] and out["deferred"] == [1, 2]   # 5000 > 100 transient tokens
    out = ctl.schedule(1.0)                                    # 0 still in flight
    assert out["batch"] == [] and out["deferred"] == [1, 2]
    ctl.complete(0, 2.0)
    out = ctl.schedule(3.0)
    assert out["batch"] == [1, 2] and out["deferred"] == []
    assert out["new_tokens"] == 2 * 10                          # the context hits on the device
    check_invariants(ctl)


@pytest.mark.parametrize("shared,deferred", [(50, False), (100, False), (101, True)])
def test_delay_hit_threshold_is_strict(shared, deferred):
    ctl = _ctl()
    base = list(range(shared))
    ctl.submit(0, base + [7000 + j for j in range(300)])
    ctl.submit(1, base + [8000 + j for j in range(300)])
    out = ctl.schedule(0.0)
    assert (out["deferred"] == [1]) is deferred


def test_deferred_requests_go_to_the_front():
    ctl = _ctl(max_batch_reqs=1)
    ctx = list(range(500))
    ctl.submit(0, ctx + [1])
    ctl.submit(1, [9000 + j for j in range(50)])
    ctl.submit(2, ctx + [2])
    out = ctl.schedule(0.0)
    assert out["batch"] == [0] and out["deferred"] == [2]
    assert ctl.queue == [2, 1]                                  # PAPER.md:317 "front of the queue"


def test_prefill_accounting_duplicate_contexts():
    """Brute-force accounting: with deferral the shared context is computed once."""
    rng = np.random.default_rng(2)
    ctx = rng.integers(0, 1000, 500).tolist()
    reqs = [ctx + rng.integers(1000, 2000, 20).tolist() for _ in range(10)]
    for defer, expect in ((True, 500 + 10 * 20), (False, 10 * 520)):
        ctl = _ctl(defer=defer)
        for i, r in enumerate(reqs):
            ctl.submit(i, r)
        total, t = 0, 0.0
        while ctl.reqs:
            out = ctl.schedule(t)
            total += out["new_tokens"]
            for rid in out["batch"]:
                ctl.complete(rid, t + 0.5)
            t += 1.0
        assert total == expect


def test_abort_restores_tree():
    ctl = _ctl()
    ctl.insert(list(range(10)), co.DEVICE, 0.0)
    before = ctl.dump()
    ctl.submit(0, list(range(10)) + [50, 51, 52, 53])
    out = ctl.schedule(1.0)
    assert out["batch"] == [0]
    ctl.abort(0)
    ctl.schedule(2.0)                                           # clears in-queue marks
    after = [(p, d, h, m, t, r) for p, d, h, m, t, r, _ in ctl.dump()]
    assert after == [(p, d, h, m, t, r) for p, d, h, m, t, r, _ in before]
    check_invariants(ctl)


# ------------------------------------------------------------------ Algorithm 1 (§4.3.2)
def test_fig7_balanced_batches():
    """PAPER.md:358-362 / Fig. 7, replayed from tests/golden/fig7_scheduling.json."""
    g = json.load(open(os.path.join(GOLDEN, "fig7_scheduling.json")))
    ctl = _ctl(max_batch_reqs=g["max_batch_reqs"], threshold=g["threshold"], ratio=g["ratio"])
    ctx = {name: list(range(base, base + g["context_tokens"])) for name, base in g["contexts"].items()}
    for name, c in g["host_resident"].items():
        ctl.insert(ctx[c], co.HOST, 0.0)
    ids = {}
    for i, (name, c, q) in enumerate(g["queue"]):
        toks = (ctx[c] if c else []) + [100000 + 1000 * i + j for j in range(q)]
        ids[name] = i
        ctl.submit(i, toks)
    names = {v: k for k, v in ids.items()}
    for t, expect in enumerate(g["batches"]):
        out = ctl.schedule(float(t))
        assert [names[r] for r in out["batch"]] == expect
        for rid in out["batch"]:
            ctl.complete(rid, t + 0.5)


def _bound_case(host, query, **kw):
    """Queue (head, candidate, filler) with room for two: the candidate enters iff it is not
    loading-bound; otherwise it waits in D and the compute-only filler takes the place."""
    ctl = _ctl(num_chunks=1 << 13, max_batch_reqs=2, **kw)
    ctl.submit(0, [10**6])                               # head: 1 token, compute 1
    ctx = list(range(host))
    if host:
        ctl.insert(ctx, co.HOST, 0.0)
    ctl.submit(1, ctx + [2 * 10**6 + j for j in range(query)])
    ctl.submit(2, [3 * 10**6 + j for j in range(50)])
    st = {r: ctl._stats(r) for r in (0, 1, 2)}
    assert st[1]["host"] == host and st[1]["compute"] == query
    return ctl.form_batch([0, 1, 2], st)[0]


@pytest.mark.parametrize("host,query,bound", [(50000, 400, True), (40000, 400, False), (0, 1, False)])
def test_loading_bound_arithmetic(host, query, bound):
    """SPEC loading_bound examples with the paper's ratio 100: head compute 1 +
    candidate 400 -> 50000 / 401 = 124.7 > 100 is bound, 40000 / 401 = 99.8 is not."""
    assert _bound_case(host, query) == ([0, 2] if bound else [0, 1])


def test_loading_bound_exact_boundary():
    """Ratio exactly at the threshold is not loading-bound (strict '>')."""
    assert _bound_case(40100, 400, ratio=100.0) == [0, 1]          # 40100 / 401 == 100.0
    assert _bound_case(40101, 400, ratio=100.0) == [0, 2]


def test_fifo_baseline_when_features_off():
    ctl = _ctl(defer=False, balance=False, bundle=False, max_batch_reqs=2)
    ctl.insert(list(range(20000)), co.HOST, 0.0)
    for i in range(4):
        ctl.submit(i, list(range(20000)) + [10**6 * (i + 1) + j for j in range(5)])
    assert ctl.schedule(0.0)["batch"] == [0, 1]                 # plain arrival order


@pytest.mark.parametrize("seed", range(4))
def test_head_always_enters_and_admitted_requests_are_balanced(seed):
    """PAPER.md:371 (starvation freedom) and Alg. 1 line 12-16 replayed on random queues."""
    rng = np.random.default_rng(100 + seed)
    ctl = _ctl(num_pages=1 << 20, max_batch_tokens=3000, max_batch_reqs=6)
    docs = [rng.integers(0, 500, int(rng.integers(200, 4000))).tolist() for _ in range(6)]
    for d in docs[:4]:
        ctl.insert(d, co.HOST, 0.0)
    rid, t = 0, 0.0
    for _ in range(30):
        for _ in range(int(rng.integers(0, 5))):
            d = docs[int(rng.integers(0, len(docs)))]
            ctl.submit(rid, d + rng.integers(1000, 2000, int(rng.integers(1, 600))).tolist())
            rid += 1
        queue_before = list(ctl.queue)
        out = ctl.schedule(t)
        eligible = [r for r in queue_before if r not in out["deferred"]]
        if eligible:
            assert out["formed"][0] == eligible[0]
        for r in out["batch"]:
            if rng.random() < 0.8:
                ctl.complete(r, t + 0.5)
            else:
                ctl.abort(r)
        check_invariants(ctl)
        t += 1.0


def test_bubble_steps_examples():
    """SPEC plan_bubble_fill examples."""
    assert co.bubble_steps(20.0, 5.0, 3.0, 8) == 5
    assert co.bubble_steps(5.0, 5.0, 3.0, 8) == 0
    assert co.bubble_steps(20.0, 5.0, 3.0, 0) == 0
    assert co.bubble_steps(20.0, 5.0, 3.0, 8, enabled=False) == 0


# ------------------------------------------------------------------ eviction and plans
def test_lru_eviction_and_writeback():
    ctl = _ctl(page_size=2, chunk_tokens=2, num_pages=4, num_chunks=8)
    a = ctl.insert([1, 2], co.DEVICE, 10.0)
    b = ctl.insert([3, 4], co.DEVICE, 20.0)
    ctl.insert([5, 6, 7, 8], co.DEVICE, 30.0)            # pool full (4 pages of 2)
    ctl.submit(0, [9, 9, 9])                             # needs 2 pages -> evict 10 s, then 20 s
    out = ctl.schedule(40.0)
    assert out["batch"] == [0]
    assert ctl.match([1, 2]) == {"total": 2, "device": 0, "host": 2, "transient": 0}
    assert ctl.match([3, 4])["host"] == 2 and ctl.match([5, 6, 7, 8])["device"] == 4
    wb = decode_plan(ctl.plan("offload"), ctl.C, ctl.P)
    assert [d for _, d in wb] == a + b                   # written back in LRU order
    ctl2 = _ctl(page_size=2, chunk_tokens=2, num_pages=2, num_chunks=8)
    ctl2.insert([1, 2, 3, 4], co.DEVICE, 0.0)
    ctl2.submit(0, [1, 2, 3, 4, 5])                      # pins its own prefix: nothing evictable
    out = ctl2.schedule(1.0)
    assert out["batch"] == [] and ctl2.queue == [0]


@pytest.mark.parametrize("P,C", [(1, 64), (16, 64), (4, 3), (64, 16)])
def test_plan_runs_decode_to_pairs(P, C):
    rng = np.random.default_rng(P * 100 + C)
    pairs = []
    h = int(rng.integers(0, 50 * C))
    d = int(rng.integers(0, 50 * P))
    for _ in range(400):                     # runs with random breaks on either side
        pairs.append((h, d))
        h = h + 1 if rng.random() < 0.8 else int(rng.integers(0, 50 * C))
        d = d + 1 if rng.random() < 0.8 else int(rng.integers(0, 50 * P))
    pairs = list(dict.fromkeys(pairs))
    plan = co.runs(pairs, C, P)
    assert decode_plan(plan, C, P) == pairs
    # greedy canonical form: no two adjacent requests could be one
    ends = np.cumsum(plan["num_tokens"])
    for e in ends[:-1]:
        (h0, d0), (h1, d1) = pairs[e - 1], pairs[e]
        hc = (h1 % C == 0) if h0 % C == C - 1 else (h1 == h0 + 1)
        dc = (d1 % P == 0) if d0 % P == P - 1 else (d1 == d0 + 1)
        assert not (hc and dc)


def test_load_plan_moves_host_copy_to_request_slots():
    ctl = _ctl(page_size=4, chunk_tokens=8, num_pages=256, num_chunks=256)
    rng = np.random.default_rng(5)
    doc = rng.integers(0, 100, 300).tolist()
    hs = ctl.insert(doc, co.HOST, 0.0)
    ctl.insert(doc[:40], co.DEVICE, 0.0)                 # first 40 tokens also on the device
    ctl.submit(0, doc + [777, 778])
    out = ctl.schedule(1.0)
    pairs = decode_plan(ctl.plan("load"), ctl.C, ctl.P)
    slots = ctl.reqs[0].slots
    assert pairs == list(zip(hs[40:], slots[40:300]))    # exactly the host-only part, in order
    assert out["new_tokens"] == 2
