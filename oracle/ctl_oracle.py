"""Plain Python oracle of the Strata control plane.  TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import this module; the product's control plane (``csrc/ctl.cpp`` behind
``include/strata_ctl.h``) shares no code with it.

What it computes, in the paper's order and notation:

* HiRadixTree with transient nodes (§4.3.1): a radix tree over token ids whose
  committed nodes point at device slots and/or host slots ("effectively serving as a page table",
  PAPER.md:221) and whose transient nodes carry ``in-queue`` / ``in-flight`` marks instead.
* Deferral on delay hit: a request whose tokens match more than ``threshold``
  tokens on transient nodes is deferred to the next round, at the front of the queue.
* Balanced batch formation, Algorithm 1, with AddBundleHit, the
  ``loading_bound`` ratio test (default 100) and the deprioritised list D.
* Bubble filling: decode steps that fit in the loading stall.
* The cache controller's load / write-back plan: the (host slot, device slot) pairs a batch needs,
  split into ``strata_xfer`` requests (R25).

Every reading of the paper taken where it is silent (R17-R26) is listed in DESIGN.md §10 and cited
at the function that applies it.  Pinned by tests/test_ctl_oracle.py (brute-force longest-prefix
match, the paper's Fig. 7 scenario, SPEC examples, conservation and plan-semantics invariants).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

IN_QUEUE, IN_FLIGHT = 1, 2
DEVICE, HOST = 0, 1


def _ceil(a: int, b: int) -> int:
    return -(-a // b)


def _common(a, b) -> int:
    n = 0
    while n < len(a) and n < len(b) and a[n] == b[n]:
        n += 1
    return n


class Node:
    def __init__(self, key, parent):
        self.key: List[int] = list(key)
        self.parent: Optional[Node] = parent
        self.children: Dict[int, Node] = {}
        self.dev: List[int] = []      # device slot (page*P + offset) per token, or empty
        self.host: List[int] = []     # host slot (chunk*C + offset) per token, or empty
        self.mark = 0                 # 0 committed, IN_QUEUE, IN_FLIGHT
        self.tref = 0                 # dispatched requests covering this transient node
        self.ref = 0                  # dispatched requests pinning this committed node
        self.last_access = 0.0


class Pool:
    """LIFO free list of units (device pages of P slots, host chunks of C slots) — R23."""

    def __init__(self, units: int, unit: int):
        self.unit = unit
        self.free = list(range(units - 1, -1, -1))    # pops 0, 1, 2, ... first
        self.live = [0] * units

    def alloc(self, ntok: int) -> List[int]:
        k = _ceil(ntok, self.unit)
        assert k <= len(self.free), "caller must ensure space"
        units = [self.free.pop() for _ in range(k)]
        slots = [units[j // self.unit] * self.unit + j % self.unit for j in range(ntok)]
        for s in slots:
            self.live[s // self.unit] += 1
        return slots

    def release(self, s: int) -> None:
        u = s // self.unit
        self.live[u] -= 1
        assert self.live[u] >= 0
        if self.live[u] == 0:
            self.free.append(u)


class Req:
    def __init__(self, tokens):
        self.tokens = list(tokens)
        self.state = "queued"
        self.k = 0                    # committed prefix pinned at dispatch
        self.slots: List[int] = []    # device slot of every token (the request's page table)


class Ctl:
    def __init__(self, page_size: int, chunk_tokens: int, num_pages: int, num_chunks: int,
                 threshold: int = 100, ratio: float = 100.0, max_batch_tokens: int = 1 << 40,
                 max_batch_reqs: int = 1 << 30, defer: bool = True, balance: bool = True,
                 bundle: bool = True):
        self.P, self.C = page_size, chunk_tokens
        self.dpool = Pool(num_pages, page_size)
        self.hpool = Pool(num_chunks, chunk_tokens)
        self.threshold, self.ratio = threshold, ratio
        self.max_tokens, self.max_reqs = max_batch_tokens, max_batch_reqs
        self.defer, self.balance, self.bundle = defer, balance, bundle
        self.root = Node([], None)
        self.queue: List[int] = []
        self.reqs: Dict[int, Req] = {}
        self.load_pairs: List[Tuple[int, int]] = []      # (host slot, device slot)
        self.offload_pairs: List[Tuple[int, int]] = []   # (host slot, device slot)

    # ---------------------------------------------------------------- tree primitives
    def _nodes(self):
        out, stack = [], [self.root]
        while stack:
            n = stack.pop()
            for c in n.children.values():
                out.append(c)
                stack.append(c)
        return out

    def path(self, n: Node) -> Tuple[int, ...]:
        parts = []
        while n is not None and n is not self.root:
            parts.append(n.key)
            n = n.parent
        return tuple(t for part in reversed(parts) for t in part)

    def _segments(self, key):
        """(node, start, matched length) along the longest stored prefix of key; no mutation."""
        segs, node, i = [], self.root, 0
        while i < len(key):
            c = node.children.get(key[i])
            if c is None:
                break
            l = _common(c.key, key[i:])
            segs.append((c, i, l))
            if l < len(c.key):
                break
            i += l
            node = c
        return segs

    @staticmethod
    def _cls(n: Node) -> str:
        return "transient" if n.mark else ("device" if n.dev else "host")

    def match(self, key) -> Dict[str, int]:
        """Longest stored prefix with its per-tier breakdown (SPEC match_prefix)."""
        out = {"total": 0, "device": 0, "host": 0, "transient": 0}
        for c, _, l in self._segments(key):
            out[self._cls(c)] += l
            out["total"] += l
        return out

    def _split(self, c: Node, at: int) -> Node:
        """Split c after `at` tokens; the new upper node keeps c's state (marks, pins, slots)."""
        up = Node(c.key[:at], c.parent)
        up.dev, up.host = c.dev[:at], c.host[:at]
        up.mark, up.tref, up.ref, up.last_access = c.mark, c.tref, c.ref, c.last_access
        c.parent.children[c.key[0]] = up
        c.key, c.dev, c.host = c.key[at:], c.dev[at:], c.host[at:]
        c.parent = up
        up.children[c.key[0]] = c
        return up

    def _align(self, key):
        """Nodes covering the longest stored prefix of key, splitting a partially matched node."""
        nodes, node, i = [], self.root, 0
        while i < len(key):
            c = node.children.get(key[i])
            if c is None:
                break
            l = _common(c.key, key[i:])
            if l < len(c.key):
                c = self._split(c, l)
            nodes.append(c)
            i += l
            node = c
        return nodes, i

    def _add_child(self, parent: Node, key) -> Node:
        n = Node(key, parent)
        parent.children[key[0]] = n
        return n

    # ---------------------------------------------------------------- transient nodes (§4.3.1)
    def _mark_in_queue(self, key) -> None:
        """Cover the unmatched rest of key by an in-queue transient node."""
        nodes, i = self._align(key)
        if i < len(key):
            self._add_child(nodes[-1] if nodes else self.root, key[i:]).mark = IN_QUEUE

    def _clear_in_queue(self) -> None:
        """R18: in-queue marks live for one scheduling round."""
        stack = [self.root]
        while stack:
            n = stack.pop()
            for t, c in list(n.children.items()):
                if c.mark == IN_QUEUE:
                    del n.children[t]
                else:
                    stack.append(c)

    # ---------------------------------------------------------------- eviction (R23)
    def _lru(self, cands) -> Node:
        return min(cands, key=lambda n: (n.last_access, self.path(n)))

    def _ensure_host(self, units: int) -> bool:
        while len(self.hpool.free) < units:
            cands = [n for n in self._nodes() if n.mark == 0 and n.host and not n.dev
                     and n.ref == 0 and not n.children]
            if not cands:
                return False
            v = self._lru(cands)
            for s in v.host:
                self.hpool.release(s)
            del v.parent.children[v.key[0]]
        return True

    def _ensure_dev(self, units: int) -> bool:
        while len(self.dpool.free) < units:
            cands = [n for n in self._nodes() if n.mark == 0 and n.dev and n.ref == 0
                     and not any(c.dev for c in n.children.values())]
            if not cands:
                return False
            v = self._lru(cands)
            if not v.host:                      # inclusive write-back before the drop
                if not self._ensure_host(_ceil(len(v.key), self.C)):
                    return False
                v.host = self.hpool.alloc(len(v.key))
                self.offload_pairs += list(zip(v.host, v.dev))
            for s in v.dev:
                self.dpool.release(s)
            v.dev = []
        return True

    # ---------------------------------------------------------------- public tree operations
    def insert(self, tokens, tier: int, now: float) -> List[int]:
        """Make `tokens` resident on `tier`; return every token's slot there (SPEC insert).
        Replaces both plans, like a scheduling round (its evictions' write-backs)."""
        self.load_pairs, self.offload_pairs = [], []
        nodes, i = self._align(tokens)
        pool, unit = (self.dpool, self.P) if tier == DEVICE else (self.hpool, self.C)
        attr = "dev" if tier == DEVICE else "host"
        need = sum(_ceil(len(n.key), unit) for n in nodes if not getattr(n, attr))
        need += _ceil(len(tokens) - i, unit)
        for n in nodes:
            n.ref += 1
        ok = self._ensure_dev(need) if tier == DEVICE else self._ensure_host(need)
        for n in nodes:
            n.ref -= 1
        if not ok:
            raise MemoryError("tier full")
        for n in nodes:
            n.mark, n.tref = 0, 0
            if not getattr(n, attr):
                setattr(n, attr, pool.alloc(len(n.key)))
            n.last_access = now
        if i < len(tokens):
            n = self._add_child(nodes[-1] if nodes else self.root, tokens[i:])
            setattr(n, attr, pool.alloc(len(tokens) - i))
            n.last_access = now
            nodes.append(n)
        return [s for n in nodes for s in getattr(n, attr)]

    # ---------------------------------------------------------------- scheduler (§4.3)
    def submit(self, rid: int, tokens) -> None:
        assert rid not in self.reqs and len(tokens) >= 1
        self.reqs[rid] = Req(tokens)
        self.queue.append(rid)

    def _key(self, rid: int):
        """R17: the last token is always prefilled, so only tokens[:n-1] can hit the cache."""
        t = self.reqs[rid].tokens
        return t[:-1]

    def _stats(self, rid: int):
        """Load and compute requirement of a request from the HiRadixTree."""
        key = self._key(rid)
        segs = [(i, l, self._cls(c)) for c, i, l in self._segments(key)]
        m = self.match(key)
        n = len(self.reqs[rid].tokens)
        return {"key": key, "segs": segs, "device": m["device"], "host": m["host"],
                "compute": n - m["device"] - m["host"]}

    @staticmethod
    def _host_overlap(sr, sb) -> int:
        """Host tokens of r inside the prefix r shares with b: what b's load already brings (R20)."""
        lcp = _common(sr["key"], sb["key"])
        return sum(max(0, min(i + l, lcp) - i) for i, l, cls in sr["segs"] if cls == "host")

    def form_batch(self, Q: List[int], st) -> Tuple[List[int], int, int]:
        """Algorithm 1, Balanced Batch Formation, line by line."""
        B: List[int] = []
        acc = {"load": 0, "compute": 0}

        def overlap(r):
            return max([self._host_overlap(st[r], st[b]) for b in B], default=0)

        def eff_load(r):                    # a bundle hit's shared context loads once (R20)
            return st[r]["host"] - overlap(r)

        def is_bundle_hit(r):
            return overlap(r) > self.threshold

        def is_full():                      # R21
            return len(B) >= self.max_reqs or acc["compute"] >= self.max_tokens

        def fits(r):                        # R21: the head always enters
            return not B or (len(B) + 1 <= self.max_reqs
                             and acc["compute"] + st[r]["compute"] <= self.max_tokens)

        def loading_bound(r):               # ratio of aggregated load to compute
            load = acc["load"] + eff_load(r)
            comp = acc["compute"] + st[r]["compute"]
            return float(load) / float(max(comp, 1)) > self.ratio

        def add(r):
            acc["load"] += eff_load(r)
            acc["compute"] += st[r]["compute"]
            B.append(r)

        def add_bundle_hit():               # procedure AddBundleHit(Q, B), lines 1-7
            if not self.bundle:
                return
            for r in list(Q):
                if is_bundle_hit(r) and fits(r):
                    add(r)
                    Q.remove(r)

        if not Q:
            return B, 0, 0
        add(Q.pop(0))                       # line 10
        add_bundle_hit()
        D: List[int] = []
        while Q and not is_full():          # line 11
            r = Q.pop(0)
            if self.balance and loading_bound(r):
                D.append(r)                 # line 14
            elif fits(r):
                add(r)                      # line 16
                add_bundle_hit()
            else:
                break                       # R21: FIFO stop at the first request that does not fit
        for r in D:                         # lines 17-19
            if is_full() or not fits(r):
                break
            add(r)
        return B, acc["load"], acc["compute"]

    def _dispatch(self, rid: int, now: float) -> bool:
        """Pin the cached prefix, load its host part, allocate the new tokens."""
        r = self.reqs[rid]
        nodes, _ = self._align(self._key(rid))
        cn = []
        for nd in nodes:
            if nd.mark:
                break
            cn.append(nd)
        tn = nodes[len(cn):]
        assert all(nd.mark for nd in tn)
        k = sum(len(nd.key) for nd in cn)
        n = len(r.tokens)
        for nd in cn:
            nd.ref += 1
        need = sum(_ceil(len(nd.key), self.P) for nd in cn if not nd.dev) + _ceil(n - k, self.P)
        if not self._ensure_dev(need):
            for nd in cn:
                nd.ref -= 1
            return False
        for nd in cn:
            if not nd.dev:
                nd.dev = self.dpool.alloc(len(nd.key))
                self.load_pairs += list(zip(nd.host, nd.dev))
            nd.last_access = now
        new = self.dpool.alloc(n - k)
        for nd in tn:                       # "marked in-flight"
            nd.mark = IN_FLIGHT
            nd.tref += 1
        r.k, r.state = k, "dispatched"
        r.slots = [s for nd in cn for s in nd.dev] + new
        return True

    def schedule(self, now: float):
        """One scheduling round: deferral (§4.3.1), Algorithm 1 (§4.3.2), dispatch + plans."""
        self.load_pairs, self.offload_pairs = [], []
        self._clear_in_queue()
        eligible, deferred = [], []
        for rid in self.queue:
            key = self._key(rid)
            if self.defer:
                if self.match(key)["transient"] > self.threshold:
                    deferred.append(rid)
                    continue
                self._mark_in_queue(key)
            eligible.append(rid)
        st = {rid: self._stats(rid) for rid in eligible}
        batch, load, compute = self.form_batch(list(eligible), st)
        done = []
        for rid in batch:
            if not self._dispatch(rid, now):
                break
            done.append(rid)
        self.queue = deferred + [rid for rid in eligible if rid not in done]   # R19
        return {"batch": done, "deferred": deferred, "formed": batch,
                "formed_load": load, "formed_compute": compute,
                "new_tokens": sum(len(self.reqs[r].tokens) - self.reqs[r].k for r in done)}

    def complete(self, rid: int, now: float) -> None:
        """The prefill of rid finished: its transient nodes become standard nodes."""
        r = self.reqs[rid]
        assert r.state == "dispatched"
        nodes, i = self._align(r.tokens)
        pos = 0
        for nd in nodes:
            L = len(nd.key)
            if pos < r.k:
                nd.ref -= 1
            elif nd.mark:
                nd.mark, nd.tref, nd.dev = 0, 0, r.slots[pos:pos + L]
            elif nd.dev:
                for s in r.slots[pos:pos + L]:          # computed twice: keep the tree's copy
                    self.dpool.release(s)
            else:
                nd.dev = r.slots[pos:pos + L]
            nd.last_access = now
            pos += L
        if pos < len(r.tokens):
            nd = self._add_child(nodes[-1] if nodes else self.root, r.tokens[pos:])
            nd.dev, nd.last_access = r.slots[pos:], now
        del self.reqs[rid]

    def abort(self, rid: int) -> None:
        r = self.reqs[rid]
        if r.state == "queued":
            self.queue.remove(rid)
            del self.reqs[rid]
            return
        nodes, _ = self._align(self._key(rid))
        pos = 0
        for nd in nodes:
            if pos < r.k:
                nd.ref -= 1
            elif nd.mark:
                nd.tref -= 1
            pos += len(nd.key)
        for s in r.slots[r.k:]:
            self.dpool.release(s)
        for nd in reversed(nodes):          # drop in-flight nodes nobody covers any more
            if nd.mark == IN_FLIGHT and nd.tref == 0 and not nd.children:
                del nd.parent.children[nd.key[0]]
            else:
                break
        del self.reqs[rid]

    # ---------------------------------------------------------------- cache-controller plans
    def plan(self, which: str):
        return runs(self.load_pairs if which == "load" else self.offload_pairs, self.C, self.P)

    def dump(self):
        """Canonical tree state for parity: sorted by path."""
        rows = []
        for n in self._nodes():
            rows.append((self.path(n), tuple(n.dev), tuple(n.host), n.mark, n.tref, n.ref,
                         n.last_access))
        return sorted(rows)


def runs(pairs, C: int, P: int):
    """R25: split (host slot, device slot) pairs into strata_xfer requests.

    Consecutive pairs stay in one request iff both sides continue the chunk / page walk of
    include/strata.h (next offset, or offset 0 of any next chunk / page).  Returns the flat arrays
    of strata_xfer: num_tokens, chunk_start, chunk_offset, host_chunks, page_start, page_offset,
    dev_pages.
    """
    groups: List[List[Tuple[int, int]]] = []
    for h, d in pairs:
        if groups:
            ph, pd = groups[-1][-1]
            hc = (h % C == 0) if ph % C == C - 1 else (h == ph + 1)
            dc = (d % P == 0) if pd % P == P - 1 else (d == pd + 1)
            if hc and dc:
                groups[-1].append((h, d))
                continue
        groups.append([(h, d)])
    out = {k: [] for k in ("num_tokens", "chunk_start", "chunk_offset", "host_chunks",
                           "page_start", "page_offset", "dev_pages")}
    for g in groups:
        out["num_tokens"].append(len(g))
        out["chunk_start"].append(len(out["host_chunks"]))
        out["page_start"].append(len(out["dev_pages"]))
        out["chunk_offset"].append(g[0][0] % C)
        out["page_offset"].append(g[0][1] % P)
        for j, (h, d) in enumerate(g):
            if j == 0 or h % C == 0:
                out["host_chunks"].append(h // C)
            if j == 0 or d % P == 0:
                out["dev_pages"].append(d // P)
    return out


def bubble_steps(t_load_ms: float, t_comp_ms: float, decode_step_ms: float, decode_reqs: int,
                 enabled: bool = True) -> int:
    """Bubble filling: decode steps that fit in the loading stall."""
    if not enabled or decode_reqs <= 0 or decode_step_ms <= 0 or t_load_ms <= t_comp_ms:
        return 0
    return int((t_load_ms - t_comp_ms) // decode_step_ms)
