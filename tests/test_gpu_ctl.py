"""The control plane drives the CUDA data path end to end, on the GPU.

Every token position of every stored prefix gets a 64-bit tag (a hash of the prefix).  The host
tier and the device pool only ever receive tags: the test writes them for contexts it inserts and
for the tokens a batch prefills (the stand-in for the model), and everything else moves through
the plans the native scheduler emits — WRITE-BACK via strata_offload, then LOAD via strata_load,
on one stream.  After every round:
  * each dispatched request's page table (strata_ctl_req_slots) holds, for its cached prefix, the
    tags of that prefix on the device (the load moved the right host rows to the right pages), and
  * every committed node of the tree holds its own tags at each of its device slots and each of its
    host slots (write-backs landed; nothing else was overwritten).
Bit-exact; both the zero-copy (LDG) and copy-engine (DMA) engines.
"""
import hashlib

import numpy as np
import pytest

from kvgen import traces

pytestmark = pytest.mark.gpu

L, H, D, E = 2, 2, 64, 2
ROW = H * D * E


def _tag(prefix) -> np.ndarray:
    h = hashlib.blake2b(np.asarray(prefix, np.int32).tobytes(), digest_size=8).digest()
    return np.tile(np.frombuffer(h, np.uint8), ROW // 8)


class Tier:
    def __init__(self, P, C, num_pages, num_chunks):
        import torch

        import paper_2508_18572_b200 as st
        self.P, self.C = P, C
        self.num_pages, self.num_chunks = num_pages, num_chunks
        self.k = [torch.zeros(num_pages * P * ROW, dtype=torch.uint8, device="cuda") for _ in range(L)]
        self.v = [torch.zeros(num_pages * P * ROW, dtype=torch.uint8, device="cuda") for _ in range(L)]
        self.pool = st.HostPool(num_layers=L, num_heads=H, head_dim=D, elem_bytes=E, page_size=P,
                                chunk_tokens=C, k_ptrs=self.k, v_ptrs=self.v, num_pages=num_pages,
                                num_chunks=num_chunks)
        self.hv = self.pool.host[: num_chunks * L * 2 * C * ROW].reshape(num_chunks, L, 2, C, ROW)

    def write_host(self, slots, rows):
        for s, r in zip(slots, rows):
            self.hv[s // self.C, :, :, s % self.C, :] = r

    def write_dev(self, slots, rows):
        import torch
        if len(slots) == 0:
            return
        idx = torch.as_tensor(np.asarray(slots, np.int64), device="cuda")
        val = torch.as_tensor(np.stack(rows), device="cuda")
        for buf in self.k + self.v:
            buf.view(-1, ROW).index_copy_(0, idx, val)

    def dev_rows(self, slots):
        import torch
        idx = torch.as_tensor(np.asarray(slots, np.int64), device="cuda")
        return [buf.view(-1, ROW).index_select(0, idx).cpu().numpy() for buf in self.k + self.v]

    def host_rows(self, slots):
        s = np.asarray(slots, np.int64)
        return [self.hv[s // self.C, l, kv, s % self.C, :] for l in range(L) for kv in range(2)]


def _run_plans(ctl, tier, engine, stream):
    keep = []
    wb = ctl.xfer("writeback")
    if wb is not None:
        tier.pool.offload(wb, stream=stream, engine=engine)
        keep.append(wb)
    ld = ctl.xfer("load")
    if ld is not None:
        tier.pool.load(ld, stream=stream, engine=engine)
        keep.append(ld)
    return keep


def _check_tree(ctl, tier):
    for path, dev, host, mark, _, _, _ in ctl.dump():
        if mark:
            continue
        start = len(path) - max(len(dev), len(host))
        want = np.stack([_tag(path[: start + j + 1]) for j in range(max(len(dev), len(host)))])
        if dev:
            for got in tier.dev_rows(dev):
                np.testing.assert_array_equal(got, want)
        if host:
            for got in tier.host_rows(host):
                np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("P,C,engine", [(1, 16, 1), (4, 16, 1), (16, 64, 1), (4, 16, 4), (1, 8, 4)])
def test_ctl_plans_drive_load_and_writeback(P, C, engine):
    import torch

    from paper_2508_18572_b200 import ctl as ctl_mod
    rng = np.random.default_rng(P * 7 + C + engine)
    num_pages, num_chunks = 1200 // P, 6000 // C
    tier = Tier(P, C, num_pages, num_chunks)
    ctl = ctl_mod.Ctl(P, C, num_pages, num_chunks, threshold=20, ratio=4.0, max_batch_tokens=700,
                      max_batch_reqs=4)
    stream = torch.cuda.current_stream().cuda_stream
    fam = traces.random_prefix_family(rng, 200, 300, vocab=3, branch=0.85)
    for j in range(10):                                   # contexts offloaded earlier
        toks = fam[j]
        slots = ctl.insert(toks, ctl_mod.HOST, 0.0)
        tier.write_host(slots, [_tag(toks[: i + 1]) for i in range(len(toks))])
    rid, t, loaded, written = 0, 1.0, 0, 0
    live = {}
    for rnd in range(40):
        for _ in range(int(rng.integers(1, 4))):
            toks = fam[int(rng.integers(0, len(fam)))] + rng.integers(0, 3, int(rng.integers(1, 30))).tolist()
            ctl.submit(rid, toks)
            live[rid] = toks
            rid += 1
        out = ctl.schedule(t)
        keep = _run_plans(ctl, tier, engine, stream)
        loaded += out["load_tokens"]
        written += out["writeback_tokens"]
        torch.cuda.synchronize()
        for r in out["batch"]:
            toks = live[r]
            slots = ctl.req_slots(r)
            k = ctl.match(toks[:-1])["device"]
            if k:
                want = np.stack([_tag(toks[: i + 1]) for i in range(k)])
                for got in tier.dev_rows(slots[:k]):
                    np.testing.assert_array_equal(got, want)   # cached prefix arrived on the device
            tier.write_dev(slots[k:], [_tag(toks[: i + 1]) for i in range(k, len(toks))])  # "prefill"
        torch.cuda.synchronize()
        for r in out["batch"]:
            ctl.complete(r, t + 0.5)
            del live[r]
        _check_tree(ctl, tier)
        del keep
        t += 1.0
    assert loaded > 0 and written > 0
    tier.pool.close()
