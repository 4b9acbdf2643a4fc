"""N>1 host-side logic on CPU (gloo, world_size 2): KV-head sharding across ranks
and the max-over-ranks timing reduction bench.py uses.  Each rank loads only its head slice from
its own host tier; the gathered union must equal the full-head load."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import kvgen
        import oracle
        from kvgen import Geometry
        oracle.build()
        H_total = 8
        full = Geometry(L=3, H=H_total, D=16, e=2, P=4, C=8, num_pages=64, num_chunks=16)
        rng = kvgen.rng_for(42)      # identical tables on every rank (TP ranks share the mapping)
        host_full = kvgen.random_bytes(rng, full.host_bytes)
        q = kvgen.make_requests(rng, [37, 70], full.P, full.C, full.num_pages, full.num_chunks, offsets=True)
        hs = kvgen.head_slice(rank, world, H_total)
        g = Geometry(full.L, len(hs), full.D, full.e, full.P, full.C, full.num_pages, full.num_chunks)
        # this rank's host tier holds only its heads (layout R1 with H_loc = H/T, R13)
        host = np.ascontiguousarray(
            host_full.reshape(full.num_chunks, full.L, 2, full.C, H_total, full.D * full.e)[:, :, :, :, hs.start:hs.stop]
        ).reshape(-1)
        nb = g.num_pages * g.P * g.token_bytes
        k = [np.zeros(nb, np.uint8) for _ in range(g.L)]
        v = [np.zeros(nb, np.uint8) for _ in range(g.L)]
        oracle.load(g, host, k, v, q, 0, g.L)
        mine = torch.from_numpy(np.stack(k + v))
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        # timing reduction: max over ranks
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            nbf = full.num_pages * full.P * full.token_bytes
            kf = [np.zeros(nbf, np.uint8) for _ in range(full.L)]
            vf = [np.zeros(nbf, np.uint8) for _ in range(full.L)]
            oracle.load(full, host_full, kf, vf, q, 0, full.L)
            ok = True
            hl = H_total // world
            for i, img in enumerate(kf + vf):
                cat = np.concatenate([p[i].numpy().reshape(-1, hl, full.D * full.e) for p in parts], axis=1)
                ok &= np.array_equal(img.reshape(-1, H_total, full.D * full.e), cat)
            out_q.put((bool(ok), float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_head_sharded_union_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    ok, tmax = q.get(timeout=10)
    assert ok, "union of head-slice loads differs from the full-head load"
    assert tmax == float(world)


def test_head_slice_partition():
    import kvgen
    for H, T in [(8, 1), (8, 2), (8, 4), (8, 8), (4, 2)]:
        seen = []
        for r in range(T):
            seen += list(kvgen.head_slice(r, T, H))
        assert seen == list(range(H))
    with pytest.raises(ValueError):
        kvgen.head_slice(0, 3, 8)


def _ctl_worker(rank, world, port, out_q):
    """Every TP rank runs its own native control plane on the same request stream; its plans index
    the same pages and chunks of its head slice, so they must be identical without any collective
    on the data path.  Ranks compare digests of every round with all_gather."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hashlib

        from kvgen import traces
        from paper_2508_18572_b200 import ctl as ctl_mod
        rng = np.random.default_rng(7)             # the request stream every rank receives
        fam = traces.random_prefix_family(rng, 200, 120, vocab=4, branch=0.8)
        c = ctl_mod.Ctl(4, 16, 300, 200, threshold=20, ratio=4.0, max_batch_reqs=4, max_batch_tokens=500)
        same = True
        rid, t = 0, 0.0
        for rnd in range(40):
            for _ in range(3):
                c.submit(rid, fam[(rid * 7) % len(fam)] + [rid % 4, (rid // 4) % 4])
                rid += 1
            out = c.schedule(t)
            h = hashlib.sha256(repr((out, c.plan("load"), c.plan("writeback"))).encode()).digest()
            mine = torch.frombuffer(bytearray(h), dtype=torch.uint8)
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)
            same &= all(torch.equal(p, parts[0]) for p in parts)
            for r in out["batch"]:
                c.complete(r, t + 0.5)
            t += 1.0
        if rank == 0:
            out_q.put(bool(same))
    finally:
        dist.destroy_process_group()


def test_control_plane_identical_across_tp_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ctl_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    assert q.get(timeout=10), "TP ranks' control planes diverged"


def _shared_tier_worker(rank, world, port, path, out_q):
    """Rank 0 creates a file-backed tier holding all heads (head-major, R28) and fills it; every
    rank maps the SAME file (paper_2508_18572_b200.shared_tier) and loads its head slice."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import dataclasses

        import kvgen
        import oracle
        from kvgen import Geometry
        from paper_2508_18572_b200.shared_tier import SharedTier
        oracle.build()
        H_total = 4
        full = Geometry(L=2, H=H_total, D=16, e=2, P=2, C=8, num_pages=64, num_chunks=12, Ht=H_total,
                        head_major=True)
        if rank == 0:
            tier = SharedTier(path, full.host_bytes, create=True)
            tier.array[:] = kvgen.random_bytes(kvgen.rng_for(5), full.host_bytes)
        dist.barrier()
        if rank != 0:
            tier = SharedTier(path, full.host_bytes, create=False)
        q = kvgen.make_requests(kvgen.rng_for(6), [40, 9], full.P, full.C, full.num_pages, full.num_chunks,
                                offsets=True)
        hs = kvgen.head_slice(rank, world, H_total)
        g = dataclasses.replace(full, H=len(hs), h0=hs.start)
        nb = g.num_pages * g.P * g.token_bytes
        k = [np.zeros(nb, np.uint8) for _ in range(g.L)]
        v = [np.zeros(nb, np.uint8) for _ in range(g.L)]
        oracle.load(g, tier.array, k, v, q, 0, g.L)
        parts = [torch.empty((2 * g.L, nb), dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(np.stack(k + v)))
        dist.barrier()
        if rank == 0:
            nbf = full.num_pages * full.P * full.token_bytes
            kf = [np.zeros(nbf, np.uint8) for _ in range(full.L)]
            vf = [np.zeros(nbf, np.uint8) for _ in range(full.L)]
            oracle.load(full, tier.array, kf, vf, q, 0, full.L)
            hl = H_total // world
            ok = all(np.array_equal(img.reshape(-1, H_total, full.D * full.e),
                                    np.concatenate([p[i].numpy().reshape(-1, hl, full.D * full.e) for p in parts], 1))
                     for i, img in enumerate(kf + vf))
            out_q.put(bool(ok))
        dist.barrier()
        tier.close()
    finally:
        dist.destroy_process_group()


def test_shared_tier_across_ranks_gloo(tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "tier.bin")
    procs = [ctx.Process(target=_shared_tier_worker, args=(r, world, port, path, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    assert q.get(timeout=10), "head slices of the shared tier do not reassemble the full-head load"
    assert not os.path.exists(path), "creator did not unlink the shared tier"


def _bench_reduce_worker(rank, world, port, out_q):
    """bench.py's own multi-rank reduction and reporting code (reduce_max, gather_floats,
    scale_record) under gloo: rank r took (1 + r) s for its steps and saw a link of (50 + r) GB/s."""
    import sys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        cv_max = bench.reduce_max(dist, world, 0.01 * (rank + 1))
        per_rank = bench.gather_floats(dist, world, [1.0 + rank, 50.0 + rank])
        rec = bench.scale_record(per_rank, bytes_per_step_per_rank=10 ** 9, steps=10)
        if rank == 0:
            out_q.put((cv_max, per_rank, rec))
    finally:
        dist.destroy_process_group()


def test_bench_reductions_gloo():
    """Weak-scaling aggregate = all ranks' bytes over the SLOWEST rank's time; each rank's fraction is
    of its OWN concurrently measured link; the line reports the minimum."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_reduce_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    cv_max, per_rank, rec = q.get(timeout=10)
    assert cv_max == pytest.approx(0.02)
    assert per_rank == [[1.0, 50.0], [2.0, 51.0]]
    assert rec["value"] == pytest.approx(2 * 10 * 1e9 / 2.0 / 1e9)       # 10 GB/s over the max time
    assert rec["per_rank_gbs"] == [10.0, 5.0]
    assert rec["per_rank_frac_of_link"] == [round(10.0 / 50.0, 4), round(5.0 / 51.0, 4)]
    assert rec["min_frac_over_ranks"] == round(5.0 / 51.0, 4)
