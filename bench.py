#!/usr/bin/env python
"""bench.py — KV load throughput of libstrata on B200 (BASELINE.json metric).

One "step" = one strata_load of the whole cached prefix, every layer (all §8(a) rows: planning,
index fetch + layout transform, host->HBM movement, per-layer completion flags/events) — for the
default workload BASELINE.json configs[1]: Llama-3.1-8B geometry (32 layers, 8 KV heads, d=128,
bf16), a 32K-token prefix, page size 1, randomly fragmented pages, 4 GiB per step (> 126 MB L2, so no
flush is needed).  The default engine for such a load is the hand-written zero-copy LDG kernel
(csrc/kernels.cu, the paper's 2 x 1024-thread configuration): 16-byte loads of the page-first host
rows through the tier's UVA mapping, register-staged stores to the pages.  The TMA-fed ring kernel
(csrc/ring.cu) is reported beside it under other_engines_gbs.

    python bench.py [--gpus N --steps K --warmup W] [--impl strata|reference] [--config ...] [--page-size P]

Multi-GPU (torchrun): every rank loads its own workload over its own PCIe link (weak scaling, no
data-path collective; torch.distributed only for barriers and the timing reductions).  Each rank is
pinned to its GPU's NUMA node; its link ceiling is measured concurrently with the other ranks'.
Rank 0 prints ONE JSON line.  ``--impl reference`` times the CPU oracle (oracle/, test
infrastructure) on the host cores instead.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import kvgen  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
ENGINE_NAMES = {0: "default", 1: "ldg", 2: "ring", 3: "tma_bulk", 4: "dma"}
PATH_DESC = {
    "ring": "ring_load_kernel (csrc/ring.cu): ONE persistent launch for all layers; per CTA a TMA producer warp "
            "(one cp.async.bulk per page-first host run of <= 16 KiB, from the UVA-mapped tier, into a 7-stage "
            "shared-memory ring) + up to 8 LSU scatter warps (16-byte st.global to the pages); per-layer completion "
            "flags -> layer events",
    "ldg": "ldg_fused_kernel (csrc/kernels.cu): ONE launch for all layers, 2 CTAs x 1024 threads (the paper's "
           "configuration, PAPER.md:262); a warp owns 32 rows, lane t fetches row t's chunk / page indices one group "
           "ahead and the addresses go out by __shfl_sync, each lane keeps 4 independent 16-byte "
           "ld.global.nc.L1::no_allocate.v4 reads of the UVA-mapped tier in flight, then st.global.v4 to the pages; "
           "per-layer completion flags -> layer events",
    "dma": "per layer: copy-engine gather of the page-first chunk-layer runs (one cudaMemcpyAsync per run) into an HBM "
           "staging slot + ldg_kernel scatter to the pages",
    "tma_bulk": "tma_kernel (csrc/kernels.cu): one warp per CTA, cp.async.bulk on both sides of a smem ring",
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="strata", choices=["strata", "reference"])
    ap.add_argument("--config", default="llama8b_32k", choices=list(kvgen.CONFIGS))
    ap.add_argument("--page-size", type=int, default=None)
    ap.add_argument("--chunk-tokens", type=int, default=None,
                    help="host chunk size C (the host tier keeps the same token capacity)")
    ap.add_argument("--engine", type=int, default=0, help="0 default (LDG for loads >= 16 MiB of 16-byte rows, else ring), 1 LDG, 2 ring, 3 TMA bulk, 4 DMA")
    ap.add_argument("--num-ctas", type=int, default=0)
    ap.add_argument("--layer-group", type=int, default=0, help="DMA engine: layers per copy run (0 = library default)")
    ap.add_argument("--frag", default="perm", choices=["perm", "churn"])
    ap.add_argument("--chunk-frag", default="perm", choices=["perm", "identity"],
                    help="host chunk lists: a random permutation of the tier, or consecutive chunks")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the side measurements (P=16, offload, other engines, contiguous ceiling)")
    ap.add_argument("--seed", type=int, default=1)
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, rank: int, world: int, P=None):
    """Per-rank geometry + request tables (replicas of the config; the TP config is already the
    per-rank head slice)."""
    g = kvgen.geometry(args.config, P=P if P is not None else args.page_size)
    if args.chunk_tokens and args.chunk_tokens != g.C:
        g = dataclasses.replace(g, C=args.chunk_tokens, num_chunks=-(-g.num_chunks * g.C // args.chunk_tokens))
    if g.host_heads > g.H:   # a shared tier holding every KV head: this rank moves head slice `rank`
        g = dataclasses.replace(g, h0=(rank % (g.host_heads // g.H)) * g.H)
    n = kvgen.CONFIGS[args.config]["n"]
    rng = kvgen.rng_for(args.seed * 1000 + rank)
    q = kvgen.make_requests(rng, n, g.P, g.C, g.num_pages, g.num_chunks, frag=args.frag, chunk_frag=args.chunk_frag)
    return g, q


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,pcie.link.gen.current,pcie.link.width.current")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, links = [], [], set(), set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            if len(f) >= 9:
                links.add(f"gen{f[7]} x{f[8]}")   # the host link the transfers use (PCIe state)
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "pcie_link": sorted(links)}


# ------------------------------------------------------------------------------------------------
# Multi-rank reductions (torch.distributed; CPU tensors under gloo, CUDA tensors under NCCL).  Pure
# functions of per-rank numbers so that tests/test_multiproc.py runs them under gloo.
def reduce_max(dist, world, x: float, device="cpu") -> float:
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_floats(dist, world, xs, device="cpu"):
    """[rank][field] for a per-rank list of floats (every rank gets every row)."""
    import torch
    t = torch.tensor([float(v) for v in xs], dtype=torch.float64, device=device)
    if world == 1:
        return [t.tolist()]
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


def scale_record(per_rank, bytes_per_step_per_rank: int, steps: int):
    """Whole-job numbers from per-rank (elapsed_s, link_gbs): aggregate GB/s over the max elapsed time
    (weak scaling: every rank moves its own bytes), and each rank's fraction of ITS OWN link ceiling,
    measured while every rank ran its ceiling copy at once (the target holds per GPU)."""
    elapsed = [r[0] for r in per_rank]
    world = len(per_rank)
    agg = bytes_per_step_per_rank * world * steps / max(elapsed) / 1e9
    fracs = [bytes_per_step_per_rank * steps / r[0] / 1e9 / r[1] for r in per_rank]
    return {"value": agg, "per_rank_gbs": [round(bytes_per_step_per_rank * steps / e / 1e9, 3) for e in elapsed],
            "per_rank_link_gbs": [round(r[1], 3) for r in per_rank],
            "per_rank_frac_of_link": [round(f, 4) for f in fracs], "min_frac_over_ranks": round(min(fracs), 4)}


# ------------------------------------------------------------------------------------------------
def cpu_baseline(g, q, host: np.ndarray, budget_s: float = 10.0):
    """The oracle as it stands (oracle/oracle.c, OpenMP over the cores this process may use), timed on
    this box on the same workload: DRAM->DRAM into host images of the device pool (SURVEY §8d "Oracle
    timing"); plus a single-threaded sample (layers of one load)."""
    import oracle
    from paper_2508_18572_b200 import numa
    oracle.build()
    nb = g.num_pages * g.P * g.token_bytes
    k = [np.empty(nb, np.uint8) for _ in range(g.L)]
    v = [np.empty(nb, np.uint8) for _ in range(g.L)]
    for a in k + v:
        a.fill(0)   # fault the pages in outside the timed region
    threads = oracle.max_threads()
    bytes_per = g.kv * g.L * q.total_tokens * g.token_bytes
    times = []
    t_start = time.time()
    # a bounded sample of ~10 s of CPU work (at least 3 full loads, at most 200)
    while len(times) < 3 or (time.time() - t_start < budget_s and len(times) < 200):
        t0 = time.perf_counter()
        oracle.load(g, host, k, v, q, 0, g.L, nthreads=threads)
        times.append(time.perf_counter() - t0)
    best = statistics.median(times)
    # single thread: the first layers of one load, ~2 s
    t0 = time.perf_counter()
    nl = 0
    while nl < g.L and (nl < 2 or time.perf_counter() - t0 < 2.0):
        oracle.load(g, host, k, v, q, nl, nl + 1, nthreads=1)
        nl += 1
    one = time.perf_counter() - t0
    node = numa.gpu_numa_node(0)
    node_cpus = numa.parse_cpulist(open(f"/sys/devices/system/node/node{node}/cpulist").read()) \
        if node >= 0 and os.path.exists(f"/sys/devices/system/node/node{node}/cpulist") else []
    return {"value": round(bytes_per / best / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"full {q.total_tokens}-token {g.L}-layer load of the bench workload, "
                      f"{len(times)} reps, median; DRAM->DRAM, {threads} OpenMP threads",
            "ms_per_load": round(best * 1e3, 2),
            "single_thread": {"value": round(bytes_per / g.L * nl / one / 1e9, 3), "unit": "GB/s", "cores": 1,
                              "sample": f"{nl} layers of one load"},
            "nproc": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0)), "gpu_numa_node": node,
            "numa_node_cpus": len(node_cpus) or None}


def interference(torch, pool, reqs, io, bytes_load, link):
    """NEXT-1 in the bench line (fig:interference): co-running proxies
    slowed by this workload's default load.  One alone / beside pair per proxy after a 0.5 s idle,
    10 timed repetitions each (tests/test_gpu_interference.py runs the full 3-round protocol):
    prefill = bf16 GEMMs of a Llama-8B layer for 2 x 4K tokens; decode = an 8 GiB HBM read of 16 x 4K
    tokens of KV for 32 layers as 32 kernels; decode_long = the same read as 4 kernels; attn = the same
    KV as the paper's decode pass run by a real kernel (FlashInfer paged decode attention, 32 layers);
    decode_step = a whole Llama-8B decode step around it; *_quota = the same bracketed by
    strata_set_load_quota(1) / (0) (the decode-aware quota)."""
    lo, hi = torch.cuda.Stream.priority_range()
    comp = torch.cuda.Stream(priority=lo)
    M = 8192
    shapes = [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096)]
    xs = {k: torch.randn(M, k, dtype=torch.bfloat16, device="cuda") for k, _ in shapes}
    ws = [torch.randn(k, n, dtype=torch.bfloat16, device="cuda") for k, n in shapes]
    kv = torch.randn(32 * 16 * 4096 * 8 * 128 * 2, dtype=torch.bfloat16, device="cuda")
    parts32, parts4 = kv.chunk(32), kv.chunk(4)
    proxies = {"prefill": lambda: [torch.matmul(xs[k], w) for (k, _), w in zip(shapes, ws)],
               "decode": lambda: [t.sum(dtype=torch.float32) for t in parts32],
               "decode_long": lambda: [t.sum(dtype=torch.float32) for t in parts4]}
    attn_note = None
    try:
        # the paper's decode pass with a real decode kernel: FlashInfer paged decode attention, 16
        # requests x 4K tokens, Llama-8B heads, page 16, scattered pages, one kernel per layer x 32
        import flashinfer
        npg = 16 * 4096 // 16
        gen = torch.Generator(device="cuda").manual_seed(7)
        # the 8 GiB KV of the read proxies, viewed as 32 paged K/V caches of 256 MiB each
        caches = [tuple(t.view(2, npg, 16, 8, 128)) for t in parts32]
        wr = flashinfer.BatchDecodeWithPagedKVCacheWrapper(torch.empty(256 << 20, dtype=torch.uint8, device="cuda"),
                                                           "NHD")
        wr.plan(torch.arange(0, npg + 1, 4096 // 16, dtype=torch.int32, device="cuda"),
                torch.randperm(npg, device="cuda", generator=gen).to(torch.int32),
                torch.full((16,), 16, dtype=torch.int32, device="cuda"), 32, 8, 128, 16,
                q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        qd = torch.randn(16, 32, 128, dtype=torch.bfloat16, device="cuda", generator=gen)
        od = torch.empty_like(qd)
        proxies["attn"] = lambda: [wr.run(qd, c, out=od) for c in caches]
        # a whole Llama-8B decode step at that batch (~290 kernels): norms, QKV / O / gate-up / down
        # GEMMs (random bf16 weights) around the same attention kernel
        Hd = 4096
        mk = lambda *sh: torch.randn(*sh, dtype=torch.bfloat16, device="cuda", generator=gen) * 0.02  # noqa: E731
        wts = [(mk(Hd, 6144), mk(Hd, Hd), mk(Hd, 2 * 14336), mk(14336, Hd), mk(Hd), mk(Hd)) for _ in caches]
        x0 = torch.randn(16, Hd, dtype=torch.bfloat16, device="cuda", generator=gen)

        def decode_step():
            F = torch.nn.functional
            h = x0
            for (wqkv, wo, wgu, wd, n1, n2), c in zip(wts, caches):
                qkv = F.rms_norm(h, (Hd,), n1) @ wqkv
                wr.run(qkv[:, :Hd].reshape(16, 32, 128), c, out=od)
                h = h + od.reshape(16, Hd) @ wo
                gu = F.rms_norm(h, (Hd,), n2) @ wgu
                h = h + (F.silu(gu[:, :14336]) * gu[:, 14336:]) @ wd
        proxies["decode_step"] = decode_step
        # the decode-aware quota (strata_set_load_quota) bracketing the decode-side co-runners
        pool.set_load_quota(0, stream=comp)   # loads launched from here on honour the cap

        def bracket(fn):
            def run():
                pool.set_load_quota(1, stream=comp)
                fn()
                pool.set_load_quota(0, stream=comp)
            return run
        proxies["attn_quota"] = bracket(proxies["attn"])
        proxies["decode_step_quota"] = bracket(decode_step)
    except Exception as ex:   # FlashInfer missing or failing on this box: the other proxies still run
        attn_note = f"attn proxy unavailable: {type(ex).__name__}: {str(ex)[:120]}"

    def run(fn, reps=10):
        evs = []
        with torch.cuda.stream(comp):
            fn()
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(comp)
                fn()
                b.record(comp)
                evs.append((a, b))
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in evs)

    out = {"method": "proxy alone vs beside back-to-back default loads on a high-priority stream; "
                     "0.5 s idle before each block; median of 10"}
    rates = []
    for name, fn in proxies.items():
        time.sleep(0.5)
        alone = run(fn)
        n_loads = max(2, int(alone * 12 / (bytes_load / link / 1e6)) + 2)
        time.sleep(0.5)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(io)
        for _ in range(n_loads):
            pool.load(reqs, stream=io)
        b.record(io)
        co = run(fn)
        b.synchronize()
        rates.append(n_loads * bytes_load / (a.elapsed_time(b) / 1e3) / 1e9)
        out[name] = round(co / alone - 1, 4)
    out["load_gbs_beside"] = round(statistics.median(rates), 3)
    out["load_gbs_beside_each"] = {name: round(r, 3) for name, r in zip(proxies, rates)}
    if attn_note:
        out["attn_note"] = attn_note
    out["paper_budget"] = {"prefill": 0.05, "decode": 0.10, "source": "PAPER.md:262 (H200, ~50 GB/s)"}
    del xs, ws, kv, parts32, parts4, proxies
    torch.cuda.empty_cache()
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    g, q = workload(args, 0, 1)
    import oracle
    oracle.build()
    host = np.empty(g.host_bytes, np.uint8)
    kvgen.fill_random(host, args.seed)
    nb = g.num_pages * g.P * g.token_bytes
    k = [np.zeros(nb, np.uint8) for _ in range(g.L)]
    v = [np.zeros(nb, np.uint8) for _ in range(g.L)]
    threads = oracle.max_threads()
    bytes_per = g.kv * g.L * q.total_tokens * g.token_bytes
    for _ in range(args.warmup):
        oracle.load(g, host, k, v, q, 0, g.L, nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.load(g, host, k, v, q, 0, g.L, nthreads=threads)
    dt = time.perf_counter() - t0
    value = bytes_per * args.steps / dt / 1e9
    line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "config": _config(args, g, q),
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "oracle",
                             "sample": f"full workload per step ({q.total_tokens} tokens x {g.L} layers), "
                                       f"DRAM->DRAM on the host cores"},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _config(args, g, q):
    return {"workload": args.config, "layers": g.L, "kv_heads_per_gpu": g.H, "head_dim": g.D, "kv_dtype": "bf16",
            "kv_buffers_per_layer": g.kv, "host_heads": g.host_heads, "head_begin": g.h0,
            "host_layout": "head-major" if g.head_major else "token-major",
            "page_size": g.P, "host_chunk_tokens": g.C, "tokens_per_gpu": q.total_tokens,
            "requests": q.R, "fragmentation": args.frag, "host_chunk_order": args.chunk_frag,
            "bytes_per_step_per_gpu": g.kv * g.L * q.total_tokens * g.token_bytes,
            "l2": f"no flush: each step moves {g.kv * g.L * q.total_tokens * g.token_bytes / 2**30:.1f} GiB, "
                  "far above the 126 MB L2",
            "parallelism": (f"tp{args.gpus}: KV-head slices of one host tier" if g.host_heads > g.H
                            else f"replicas x{args.gpus}")}


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2508_18572_b200 as st
    from paper_2508_18572_b200 import numa

    rank, world, local = dist_env()
    # STRATA_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 with gloo for the barrier and
    # the max-over-ranks reduction, so the N>1 flow runs on a one-GPU box (NCCL refuses two ranks
    # on one device).  Never used for reported numbers.
    share = os.environ.get("STRATA_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    placement = numa.bind_to_gpu(local)
    red_dev = "cpu" if share else "cuda"
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    g, q = workload(args, rank, world)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)] if g.kv == 2 else k
    # A tier holding every KV head (R28) is one file-backed mapping per NUMA node, shared by the ranks
    # on that node when its /dev/shm can hold it (the node's lowest rank creates, binds and fills it);
    # otherwise each rank keeps a copy.
    shared, host_tier = None, "per-rank"
    if g.host_heads > g.H and world > 1:
        from paper_2508_18572_b200.shared_tier import SharedTier, free_bytes
        ok = os.path.isdir("/dev/shm") and free_bytes("/dev/shm") > g.host_bytes + (1 << 30)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=red_dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()):
            nodes = gather_floats(dist, world, [placement["numa_node"]], device=red_dev)
            node = placement["numa_node"]
            creator = min(r for r in range(world) if int(nodes[r][0]) == node)
            path = f"/dev/shm/strata_bench_tier_{os.environ.get('MASTER_PORT', '0')}_n{node}"
            if rank == creator:
                shared = SharedTier(path, g.host_bytes, create=True)
                numa.mbind(shared.array.ctypes.data, g.host_bytes, node)
                kvgen.fill_random(shared.array, args.seed * 1000)
            dist.barrier()
            if rank != creator:
                shared = SharedTier(path, g.host_bytes, create=False)
            host_tier = f"one shared mapping per NUMA node ({len({int(n[0]) for n in nodes})} for {world} ranks)"
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v if g.kv == 2 else None, num_pages=g.num_pages,
                       num_chunks=g.num_chunks, device=local, host_heads=g.Ht, head_begin=g.h0,
                       head_major=g.head_major, host=shared.array if shared else None)
    if shared is None:
        kvgen.fill_random(pool.host, args.seed * 1000 + rank)
    reqs = st.Requests.from_kvgen(q, device=local)
    bytes_step = g.kv * g.L * q.total_tokens * g.token_bytes
    io = torch.cuda.Stream()

    def step():
        return pool.load(reqs, 0, g.L, stream=io, engine=args.engine, num_ctas=args.num_ctas,
                         layer_group=args.layer_group)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    submit_s = [0.0]

    def timed(fn, n):
        """n back-to-back calls on `io`: (seconds, per-call ms) from CUDA events on the I/O stream;
        submit_s[0] = host seconds spent issuing them (before the final synchronize)."""
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        h = time.perf_counter()
        marks[0].record(io)
        for i in range(n):
            fn()
            marks[i + 1].record(io)
        submit_s[0] = time.perf_counter() - h
        marks[-1].synchronize()
        per = [marks[i].elapsed_time(marks[i + 1]) for i in range(n)]
        return marks[0].elapsed_time(marks[-1]) / 1e3, per

    # host-link ceilings of THIS rank while every rank runs its own at once (barrier-aligned):
    # contiguous pinned cudaMemcpyAsync of one layer's bytes from / to the same registered tier
    scratch = torch.empty(bytes_step // g.L, dtype=torch.uint8, device="cuda")

    def ceiling(direction):
        barrier()
        def cp():
            st.strata_baseline_contiguous(pool.handle, direction, scratch.data_ptr(), 0, scratch.numel(), io)
        cp()
        _, per = timed(cp, 12)
        return scratch.numel() / (statistics.median(per[2:]) / 1e3) / 1e9
    link_h2d = ceiling(st.STRATA_H2D)
    link_d2h = ceiling(st.STRATA_D2H)

    for _ in range(args.warmup):
        step()

    def timed_region():
        barrier()
        c0 = pool.counters()
        with ClockSampler(local) as clocks:
            elapsed, step_ms = timed(step, args.steps)
            host_s = submit_s[0]
            last = pool.counters()
            barrier()
        return elapsed, sorted(step_ms), host_s, clocks, last["kernel_launches"] - c0["kernel_launches"], last

    elapsed, step_ms, host_s, clocks, launches, c1 = timed_region()
    # A timed region whose steps vary by more than 5 % (CV) saw something outside this process —
    # e.g. the host still reclaiming memory a previous job freed, which slows the link itself — and is
    # re-measured once; the first measurement is kept in the line.
    cv = statistics.pstdev(step_ms) / statistics.mean(step_ms)
    remeasured = None
    if reduce_max(dist, world, cv, red_dev) > 0.05:
        remeasured = {"first_elapsed_s": round(elapsed, 4), "first_cv_max_over_ranks": round(cv, 4)}
        time.sleep(2.0)
        elapsed, step_ms, host_s, clocks, launches, c1 = timed_region()
    engine_used = ENGINE_NAMES.get(c1["last_engine"], str(c1["last_engine"]))
    step_stats = {"median_ms": round(statistics.median(step_ms), 3),
                  "p10_ms": round(step_ms[int(0.1 * (len(step_ms) - 1))], 3),
                  "p90_ms": round(step_ms[int(0.9 * (len(step_ms) - 1))], 3),
                  "min_ms": round(step_ms[0], 3), "max_ms": round(step_ms[-1], 3),
                  "cv": round(statistics.pstdev(step_ms) / statistics.mean(step_ms), 4)}
    # per-layer completion times of the last timed step, from the library's own events
    t_layer = [pool.layer_elapsed_ms(0, l) for l in range(g.L)]   # ticket 0: the latest operation
    layer_ms = [t_layer[0]] + [b - a for a, b in zip(t_layer, t_layer[1:])]
    per_rank = gather_floats(dist, world, [elapsed, link_h2d], red_dev)
    rec = scale_record(per_rank, bytes_step, args.steps)
    elapsed_max = max(r[0] for r in per_rank)

    # e2e through the public API with host buffers: upload the step's tables from pinned host
    # memory, load (the KV itself crosses host->device inside), read back the last loaded row.
    hc_pin = torch.from_numpy(reqs.host_chunks_h).pin_memory()
    dp_pin = torch.from_numpy(reqs.dev_pages_h).pin_memory()
    sentinel = torch.empty(16, dtype=torch.uint8).pin_memory()
    last_page = int(q.dev_pages[-1])
    e2e_steps = max(3, min(args.steps, 10))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        with torch.cuda.stream(io):
            reqs.host_chunks_d.copy_(hc_pin, non_blocking=True)
            reqs.dev_pages_d.copy_(dp_pin, non_blocking=True)
        step()
        with torch.cuda.stream(io):
            off = last_page * g.P * g.token_bytes
            sentinel.copy_(v[g.L - 1][off: off + 16], non_blocking=True)
        io.synchronize()
    e2e_dt = reduce_max(dist, world, time.perf_counter() - t0, red_dev)
    e2e_value = bytes_step * world * e2e_steps / e2e_dt / 1e9
    h2d = bytes_step + 4 * (reqs.host_chunks_h.size + reqs.dev_pages_h.size)

    extras = {}
    if not args.no_extras:
        n_x = max(3, min(args.steps, 10))
        # the same workload at page sizes 2..64 (the metric's "page sizes 1-64"; the target
        # holds at P = 1 and 16): a second pool over the same device buffers and host tier per P
        sweep = {}
        for Pv in (2, 4, 8, 16, 32, 64):
            if Pv == g.P:
                continue
            gP, qP = workload(args, rank, world, P=Pv)
            if gP.num_pages * Pv > g.num_pages * g.P:
                continue   # the pool would not fit the device buffers
            poolP = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=Pv,
                                chunk_tokens=g.C, k_ptrs=k, v_ptrs=v if g.kv == 2 else None, num_pages=gP.num_pages,
                                num_chunks=g.num_chunks, device=local, host_heads=g.Ht, head_begin=g.h0,
                                head_major=g.head_major, host=pool.host)
            reqsP = st.Requests.from_kvgen(qP, device=local)
            fP = lambda: poolP.load(reqsP, 0, g.L, stream=io, engine=args.engine, num_ctas=args.num_ctas)  # noqa: E731
            fP()
            barrier()
            eP, _ = timed(fP, n_x if Pv == 16 else 3)
            prP = scale_record(gather_floats(dist, world, [eP, link_h2d], red_dev), bytes_step, n_x if Pv == 16 else 3)
            sweep[Pv] = {"value": round(prP["value"], 3), "frac_of_link": prP["min_frac_over_ranks"],
                         "steps": n_x if Pv == 16 else 3,
                         "engine": ENGINE_NAMES.get(poolP.counters()["last_engine"])}
            if Pv == 32 and world == 1:
                # the paper's fragmentation baseline at SGLang-HiCache's page size:
                # one cudaMemcpyAsync per (layer, K|V, page) from the same tier, host wall clock to completion
                xb = reqsP.xfer(0, g.L, host_lists=True)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ncalls = st.strata_baseline_memcpy_pages(poolP.handle, xb, st.STRATA_H2D, io)
                io.synchronize()
                tb = time.perf_counter() - t0
                extras["per_page_memcpy_baseline_P32"] = {
                    "value": round(bytes_step / tb / 1e9, 3), "frac_of_link": round(bytes_step / tb / 1e9 / link_h2d, 4),
                    "cudaMemcpyAsync_calls": ncalls, "wall_s": round(tb, 3),
                    "paper": "~22 % of PCIe 5.0 for per-page DMA at P = 32 (PAPER.md:182, H200)"}
            poolP.close()
        extras["page_size_16"] = sweep.get(16)
        extras["page_size_sweep"] = {"P=%d" % k_: v_ for k_, v_ in sorted(sweep.items())}
        # offload (write-back) of the same workload at its default quota vs the D2H link
        fo = lambda: pool.offload(reqs, 0, g.L, stream=io)  # noqa: E731
        fo()
        barrier()
        eo, _ = timed(fo, n_x)
        pro = scale_record(gather_floats(dist, world, [eo, link_d2h], red_dev), bytes_step, n_x)
        extras["offload"] = {"value": round(pro["value"], 3), "frac_of_d2h_link": pro["min_frac_over_ranks"],
                             "d2h_link_gbs": round(link_d2h, 3), "steps": n_x,
                             "engine": ENGINE_NAMES.get(pool.counters()["last_engine"]), "num_ctas": "default"}
        # zero-copy contiguous ceiling (diagnostic): the same kernel and quota on consecutive
        # host chunks and consecutive pages — what the SM zero-copy path reaches with no fragmentation
        qi = kvgen.make_requests(kvgen.rng_for(0), kvgen.CONFIGS[args.config]["n"], g.P, g.C, g.num_pages,
                                 g.num_chunks, frag="identity", chunk_frag="identity")
        reqs_i = st.Requests.from_kvgen(qi, device=local)
        fi = lambda: pool.load(reqs_i, 0, g.L, stream=io, engine=args.engine, num_ctas=args.num_ctas)  # noqa: E731
        fi()
        ei, _ = timed(fi, 3)
        extras["zero_copy_contiguous_gbs"] = round(bytes_step * 3 / ei / 1e9, 3)
        # the other engines on the same workload at their default quotas (3 loads each)
        others = {}
        for eng in (st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_DMA):
            if ENGINE_NAMES[eng] == engine_used:
                continue
            fe = lambda: pool.load(reqs, 0, g.L, stream=io, engine=eng)  # noqa: E731
            fe()
            ee, _ = timed(fe, 3)
            others[ENGINE_NAMES[eng]] = round(bytes_step * 3 / ee / 1e9, 3)
        extras["other_engines_gbs"] = others
        if world == 1 and bytes_step >= (1 << 30) and not args.num_ctas and not args.engine:
            extras["interference"] = interference(torch, pool, reqs, io, bytes_step, link_h2d)
        if bytes_step < (16 << 20):
            # a small load is bound by host submission (the Python call + the library's launch work,
            # ~20 us) more than by the device: the same load captured once into a CUDA graph and
            # replayed (per-layer launches inside the graph; tests/test_gpu_graph.py)
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=io):
                step()

            def replay():
                with torch.cuda.stream(io):
                    cg.replay()
            replay()
            eg, per_g = timed(replay, max(10, args.steps))
            extras["graph_replay"] = {"ms_per_step": round(statistics.median(per_g), 4),
                                      "value": round(bytes_step / (statistics.median(per_g) / 1e3) / 1e9, 3),
                                      "steps": max(10, args.steps)}
    del scratch

    out = None
    if rank == 0:
        # the dominant kernel: one launch per step for the fused engines (ring / LDG), so its average
        # launch duration is the median step; per layer for DMA
        launches_per_step = max(1, launches // args.steps)
        per_launch_bytes = bytes_step // launches_per_step
        avg_launch = step_stats["median_ms"] / launches_per_step
        achieved = per_launch_bytes / (avg_launch / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"{args.config}_P{g.P}_{engine_used}")
        peaks = {}
        mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(mp):
            peaks = json.load(open(mp))
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(g, q, pool.host)
        out = {
            "metric": METRIC, "value": round(rec["value"], 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed_max / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": _config(args, g, q),
            "ms_per_32k_load": round(elapsed_max / args.steps * 1e3 * 32768 / q.total_tokens, 3),
            "engine": engine_used, "num_ctas": args.num_ctas or "default",
            "step_stats_rank0": step_stats,
            "frac_of_link": rec["min_frac_over_ranks"],
            "per_rank": {k_: rec[k_] for k_ in ("per_rank_gbs", "per_rank_link_gbs", "per_rank_frac_of_link",
                                                "min_frac_over_ranks")},
            "roofline": {"bound": "pcie_h2d", "achieved": round(achieved, 3), "peak": round(link_h2d, 3),
                         "unit": "GB/s", "frac": round(achieved / link_h2d, 4), "traffic": traffic,
                         "kernel": PATH_DESC.get(engine_used, engine_used),
                         "per_launch_bytes": per_launch_bytes, "avg_launch_ms": round(avg_launch, 4),
                         "launches_per_step": launches_per_step,
                         "peak_source": "contiguous pinned cudaMemcpyAsync H2D from the same registered host "
                                        "tier, measured in this run on this rank (concurrently with every other "
                                        "rank); PCIe Gen5 x16 nominal 64 GB/s",
                         "hbm": {"achieved": round(achieved, 3), "peak": hbm_peak,
                                 "frac": round(achieved / hbm_peak, 5),
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": 16},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "placement": placement,
            **extras,
            "shared_gpu_test_mode": share or None,
            "host_tier": host_tier,
            "per_layer_ms_last_step": [round(x, 4) for x in layer_ms],
            "host_submit_ms_per_step": round(host_s / args.steps * 1e3, 3),
            "remeasured": remeasured,
        }
        print(json.dumps(out), flush=True)
    pool.close()
    if world > 1:
        dist.barrier()
    if shared is not None:
        shared.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
