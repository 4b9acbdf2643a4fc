#!/usr/bin/env python
"""bench.py — KV load throughput of libstrata on B200 (BASELINE.json metric).

One "step" = one strata_load of the whole cached prefix, every layer (all §8(a) rows: planning,
index fetch + layout transform, host->HBM movement, per-layer events) — for the default workload
BASELINE.json configs[1]: Llama-3.1-8B geometry (32 layers, 8 KV heads, d=128, bf16), a 32K-token
prefix, page size 1, randomly fragmented pages, 4 GiB per step (> 126 MB L2, so no flush needed).

    python bench.py [--gpus N --steps K --warmup W] [--impl strata|reference] [--config ...] [--page-size P]

Multi-GPU (torchrun): every rank loads its own replica workload over its own PCIe link (weak
scaling, no data-path collective; NCCL only for the start barrier and the max-over-ranks timing).
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
ENGINE_NAMES = {0: "default", 1: "ldg", 2: "tma", 3: "tma_bulk", 4: "dma"}
SM_ZERO_COPY_CEILING = 51.44   # GB/s, profiles/r01/probe.jsonl: SM-issued host reads, best of the sweep
PATH_DESC = {
    "dma": "per layer: copy-engine gather of the page-first chunk-layer runs (cudaMemcpyBatchAsync on one in-order copy stream) "
           "into an HBM staging slot + ldg_kernel scatter to the pages; one event per layer",
    "ldg": "ldg_kernel, zero-copy LDG/STG from mapped host memory, one launch + event per layer",
    "tma": "tma_ws_load_kernel, zero-copy cp.async.bulk ring, one launch + event per layer",
    "tma_bulk": "tma_kernel, zero-copy cp.async.bulk ring, one launch + event per layer",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="strata", choices=["strata", "reference"])
    ap.add_argument("--config", default="llama8b_32k", choices=list(kvgen.CONFIGS))
    ap.add_argument("--page-size", type=int, default=None)
    ap.add_argument("--chunk-tokens", type=int, default=None,
                    help="host chunk size C (the host tier keeps the same token capacity)")
    ap.add_argument("--engine", type=int, default=0, help="0 default, 1 LDG, 2 TMA")
    ap.add_argument("--num-ctas", type=int, default=0)
    ap.add_argument("--layer-group", type=int, default=0, help="DMA engine: layers per copy run (0 = library default)")
    ap.add_argument("--frag", default="perm", choices=["perm", "churn"])
    ap.add_argument("--chunk-frag", default="perm", choices=["perm", "identity"],
                    help="host chunk lists: a random permutation of the tier, or consecutive chunks")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, rank: int, world: int):
    """Per-rank geometry + request tables (replicas of the config; the TP config is already the
    per-rank head slice)."""
    g = kvgen.geometry(args.config, P=args.page_size)
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


def cpu_baseline(g, q, host: np.ndarray, budget_s: float = 10.0):
    """The oracle as it stands (oracle/oracle.c, OpenMP over all host cores), timed on this box on the
    same workload: DRAM->DRAM into host images of the device pool (SURVEY.md §8d "Oracle timing")."""
    import oracle
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
    return {"value": round(bytes_per / best / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"full {q.total_tokens}-token {g.L}-layer load of the bench workload, "
                      f"{len(times)} reps, median; DRAM->DRAM, {threads} OpenMP threads",
            "ms_per_load": round(best * 1e3, 2)}


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
            "requests": q.R, "fragmentation": args.frag, "host_chunk_order": args.chunk_frag, "bytes_per_step_per_gpu": g.kv * g.L * q.total_tokens * g.token_bytes,
            "l2": f"no flush: each step moves {g.kv * g.L * q.total_tokens * g.token_bytes / 2**30:.1f} GiB, "
                  "far above the 126 MB L2", "parallelism": (f"tp{args.gpus}: KV-head slices of one host tier" if g.host_heads > g.H
                            else f"replicas x{args.gpus}")}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2508_18572_b200 as st

    rank, world, local = dist_env()
    # STRATA_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 with gloo for the barrier and
    # the max-over-ranks reduction, so the N>1 flow runs on a one-GPU box (NCCL refuses two ranks
    # on one device).  Never used for reported numbers.
    share = os.environ.get("STRATA_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
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
    # A tier holding every KV head (R28) is ONE file-backed mapping shared by the ranks when the
    # node's /dev/shm can hold it (rank 0 creates and fills it); otherwise each rank keeps a copy.
    shared, host_tier = None, "per-rank"
    if g.host_heads > g.H and world > 1:
        from paper_2508_18572_b200.shared_tier import SharedTier, free_bytes
        ok = os.path.isdir("/dev/shm") and free_bytes("/dev/shm") > g.host_bytes + (1 << 30)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=red_dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()):
            path = f"/dev/shm/strata_bench_tier_{os.environ.get('MASTER_PORT', '0')}"
            if rank == 0:
                shared = SharedTier(path, g.host_bytes, create=True)
                kvgen.fill_random(shared.array, args.seed * 1000)
            dist.barrier()
            if rank != 0:
                shared = SharedTier(path, g.host_bytes, create=False)
            host_tier = f"one shared mapping for {world} ranks"
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

    for _ in range(args.warmup):
        step()
    def timed_region():
        barrier()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        c0 = pool.counters()
        with ClockSampler(local) as clocks:
            start.record(io)
            last = None
            host_s = 0.0   # CPU time inside the strata_load calls (submission; blocks only when queued ahead)
            for i in range(args.steps):
                marks[i].record(io)
                h0 = time.perf_counter()
                last = step()
                host_s += time.perf_counter() - h0
            marks[-1].record(io)
            end.record(io)
            barrier()
        c1 = pool.counters()
        step_ms = sorted(marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps))
        return (start.elapsed_time(end) / 1e3, step_ms, host_s, last, clocks,
                c1["kernel_launches"] - c0["kernel_launches"], c1)

    elapsed, step_ms, host_s, last, clocks, launches, c1 = timed_region()
    # A timed region whose steps vary by more than 5 % (CV) saw something outside this process —
    # e.g. the host still reclaiming memory a previous job freed, which slows the link itself — and is
    # re-measured once; the first measurement is kept in the line.
    cv = statistics.pstdev(step_ms) / statistics.mean(step_ms)
    tcv = torch.tensor([cv], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(tcv, op=dist.ReduceOp.MAX)
    remeasured = None
    if float(tcv.item()) > 0.05:
        remeasured = {"first_elapsed_s": round(elapsed, 4), "first_cv_max_over_ranks": round(float(tcv.item()), 4)}
        time.sleep(2.0)
        elapsed, step_ms, host_s, last, clocks, launches, c1 = timed_region()
    engine_used = ENGINE_NAMES.get(c1["last_engine"], str(c1["last_engine"]))
    step_stats = {"median_ms": round(statistics.median(step_ms), 3),
                  "p10_ms": round(step_ms[int(0.1 * (len(step_ms) - 1))], 3),
                  "p90_ms": round(step_ms[int(0.9 * (len(step_ms) - 1))], 3),
                  "min_ms": round(step_ms[0], 3), "max_ms": round(step_ms[-1], 3),
                  "cv": round(statistics.pstdev(step_ms) / statistics.mean(step_ms), 4)}
    # per-layer (= per-launch) durations of the last timed step, from the library's own events
    t_layer = [pool.layer_elapsed_ms(last, l) for l in range(g.L)]
    launch_ms = [t_layer[0]] + [b - a for a, b in zip(t_layer, t_layer[1:])]
    t = torch.tensor([elapsed], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    value = bytes_step * world * args.steps / elapsed_max / 1e9

    # link roofline: one contiguous cudaMemcpyAsync of the same bytes-per-layer from the same host tier
    scratch = torch.empty(bytes_step // g.L, dtype=torch.uint8, device="cuda")
    rt = []
    for i in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(io)
        for _l in range(4):
            st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, scratch.data_ptr(), 0, scratch.numel(), io)
        b.record(io)
        b.synchronize()
        if i >= 3:
            rt.append(4 * scratch.numel() / (a.elapsed_time(b) / 1e3) / 1e9)
    link_peak = statistics.median(rt)
    del scratch

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
            sentinel.copy_(v[g.L - 1][last_page * g.P * g.token_bytes: last_page * g.P * g.token_bytes + 16],
                           non_blocking=True)
        io.synchronize()
    e2e_dt = time.perf_counter() - t0
    te = torch.tensor([e2e_dt], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = bytes_step * world * e2e_steps / float(te.item()) / 1e9
    h2d = bytes_step + 4 * (reqs.host_chunks_h.size + reqs.dev_pages_h.size)

    # the other engines on the same workload, default SM quota, for comparison in the same line
    others = {}
    for eng in (st.STRATA_ENGINE_LDG, st.STRATA_ENGINE_TMA, st.STRATA_ENGINE_DMA):
        if ENGINE_NAMES[eng] == engine_used:
            continue
        pool.load(reqs, 0, g.L, stream=io, engine=eng)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(io)
        for _ in range(3):
            pool.load(reqs, 0, g.L, stream=io, engine=eng)
        b.record(io)
        b.synchronize()
        others[ENGINE_NAMES[eng]] = round(3 * bytes_step / (a.elapsed_time(b) / 1e3) / 1e9, 3)

    out = None
    if rank == 0:
        # per layer (= per launch for the kernel engines; per copy+scatter group for DMA): the median
        # timed step divided over its layers, from CUDA events on the I/O stream
        per_launch_bytes = bytes_step // g.L
        avg_launch = step_stats["median_ms"] / g.L
        achieved = per_launch_bytes / (avg_launch / 1e3) / 1e9
        # the hand-written zero-copy kernels against both ceilings: the link, and the SM-issued
        # zero-copy read plateau measured by tools/probe/probe.cu on this pool (51.44 GB/s)
        zc = {}
        for name in ("ldg", "tma"):
            gbs = others.get(name) if name != engine_used else round(value / world, 3)
            if gbs is not None:
                zc[name] = {"value": gbs, "frac_of_link": round(gbs / link_peak, 4),
                            "frac_of_sm_zero_copy_ceiling": round(gbs / SM_ZERO_COPY_CEILING, 4),
                            "num_ctas": "default (2 x 1024 threads)" if name == "ldg" else "default (2 x 512 threads)"}
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"{args.config}_P{g.P}_{engine_used}")
        path = PATH_DESC.get(engine_used, engine_used)
        peaks = {}
        mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(mp):
            peaks = json.load(open(mp))
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(g, q, pool.host)
        batches = -(-q.R // 128)
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed_max / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": _config(args, g, q),
            "ms_per_32k_load": round(elapsed_max / args.steps * 1e3 * 32768 / q.total_tokens, 3),
            "step_stats_rank0": step_stats,
            "frac_of_link": round(value / world / link_peak, 4),
            "roofline": {"bound": "pcie_h2d", "achieved": round(achieved, 3), "peak": round(link_peak, 3),
                         "unit": "GB/s", "frac": round(achieved / link_peak, 4), "traffic": traffic,
                         "kernel": path,
                         "per_launch_bytes": per_launch_bytes, "avg_launch_ms": round(avg_launch, 4),
                         "peak_source": "contiguous pinned cudaMemcpyAsync H2D from the same registered host "
                                        "tier, measured in this run (PCIe Gen5 x16 nominal 64 GB/s)",
                         "hbm": {"achieved": round(achieved, 3), "peak": hbm_peak,
                                 "frac": round(achieved / hbm_peak, 5),
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": 16},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "engine": engine_used, "num_ctas": args.num_ctas or "default",
            "layer_group": args.layer_group or "default",
            "other_engines_gbs": others,
            "shared_gpu_test_mode": share or None,
            "host_tier": host_tier,
            "zero_copy_kernels": zc,
            "per_layer_ms_last_step": [round(x, 4) for x in launch_ms],
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
