#!/usr/bin/env python
"""PCIe link evidence independent of CUDA-event timing (SURVEY.md §8d "PCIe timeline"; nsys is not
in this image, NVML is).

For each engine and direction on the Llama-8B 32K workload (4 GiB per operation):
  * NVML PCIe byte counters (NVML_FI_DEV_PCIE_COUNT_RX_BYTES / TX_BYTES), read every 5 ms during K
    back-to-back operations and accumulated modulo 2^32 (they are 32-bit counters: a first version
    that read them only before and after saw them wrap): bytes that crossed the link per operation
    against the algorithmic bytes (the link-side "traffic"),
  * nvmlDeviceGetPcieThroughput samples (NVML's ~20 ms windows) during the operations: a timeline
    of link throughput that must sit at the event-timed rate for the whole run.
One JSON line per (engine, direction).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import pynvml  # noqa: E402
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def counters(h):
    vals = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_PCIE_COUNT_RX_BYTES,
                                               pynvml.NVML_FI_DEV_PCIE_COUNT_TX_BYTES])
    out = []
    for v in vals:
        if v.nvmlReturn != pynvml.NVML_SUCCESS:
            out.append(None)
        else:
            out.append(int(v.value.ullVal))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", type=int, default=10)
    ap.add_argument("--engines", default="4,1,2")
    args = ap.parse_args()
    pynvml.nvmlInit()
    torch.cuda.set_device(0)
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    g = kvgen.geometry("llama8b_32k")
    q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    kvgen.fill_random(pool.host, 7)
    reqs = st.Requests.from_kvgen(q)
    alg = 2 * g.L * q.total_tokens * g.token_bytes
    io = torch.cuda.Stream()
    for eng in [int(x) for x in args.engines.split(",")]:
        for direction in ("load", "offload"):
            if direction == "offload" and eng == st.STRATA_ENGINE_TMA:
                continue
            op = pool.load if direction == "load" else pool.offload
            op(reqs, stream=io, engine=eng)
            torch.cuda.synchronize()
            samples = []
            acc = [0, 0]
            stop = False

            def sampler():
                key = pynvml.NVML_PCIE_UTIL_RX_BYTES if direction == "load" else pynvml.NVML_PCIE_UTIL_TX_BYTES
                prev = counters(h)
                n = 0
                while not stop:
                    cur = counters(h)
                    for i in (0, 1):
                        if prev[i] is not None and cur[i] is not None:
                            acc[i] += (cur[i] - prev[i]) % (1 << 32)
                    prev = cur
                    n += 1
                    if n % 4 == 0:
                        try:
                            samples.append(pynvml.nvmlDeviceGetPcieThroughput(h, key) * 1024 / 1e9)   # KB/s -> GB/s
                        except pynvml.NVMLError:
                            pass
                    time.sleep(0.005)
            t = threading.Thread(target=sampler, daemon=True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t.start()
            a.record(io)
            for _ in range(args.ops):
                op(reqs, stream=io, engine=eng)
            b.record(io)
            b.synchronize()
            stop = True
            t.join()
            ms = a.elapsed_time(b)
            rec = {"engine": {1: "ldg", 2: "tma", 4: "dma"}[eng], "direction": direction, "ops": args.ops,
                   "algorithmic_bytes_per_op": alg, "event_gbs": round(args.ops * alg / (ms / 1e3) / 1e9, 2)}
            for name, i in (("rx", 0), ("tx", 1)):
                rec[f"pcie_{name}_bytes_per_op"] = acc[i] // args.ops
                rec[f"pcie_{name}_over_algorithmic"] = round(acc[i] / args.ops / alg, 4)
            if samples:
                mid = samples[len(samples) // 10: len(samples) - len(samples) // 10] or samples
                rec["nvml_throughput_gbs"] = {"median": round(statistics.median(mid), 2),
                                              "p10": round(sorted(mid)[len(mid) // 10], 2),
                                              "max": round(max(mid), 2), "samples": len(samples)}
            print(json.dumps(rec), flush=True)
    pool.close()


if __name__ == "__main__":
    main()
