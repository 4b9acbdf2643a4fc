#!/usr/bin/env python
"""Why copy-engine traffic slows HBM-bound work on B200 (DESIGN.md §6 "Interference").

profiles/r01/interference3.jsonl: a plain contiguous cudaMemcpyAsync H2D loop, no kernel at all,
slows the decode proxy (HBM-streaming reduction) by ~25 %, while the zero-copy LDG kernel moving
the same bytes from 1 SM costs ~4 %.  This tool separates the candidate causes by co-running
proxies with copy-engine loops that differ in one property each:

  copy loops   h2d_big    H2D 128 MiB into a 128 MiB device buffer (HBM-resident destination)
               h2d_small  H2D 4 MiB into one 4 MiB device buffer, repeated (L2-resident destination)
               d2h_big    D2H 128 MiB (the copy engine reads HBM, writes host)
               h2h        pinned host -> pinned host 64 MiB (no GPU memory touched at all)
  proxies      decode     HBM-streaming reduction over 32 x 256 MiB (the interference.py proxy)
               l2         the same reduction over a 32 MiB tensor, 256 times (L2-resident)
               alu        in-place sin() of a 4 MiB tensor, 400 times (SM-bound)

and samples SM / memory clocks and power with NVML during every phase.  decode_graph / alu_graph
are the same proxies replayed from a CUDA graph.  One JSON line per pair.
"""
from __future__ import annotations

import argparse
import json
import statistics
import threading
import time

import torch


def make_proxies():
    kv = [torch.randn(16 * 4096 * 8 * 128 * 2, dtype=torch.bfloat16, device="cuda") for _ in range(32)]
    small = torch.randn(16 << 20, dtype=torch.bfloat16, device="cuda")          # 32 MiB
    alu = torch.randn(1 << 20, dtype=torch.float32, device="cuda")              # 4 MiB

    def decode():
        for t in kv:
            t.sum(dtype=torch.float32)

    def l2():
        for _ in range(256):
            small.sum(dtype=torch.float32)

    def alu_fn():
        for _ in range(400):
            alu.sin_()
    return {"decode": decode, "l2": l2, "alu": alu_fn}


def as_graph(fn, stream):
    """The same work captured once as a CUDA graph: its launches come from device-resident work
    descriptors instead of per-kernel pushbuffer fetches (how serving engines run decode)."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            fn()
    g.replay()
    torch.cuda.synchronize()
    return g.replay


class Nvml:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.n = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.samples = []
        self.stop = False

    def __enter__(self):
        self.samples = []
        self.stop = False
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        n = self.n
        while not self.stop:
            try:
                self.samples.append((n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM),
                                     n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_MEM),
                                     n.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
            except Exception:
                pass
            time.sleep(0.02)

    def __exit__(self, *exc):
        self.stop = True
        self.t.join()

    def summary(self):
        if not self.samples:
            return {}
        sm, mem, pw = zip(*self.samples)
        return {"sm_mhz": statistics.median(sm), "mem_mhz": statistics.median(mem),
                "power_w": round(statistics.median(pw), 1)}


def time_fn(fn, stream, reps):
    evs = []
    with torch.cuda.stream(stream):
        fn()
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            evs.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=15)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    comp = torch.cuda.Stream()
    cs = torch.cuda.Stream()
    proxies = make_proxies()
    for name in ("decode", "alu"):
        proxies[name + "_graph"] = as_graph(proxies[name], comp)
    hbig = torch.empty(128 << 20, dtype=torch.uint8).pin_memory()
    hsmall = torch.empty(4 << 20, dtype=torch.uint8).pin_memory()
    hh_src = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
    hh_dst = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
    dbig = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    dsmall = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
    loops = {
        "h2d_big": (lambda: dbig.copy_(hbig, non_blocking=True), 128 << 20),
        "h2d_small": (lambda: dsmall.copy_(hsmall, non_blocking=True), 4 << 20),
        "d2h_big": (lambda: hbig.copy_(dbig, non_blocking=True), 128 << 20),
        "h2h": (lambda: hh_dst.copy_(hh_src, non_blocking=True), 64 << 20),
    }
    nv = Nvml()
    alone = {}
    for name, fn in proxies.items():
        with nv:
            alone[name] = time_fn(fn, comp, args.reps)
        print(json.dumps({"kind": "proxy_alone", "proxy": name, "ms": round(alone[name], 4), **nv.summary()}),
              flush=True)
    for lname, (cp, nbytes) in loops.items():
        # copy loop alone: bandwidth
        with torch.cuda.stream(cs):
            cp()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cs)
            for _ in range(20):
                cp()
            b.record(cs)
        b.synchronize()
        gbs = 20 * nbytes / (a.elapsed_time(b) / 1e3) / 1e9
        for pname, fn in proxies.items():
            n = int(alone[pname] * (args.reps + 2) / (nbytes / gbs / 1e6)) + 4
            torch.cuda.synchronize()
            with torch.cuda.stream(cs):
                for _ in range(n):
                    cp()
            with nv:
                t = time_fn(fn, comp, args.reps)
            torch.cuda.synchronize()
            print(json.dumps({"kind": "corun", "copy": lname, "copy_gbs_alone": round(gbs, 2), "proxy": pname,
                              "alone_ms": round(alone[pname], 4), "corun_ms": round(t, 4),
                              "slowdown": round(t / alone[pname] - 1, 4), **nv.summary()}), flush=True)


if __name__ == "__main__":
    main()
