#!/usr/bin/env python
"""Small-load latency: eager strata_load vs CUDA-graph replay (short prefixes, "without performance
degradation in small context scenarios").

For short cached prefixes the call is bound by host work (Python/ctypes marshalling, planning,
per-layer launches + event records), not by the link.  Request tables travel in kernel parameters,
so the same load can be captured once into a CUDA graph and replayed; the graph re-reads the host
tier at replay time.  Reports the median wall time from issue to completion (host clock, stream
synchronised) and the device time between events, for eager calls and graph replays.
One JSON object per line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="1024,4096,16384")
    ap.add_argument("--engines", default="1,2")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    cases = [("tiny", 1024)] + [("llama8b_32k", int(t)) for t in args.tokens.split(",")]
    for cfg, n in cases:
        g = kvgen.geometry(cfg)
        q = kvgen.make_requests(kvgen.rng_for(3), [n], g.P, g.C, g.num_pages, g.num_chunks)
        nb = g.num_pages * g.P * g.token_bytes
        k = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        v = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P,
                           chunk_tokens=g.C, k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
        reqs = st.Requests.from_kvgen(q)
        nbytes = 2 * g.L * n * g.token_bytes
        s = torch.cuda.Stream()
        for eng in [int(x) for x in args.engines.split(",")]:
            def eager():
                pool.load(reqs, stream=s, engine=eng)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                eager()
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=s):
                pool.load(reqs, stream=torch.cuda.current_stream(), engine=eng)
            for mode, fn in (("eager", eager), ("graph", graph.replay)):
                walls, devs = [], []
                for i in range(args.reps + 5):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    with torch.cuda.stream(s):
                        a.record(s)
                        fn()
                        b.record(s)
                    b.synchronize()
                    if i >= 5:
                        walls.append((time.perf_counter() - t0) * 1e6)
                        devs.append(a.elapsed_time(b) * 1e3)
                w = statistics.median(walls)
                print(json.dumps({"config": cfg, "tokens": n, "layers": g.L, "bytes": nbytes, "engine": eng,
                                  "mode": mode, "wall_us": round(w, 1), "device_us": round(statistics.median(devs), 1),
                                  "gbs_wall": round(nbytes / (w / 1e6) / 1e9, 2)}), flush=True)
        pool.close()
        del k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
