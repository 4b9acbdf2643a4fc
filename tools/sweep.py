#!/usr/bin/env python
"""Sweep the load/offload kernels and the copy-engine baselines on one GPU.

For each page size: engine x SM quota (num_ctas) for strata_load and strata_offload, the per-page
cudaMemcpyAsync loop and the contiguous memcpy roofline, all from the same
registered host tier.  One JSON object per line on stdout.

    python tools/sweep.py [--config llama8b_32k] [--pages 1,16] [--ctas 1,2,4,8,16,32,148]
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


def timed(fn, io, reps=5, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        a.record(io)
        fn()
        b.record(io)
        b.synchronize()
        ts.append((a.elapsed_time(b) / 1e3, time.perf_counter() - w0))
    ev = statistics.median(t[0] for t in ts)
    wall = statistics.median(t[1] for t in ts)
    return ev, wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b_32k")
    ap.add_argument("--pages", default="1,16")
    ap.add_argument("--ctas", default="1,2,4,8,16,32,148")
    ap.add_argument("--engines", default="1,2")
    ap.add_argument("--baselines", default="1")
    ap.add_argument("--layers", type=int, default=0, help="override L (0 = config)")
    ap.add_argument("--frag", default="perm")
    ap.add_argument("--chunk-frag", default="perm", help="host chunk order: perm | identity")
    ap.add_argument("--flags", type=int, default=0, help="strata_pool_desc.flags (host allocation)")
    ap.add_argument("--tag", default="")
    ap.add_argument("--threads", type=int, default=0, help="LDG engine threads per CTA (0 = default)")
    ap.add_argument("--groups", default="0", help="DMA layer_group values to sweep")
    ap.add_argument("--host-chunks", type=int, default=0, help="override the host tier capacity (chunks)")
    args = ap.parse_args()
    io = torch.cuda.Stream()
    for P in [int(x) for x in args.pages.split(",")]:
        over = {"L": args.layers} if args.layers else {}
        if args.host_chunks:
            over["num_chunks"] = args.host_chunks
        g = kvgen.geometry(args.config, P=P, **over)
        n = kvgen.CONFIGS[args.config]["n"]
        q = kvgen.make_requests(kvgen.rng_for(1), n, g.P, g.C, g.num_pages, g.num_chunks, frag=args.frag,
                                chunk_frag=args.chunk_frag)
        nb = g.num_pages * g.P * g.token_bytes
        k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)] if g.kv == 2 else None
        pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P,
                           chunk_tokens=g.C, k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks,
                           flags=args.flags, host_heads=g.Ht, head_begin=g.h0, head_major=g.head_major)
        kvgen.fill_random(pool.host, 3)
        reqs = st.Requests.from_kvgen(q)
        nbytes = g.kv * g.L * q.total_tokens * g.token_bytes
        base = {"config": args.config, "P": P, "L": g.L, "tokens": q.total_tokens, "bytes": nbytes, "frag": args.frag,
                "chunk_frag": args.chunk_frag, "flags": args.flags, "tag": args.tag,
                "host_tier_bytes": g.host_bytes}
        for eng in [int(x) for x in args.engines.split(",")]:
          for G in ([int(x) for x in args.groups.split(",")] if eng == 4 else [0]):
            for c in [int(x) for x in args.ctas.split(",")]:
                for d, fn in (("h2d", pool.load), ("d2h", pool.offload)):
                    ev, wall = timed(lambda: fn(reqs, stream=io, engine=eng, num_ctas=c, threads=args.threads,
                                                layer_group=G), io)
                    print(json.dumps({**base, "method": "strata", "dir": d, "engine": eng, "ctas": c, "threads": args.threads,
                                      "layer_group": G,
                                      "ms": round(ev * 1e3, 3), "wall_ms": round(wall * 1e3, 3),
                                      "gbs": round(nbytes / ev / 1e9, 3)}), flush=True)
        if args.baselines == "1":
            for name, fn in (("memcpy_pages", st.strata_baseline_memcpy_pages),):
                for d, dd in (("h2d", st.STRATA_H2D), ("d2h", st.STRATA_D2H)):
                    x = reqs.xfer(0, g.L, host_lists=True)
                    cnt = [0]

                    def run():
                        cnt[0] = fn(pool.handle, x, dd, io)
                    reps = 3 if P == 1 else 5
                    ev, wall = timed(run, io, reps=reps, warm=1)
                    t = max(ev, wall)
                    print(json.dumps({**base, "method": name, "dir": d, "calls": cnt[0], "ms": round(ev * 1e3, 3),
                                      "wall_ms": round(wall * 1e3, 3), "gbs": round(nbytes / t / 1e9, 3),
                                      "gbs_event": round(nbytes / ev / 1e9, 3)}), flush=True)
            per_layer = nbytes // g.L
            scratch = torch.empty(per_layer, dtype=torch.uint8, device="cuda")
            for d, dd in (("h2d", st.STRATA_H2D), ("d2h", st.STRATA_D2H)):
                def run():
                    for _ in range(g.L):
                        st.strata_baseline_contiguous(pool.handle, dd, scratch.data_ptr(), 0, per_layer, io)
                ev, wall = timed(run, io)
                print(json.dumps({**base, "method": "contiguous_memcpy", "dir": d, "ms": round(ev * 1e3, 3),
                                  "gbs": round(nbytes / ev / 1e9, 3)}), flush=True)
            del scratch
        pool.close()
        del k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
