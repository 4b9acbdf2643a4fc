#!/usr/bin/env python
"""Host-side cost of strata_load calls (does the calling thread block?).

For each engine: (a) the wall time of ONE call with the GPU idle, (b) the wall time of each of N
back-to-back calls on one stream (a serving engine's scheduler thread issuing loads ahead of the
GPU), next to the device time of the load.  One JSON object per line.

    python tools/submit_probe.py [--config llama8b_32k] [--engines 2,1,4] [--n 10]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b_32k")
    ap.add_argument("--engines", default="2,1,4")
    ap.add_argument("--n", type=int, default=10)
    ap.add_argument("--chunk-frag", default="perm")
    args = ap.parse_args()
    g = kvgen.geometry(args.config)
    q = kvgen.make_requests(kvgen.rng_for(1), kvgen.CONFIGS[args.config]["n"], g.P, g.C, g.num_pages,
                            g.num_chunks, chunk_frag=args.chunk_frag)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)] if g.kv == 2 else None
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    reqs = st.Requests.from_kvgen(q)
    io = torch.cuda.Stream()
    for eng in [int(e) for e in args.engines.split(",")]:
        pool.load(reqs, stream=io, engine=eng)
        torch.cuda.synchronize()
        single = []
        for _ in range(3):
            t0 = time.perf_counter()
            t = pool.load(reqs, stream=io, engine=eng)
            single.append((time.perf_counter() - t0) * 1e3)
            dev = pool.layer_elapsed_ms(t, g.L - 1)
            torch.cuda.synchronize()
        calls = []
        for _ in range(args.n):
            t0 = time.perf_counter()
            pool.load(reqs, stream=io, engine=eng)
            calls.append((time.perf_counter() - t0) * 1e3)
        t0 = time.perf_counter()
        torch.cuda.synchronize()
        drain = (time.perf_counter() - t0) * 1e3
        print(json.dumps({"config": args.config, "engine": eng, "engine_used": pool.counters()["last_engine"],
                          "fused_env": os.environ.get("STRATA_LDG_FUSED", "default"),
                          "single_call_ms": [round(x, 3) for x in single], "device_ms": round(dev, 3),
                          "back_to_back_call_ms": [round(x, 3) for x in calls], "drain_ms": round(drain, 3)}),
              flush=True)
    pool.close()


if __name__ == "__main__":
    main()
