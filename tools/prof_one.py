#!/usr/bin/env python
"""A short, ncu-friendly driver: a few strata_load / strata_offload launches of one config with a
reduced layer count (every per-layer launch is identical, so L only scales the run length).

    ncu --set full -k regex:tma_kernel -s 2 -c 1 -o gpurun_out/prof python tools/prof_one.py --engine 2
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b_32k")
    ap.add_argument("--P", type=int, default=1)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--engine", type=int, default=2)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--dir", default="h2d")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    g = kvgen.geometry(args.config, P=args.P, L=args.layers)
    q = kvgen.make_requests(kvgen.rng_for(1), kvgen.CONFIGS[args.config]["n"], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v if g.kv == 2 else None, num_pages=g.num_pages, num_chunks=g.num_chunks,
                       host_heads=g.Ht, head_begin=g.h0, head_major=g.head_major)
    kvgen.fill_random(pool.host, 3)
    reqs = st.Requests.from_kvgen(q)
    fn = pool.load if args.dir == "h2d" else pool.offload
    for _ in range(args.reps):
        fn(reqs, engine=args.engine, num_ctas=args.ctas, threads=args.threads)
    torch.cuda.synchronize()
    pool.close()


if __name__ == "__main__":
    main()
