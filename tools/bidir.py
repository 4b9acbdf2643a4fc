#!/usr/bin/env python
"""Load and offload at the same time (SURVEY.md §8d "Bidirectional"; config 4, Llama-3.1-70B TP=8
rank slice: 80 layers, 1 KV head, d=128, 128K tokens per direction).

PCIe is full duplex: a serving engine loads cached prefixes for the next batch while it backs up
 the KV of finished prefills.  The load reads chunk set A into page set A on one
stream; the offload writes page set B into chunk set B on another.  Reported against the
concurrent contiguous H2D + D2H cudaMemcpyAsync ceiling from the same registered host tier.
One JSON object per line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama70b_tp8")
    ap.add_argument("--tokens", type=int, default=0, help="tokens per direction (0 = config)")
    ap.add_argument("--load-engine", type=int, default=0)
    ap.add_argument("--offload-engine", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--grid", default="",
                    help="load+offload operating points 'load_ctas:load_inflight_kib:off_ctas:off_inflight_kib,...' "
                         "(0 = library default), measured after the two one-direction runs")
    args = ap.parse_args()
    base = kvgen.geometry(args.config)
    n = args.tokens or kvgen.CONFIGS[args.config]["n"][0]
    # room for two disjoint sets of pages and chunks
    g = kvgen.Geometry(base.L, base.H, base.D, base.e, base.P, base.C, 2 * base.num_pages, 2 * base.num_chunks)
    rng = kvgen.rng_for(7)
    qa = kvgen.make_requests(rng, [n], g.P, g.C, g.num_pages // 2, g.num_chunks // 2)
    qb = kvgen.make_requests(rng, [n], g.P, g.C, g.num_pages // 2, g.num_chunks // 2)
    qb.dev_pages = (qb.dev_pages + g.num_pages // 2).astype(np.int32)
    qb.host_chunks = (qb.host_chunks + g.num_chunks // 2).astype(np.int32)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    kvgen.fill_random(pool.host, 1)
    ra, rb = st.Requests.from_kvgen(qa), st.Requests.from_kvgen(qb)
    nbytes = 2 * g.L * n * g.token_bytes
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

    def run(which, lc=0, li=0, oc=0, oi=0):
        torch.cuda.synchronize()
        a0, a1, b0, b1 = ev(), ev(), ev(), ev()
        if "load" in which:
            a0.record(sa)
            pool.load(ra, stream=sa, engine=args.load_engine, num_ctas=lc, inflight_kib=li)
            a1.record(sa)
        if "offload" in which:
            b0.record(sb)
            pool.offload(rb, stream=sb, engine=args.offload_engine, num_ctas=oc, inflight_kib=oi)
            b1.record(sb)
        torch.cuda.synchronize()
        out = {}
        if "load" in which:
            out["load_ms"] = a0.elapsed_time(a1)
        if "offload" in which:
            out["offload_ms"] = b0.elapsed_time(b1)
        return out

    solo_gbs = {}

    def med(rs, key):
        return statistics.median(r[key] for r in rs)

    points = [(w, (0, 0, 0, 0)) for w in (("load",), ("offload",), ("load", "offload"))]
    if args.grid:
        points = points[:2] + [(("load", "offload"), tuple(int(v) for v in spec.split(":"))) for spec in args.grid.split(",")]
    for which, knobs in points:
        run(which, *knobs)
        rs = [run(which, *knobs) for _ in range(args.reps)]
        rec = {"config": args.config, "tokens_per_direction": n, "bytes_per_direction": nbytes, "mode": "+".join(which),
               "load_ctas": knobs[0], "load_inflight_kib": knobs[1], "offload_ctas": knobs[2],
               "offload_inflight_kib": knobs[3]}
        for key in ("load_ms", "offload_ms"):
            if key in rs[0]:
                rec[key] = round(med(rs, key), 3)
                rec[key.replace("_ms", "_gbs")] = round(nbytes / (med(rs, key) / 1e3) / 1e9, 2)
        if len(which) == 2:
            # rates while BOTH run: the direction that finishes first ran alone for none of its time; the
            # other moved the rest of its bytes alone afterwards at its solo rate (measured above or 51)
            t_a, t_b = rec["load_ms"], rec["offload_ms"]
            first, t_first, t_second = ("offload", t_b, t_a) if t_b <= t_a else ("load", t_a, t_b)
            solo = solo_gbs.get("load" if first == "offload" else "offload", 51.0)
            moved_alone = solo * (t_second - t_first) / 1e3 * 1e9
            rec["overlap_gbs"] = {first: round(nbytes / (t_first / 1e3) / 1e9, 2),
                                  ("load" if first == "offload" else "offload"):
                                      round(max(0.0, nbytes - moved_alone) / (t_first / 1e3) / 1e9, 2)}
        else:
            solo_gbs[which[0]] = rec[which[0] + "_gbs"]
        print(json.dumps(rec), flush=True)

    # concurrent contiguous memcpy ceiling from the same host tier
    per_layer = nbytes // g.L
    dh, dd = torch.empty(per_layer, dtype=torch.uint8, device="cuda"), torch.empty(per_layer, dtype=torch.uint8,
                                                                                  device="cuda")
    res = []
    for _ in range(args.reps + 1):
        torch.cuda.synchronize()
        a0, a1, b0, b1 = ev(), ev(), ev(), ev()
        a0.record(sa)
        b0.record(sb)
        for _l in range(g.L):
            st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, dh.data_ptr(), 0, per_layer, sa)
            st.strata_baseline_contiguous(pool.handle, st.STRATA_D2H, dd.data_ptr(), nbytes, per_layer, sb)
        a1.record(sa)
        b1.record(sb)
        torch.cuda.synchronize()
        res.append((a0.elapsed_time(a1), b0.elapsed_time(b1)))
    h2d = statistics.median(r[0] for r in res[1:])
    d2h = statistics.median(r[1] for r in res[1:])
    print(json.dumps({"config": args.config, "mode": "contiguous_memcpy_bidir", "bytes_per_direction": nbytes,
                      "load_gbs": round(nbytes / (h2d / 1e3) / 1e9, 2),
                      "offload_gbs": round(nbytes / (d2h / 1e3) / 1e9, 2)}), flush=True)
    pool.close()


if __name__ == "__main__":
    main()
