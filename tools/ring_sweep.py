#!/usr/bin/env python
"""Ring engine (STRATA_ENGINE_TMA, csrc/ring.cu) geometry sweep on one GPU: SM quota x scatter warps x
piece size for loads, SM quota x piece size for offloads, on the bench workloads.  Every point is
checked bit-exact against the LDG engine's result of the same operation (sampled layers), so a
geometry that breaks parity shows up here, not only in the test suite.  One JSON line per point.

    python tools/ring_sweep.py [--configs llama8b_32k:1,llama8b_32k:16,llama70b_tp8:1] [--ctas 1,2,4]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def gbs(fn, io, nbytes, reps):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(io)
        fn()
        b.record(io)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return nbytes / statistics.median(ts) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="llama8b_32k:1,llama8b_32k:16,llama70b_tp8:1")
    ap.add_argument("--ctas", default="1,2,4")
    ap.add_argument("--warps", default="4,8,16", help="load scatter warps")
    ap.add_argument("--gather-warps", default="2,4,8", help="offload gather warps")
    ap.add_argument("--stage-kb", default="16,32,64")
    ap.add_argument("--dirs", default="load,offload")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--flags", type=int, default=0, help="strata_pool_desc.flags (host allocation variants)")
    ap.add_argument("--frag", default="perm", help="page table: perm | identity | churn")
    ap.add_argument("--chunk-frag", default="perm", help="host chunk order: perm | identity")
    ap.add_argument("--tag", default="")
    ap.add_argument("--layers", type=int, default=0, help="override L (0 = the config's)")
    ap.add_argument("--bulk-store", default="0", help="load: 0 st.global scatter, 1 cp.async.bulk stores (list)")
    ap.add_argument("--inflight-kb", default="0", help="host KiB in flight over all CTAs (list; 0 = library default)")
    args = ap.parse_args()
    io = torch.cuda.Stream()
    for spec in args.configs.split(","):
        name, P = spec.split(":")
        g = kvgen.geometry(name, P=int(P), **({"L": args.layers} if args.layers else {}))
        q = kvgen.make_requests(kvgen.rng_for(1), kvgen.CONFIGS[name]["n"], g.P, g.C, g.num_pages, g.num_chunks,
                                frag=args.frag, chunk_frag=args.chunk_frag)
        nb = g.num_pages * g.P * g.token_bytes
        k = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        v = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)] if g.kv == 2 else None
        pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P,
                           chunk_tokens=g.C, k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks,
                           host_heads=g.Ht, head_begin=g.h0, head_major=g.head_major, flags=args.flags)
        kvgen.fill_random(pool.host, 3)
        reqs = st.Requests.from_kvgen(q)
        nbytes = g.kv * g.L * q.total_tokens * g.token_bytes
        check_layers = sorted({0, g.L // 2, g.L - 1})
        # reference image: LDG engine load
        pool.load(reqs, stream=io, engine=st.STRATA_ENGINE_LDG)
        io.synchronize()
        ref = {l: (k[l].clone(), v[l].clone() if v else None) for l in check_layers}
        # offload check: the tier rewritten with its own bytes (skipped for tiers too large to copy on the host)
        host_ref = pool.host.copy() if g.host_bytes <= (16 << 30) else None
        # link ceilings through a scratch buffer (not the pool's buffers: the offload check needs them)
        scratch = torch.empty(min(nb, 256 << 20), dtype=torch.uint8, device="cuda")
        sb = scratch.numel()
        link = gbs(lambda: st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, scratch.data_ptr(), 0, sb, io),
                   io, sb, 5)
        link_d2h = gbs(lambda: st.strata_baseline_contiguous(pool.handle, st.STRATA_D2H, scratch.data_ptr(), 0, sb, io),
                       io, sb, 5)
        del scratch
        print(json.dumps({"kind": "link", "config": name, "P": g.P, "h2d_gbs": round(link, 2),
                          "d2h_gbs": round(link_d2h, 2)}), flush=True)
        for d in args.dirs.split(","):
            for c in [int(x) for x in args.ctas.split(",")]:
                for w in [int(x) for x in (args.warps if d == "load" else args.gather_warps).split(",")]:
                    for skb, bs, ifk in [(a_, b_, c_) for a_ in args.stage_kb.split(",")
                                         for b_ in (args.bulk_store.split(",") if d == "load" else ["0"])
                                         for c_ in args.inflight_kb.split(",")]:
                        skb = int(skb)
                        ifk = int(ifk)
                        os.environ["STRATA_RING_STAGE_KB"] = str(skb)
                        os.environ["STRATA_RING_BULK_STORE"] = bs
                        os.environ["STRATA_RING_WARPS" if d == "load" else "STRATA_RING_GATHER_WARPS"] = str(w)
                        if d == "load":
                            for l in check_layers:
                                k[l].zero_()
                                if v:
                                    v[l].zero_()
                            fn = lambda: pool.load(reqs, stream=io, engine=st.STRATA_ENGINE_TMA, num_ctas=c, inflight_kib=ifk)  # noqa: E731
                        else:
                            fn = lambda: pool.offload(reqs, stream=io, engine=st.STRATA_ENGINE_TMA, num_ctas=c, inflight_kib=ifk)  # noqa: E731
                        r = gbs(fn, io, nbytes, args.reps)
                        io.synchronize()
                        if d == "load":
                            ok = all(torch.equal(k[l], ref[l][0]) and (v is None or torch.equal(v[l], ref[l][1]))
                                     for l in check_layers)
                        else:
                            ok = None if host_ref is None else bool((pool.host == host_ref).all())   # loaded from this tier: offload rewrites the same bytes
                        print(json.dumps({"kind": "ring", "tag": args.tag, "L": g.L, "flags": args.flags, "frag": args.frag,
                                          "chunk_frag": args.chunk_frag, "config": name, "P": g.P, "dir": d, "ctas": c, "warps": w,
                                          "stage_kb": skb, "bulk_store": int(bs), "inflight_kb": ifk, "gbs": round(r, 2),
                                          "us": round(nbytes / r / 1e3, 2),
                                          "frac_link": round(r / (link if d == "load" else link_d2h), 4),
                                          "parity": ok}), flush=True)
        for key in ("STRATA_RING_STAGE_KB", "STRATA_RING_WARPS", "STRATA_RING_GATHER_WARPS", "STRATA_RING_BULK_STORE"):
            os.environ.pop(key, None)
        pool.close()
        del k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
