#!/usr/bin/env python
"""Bubble filling (§4.3.3).

"when request G requires a long context load, the scheduler defers computation of the prepared
prefill batch and instead issues a decoding batch to the model executor to run concurrently with
the context loading ... decoding batches ... primarily saturate HBM bandwidth, whereas loading
tasks saturate PCIe bandwidth".

Workload (Llama-3.1-8B geometry): a prefill batch of `new` tokens over a 32K-token cached context
that must be loaded from the host tier, and a running decode batch (16 requests x 4K tokens).
  prefill  per layer: the layer's dense GEMMs for `new` tokens, gated by strata_wait_layer;
  decode   one step = a read of the decode batch's KV for all 32 layers (HBM bound, 8 GiB) + the
           layer GEMMs for 16 tokens.
The number of decode steps that fit in the stall comes from the native control plane
(strata_ctl_bubble_steps(t_load, t_prefill, t_step)), with times measured alone.  Two schedules of
the same work (the load, the prefill, N decode steps):
  prefill_first  load || layer-wise prefill, then the N decode steps (SGLang's prefill-first)
  bubble_fill    load || N decode steps, then the layer-wise prefill
Reported: makespan of each, speedup, the load's bandwidth under the co-run. One JSON line each.
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
from paper_2508_18572_b200 import ctl as ctl_mod  # noqa: E402

HIDDEN = 4096
GEMMS = [(HIDDEN, 6144), (HIDDEN, HIDDEN), (HIDDEN, 28672), (14336, HIDDEN)]


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--new", default="256,1024,4096")
    ap.add_argument("--engines", default="4,1")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--graph", type=int, default=0,
                    help="replay each decode step from a CUDA graph, as serving engines run decode")
    args = ap.parse_args()

    g = kvgen.geometry("llama8b_32k")
    q = kvgen.make_requests(kvgen.rng_for(3), [32768], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    reqs = st.Requests.from_kvgen(q)
    load_bytes = 2 * g.L * q.total_tokens * g.token_bytes
    io, comp = torch.cuda.Stream(), torch.cuda.Stream()
    weights = [torch.randn(a, b, dtype=torch.bfloat16, device="cuda") * 0.02 for a, b in GEMMS]
    dec_kv = [torch.randn(16 * 4096 * 8 * 128 * 2, dtype=torch.bfloat16, device="cuda") for _ in range(g.L)]
    dec_act = {d: torch.randn(16, d, dtype=torch.bfloat16, device="cuda") for d in (HIDDEN, 14336)}

    def decode_step():
        for l in range(g.L):
            dec_kv[l].sum(dtype=torch.float32)
            for w in weights:
                torch.matmul(dec_act[w.shape[0]], w)

    if args.graph:
        eager_step = decode_step
        dg = torch.cuda.CUDAGraph()
        with torch.cuda.stream(comp):
            eager_step()
            torch.cuda.synchronize()
            with torch.cuda.graph(dg, stream=comp):
                eager_step()
        decode_step = dg.replay  # noqa: F811

    def timed(fn, stream):
        a, b = ev(), ev()
        with torch.cuda.stream(stream):
            a.record(stream)
            fn()
            b.record(stream)
        b.synchronize()
        return a.elapsed_time(b)

    for new in [int(x) for x in args.new.split(",")]:
        acts = {d: torch.randn(new, d, dtype=torch.bfloat16, device="cuda") for d in (HIDDEN, 14336)}

        def layer(l):
            for w in weights:
                torch.matmul(acts[w.shape[0]], w)

        def prefill_resident():
            for l in range(g.L):
                layer(l)

        for fn in (prefill_resident, decode_step):       # warm-up (cuBLAS heuristics)
            timed(fn, comp)
        t_comp = statistics.median(timed(prefill_resident, comp) for _ in range(args.reps))
        t_step = statistics.median(timed(decode_step, comp) for _ in range(args.reps))
        for eng in [int(x) for x in args.engines.split(",")]:
            pool.load(reqs, stream=io, engine=eng)
            torch.cuda.synchronize()
            t_load = statistics.median(timed(lambda: pool.load(reqs, stream=io, engine=eng), io)
                                       for _ in range(args.reps))
            steps = ctl_mod.bubble_steps(t_load, t_comp, t_step, 16)
            res = {}
            for policy in ("prefill_first", "bubble_fill"):
                spans, loads = [], []
                for _ in range(args.reps):
                    torch.cuda.synchronize()
                    a, b, c = ev(), ev(), ev()
                    a.record(io)
                    comp.wait_stream(io)
                    ticket = pool.load(reqs, stream=io, engine=eng)
                    b.record(io)
                    with torch.cuda.stream(comp):
                        if policy == "bubble_fill":
                            for _ in range(steps):
                                decode_step()
                        for l in range(g.L):
                            pool.wait_layer(ticket, l, comp)
                            layer(l)
                        if policy == "prefill_first":
                            for _ in range(steps):
                                decode_step()
                        c.record(comp)
                    c.synchronize()
                    spans.append(a.elapsed_time(c))
                    loads.append(a.elapsed_time(b))
                res[policy] = (statistics.median(spans), statistics.median(loads))
            pf, bf = res["prefill_first"], res["bubble_fill"]
            print(json.dumps({
                "new": new, "cached": q.total_tokens, "decode_graph": args.graph, "load_compute_ratio": round(q.total_tokens / new, 1),
                "engine": {1: "ldg", 4: "dma"}.get(eng, eng), "load_alone_ms": round(t_load, 3),
                "prefill_alone_ms": round(t_comp, 3), "decode_step_alone_ms": round(t_step, 3),
                "bubble_steps": steps, "prefill_first_ms": round(pf[0], 3), "bubble_fill_ms": round(bf[0], 3),
                "speedup": round(pf[0] / bf[0], 3),
                "load_gbs_prefill_first": round(load_bytes / (pf[1] / 1e3) / 1e9, 2),
                "load_gbs_bubble_fill": round(load_bytes / (bf[1] / 1e3) / 1e9, 2)}), flush=True)
    pool.close()


if __name__ == "__main__":
    main()
