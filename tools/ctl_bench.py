"""NEXT-4 measurement: the control plane on the paper's workload shape.

CPU leg (`--cpu`): scheduling cost of the native control plane vs the Python oracle — one round =
deferral + Algorithm 1 + dispatch + plans — on a LooGLE-shaped queue (documents of
21,613 tokens on average, several questions each).

GPU leg (default): a serving-loop replay at Llama-3.1-8B geometry.  All documents start in the
host tier (offloaded earlier); the device pool holds only a few.  Each round the native scheduler
forms a batch, and its WRITE-BACK and LOAD plans run through strata_offload / strata_load on one
stream; the batch then "completes" (no model: the measurement is the I/O the plans cause).
Reported per policy (Strata = deferral + balanced batching + bundle hits; FIFO = all three off):
tokens and bytes loaded / written back, rounds, plan-driven load GB/s (CUDA events on the I/O
stream) against the live contiguous-memcpy link.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from kvgen import traces  # noqa: E402


def cpu_leg(args):
    from oracle import ctl_oracle as co
    from paper_2508_18572_b200 import ctl as ctl_mod
    rng = np.random.default_rng(0)
    reqs, docs = traces.shared_context_trace(rng, args.docs, args.questions, args.doc_len, (20, 200),
                                             order="max", return_docs=True)
    out = []
    for name, mk in (("native", lambda: ctl_mod.Ctl(1, 64, 1 << 22, 1 << 16, max_batch_reqs=8)),
                     ("oracle", lambda: co.Ctl(1, 64, 1 << 22, 1 << 16, max_batch_reqs=8))):
        c = mk()
        for d in docs:
            c.insert(d, 1, 0.0)                # every document was offloaded to the host tier before
        t0 = time.perf_counter()
        for i, r in enumerate(reqs):
            c.submit(i, r)
        t_submit = time.perf_counter() - t0
        rounds, t_sched, t_done = 0, 0.0, 0.0
        t = 1.0
        while True:
            t0 = time.perf_counter()
            o = c.schedule(t)
            t_sched += time.perf_counter() - t0
            if not o["batch"]:
                break
            t0 = time.perf_counter()
            for r in o["batch"]:
                c.complete(r, t + 0.5)
            t_done += time.perf_counter() - t0
            rounds += 1
            t += 1.0
        rec = {"leg": "cpu", "impl": name, "requests": len(reqs), "doc_len": args.doc_len,
               "rounds": rounds, "submit_ms": round(t_submit * 1e3, 3),
               "schedule_ms_per_round": round(t_sched / max(rounds, 1) * 1e3, 3),
               "complete_ms_per_req": round(t_done / len(reqs) * 1e3, 4)}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    return out


def gpu_leg(args):
    import torch

    import paper_2508_18572_b200 as st
    from paper_2508_18572_b200 import ctl as ctl_mod
    Lyr, H, D, E, P, C = 32, 8, 128, 2, args.page_size, 64
    tok_bytes = Lyr * 2 * H * D * E
    rng = np.random.default_rng(1)
    reqs, docs = traces.shared_context_trace(rng, args.docs, args.questions, args.doc_len, (20, 200),
                                             order=args.order, return_docs=True)
    need_host = sum(-(-len(d) // C) for d in docs) + 4 * len(reqs)
    num_chunks = need_host + 64
    num_pages = -(-args.device_tokens // P)
    row = H * D * E
    k = [torch.empty(num_pages * P * row, dtype=torch.uint8, device="cuda") for _ in range(Lyr)]
    v = [torch.empty(num_pages * P * row, dtype=torch.uint8, device="cuda") for _ in range(Lyr)]
    pool = st.HostPool(num_layers=Lyr, num_heads=H, head_dim=D, elem_bytes=E, page_size=P, chunk_tokens=C,
                       k_ptrs=k, v_ptrs=v, num_pages=num_pages, num_chunks=num_chunks)
    stream = torch.cuda.Stream()
    s_ptr = stream.cuda_stream
    # live link roofline from the same registered tier
    nbytes = 1 << 30
    src = torch.from_numpy(pool.host[:nbytes])
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(stream):
        for _ in range(2):
            dst.copy_(src, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(4):
            dst.copy_(src, non_blocking=True)
        e1.record(stream)
    stream.synchronize()
    link = 4 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
    del dst
    results = []
    for policy in args.policies:
        on = policy == "strata"
        c = ctl_mod.Ctl(P, C, num_pages, num_chunks, max_batch_reqs=args.max_batch_reqs,
                        defer=on, balance=on, bundle=on)
        for d in docs:
            c.insert(d, ctl_mod.HOST, 0.0)
        for i, r in enumerate(reqs):
            c.submit(i, r)
        # The scheduler runs ahead of the GPU, as an asynchronous serving scheduler does: each
        # round's plans are enqueued on the I/O stream and the next round is formed while they run
        # (stream order keeps write-backs before the loads that reuse their pages).
        t, rounds = 1.0, 0
        load_tok = wb_tok = 0
        sched_ms = 0.0
        marks, keep = [], []
        start = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        while True:
            t0 = time.perf_counter()
            o = c.schedule(t)
            sched_ms += (time.perf_counter() - t0) * 1e3
            if not o["batch"]:
                break
            wb, ld = c.xfer("writeback"), c.xfer("load")
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(stream)
            if wb is not None:
                pool.offload(wb, stream=s_ptr, engine=args.engine)
            ev[1].record(stream)
            if ld is not None:
                pool.load(ld, stream=s_ptr, engine=args.engine)
            ev[2].record(stream)
            marks.append(ev)
            keep += [wb, ld]
            load_tok += o["load_tokens"]
            wb_tok += o["writeback_tokens"]
            for r in o["batch"]:
                c.complete(r, t + 0.5)
            rounds += 1
            t += 1.0
        end = torch.cuda.Event(enable_timing=True)
        end.record(stream)
        stream.synchronize()
        wb_ms = sum(ev[0].elapsed_time(ev[1]) for ev in marks)
        load_ms = sum(ev[1].elapsed_time(ev[2]) for ev in marks)
        total_ms = start.elapsed_time(end)
        del keep
        rec = {"leg": "gpu", "policy": policy, "order": args.order, "engine": args.engine,
               "docs": args.docs, "questions": args.questions, "doc_len": args.doc_len,
               "device_tokens": args.device_tokens, "page_size": P, "rounds": rounds,
               "load_tokens": load_tok, "load_gib": round(load_tok * tok_bytes / 2**30, 3),
               "writeback_tokens": wb_tok, "load_ms": round(load_ms, 3), "writeback_ms": round(wb_ms, 3),
               "load_gbs": round(load_tok * tok_bytes / (load_ms / 1e3) / 1e9, 2) if load_ms else None,
               "writeback_gbs": round(wb_tok * tok_bytes / (wb_ms / 1e3) / 1e9, 2) if wb_tok else None,
               "link_gbs": round(link, 2), "schedule_ms_total": round(sched_ms, 2),
               "gpu_ms_total": round(total_ms, 3),
               "io_gbs_total": round((load_tok + wb_tok) * tok_bytes / (total_ms / 1e3) / 1e9, 2)}
        if rec["load_gbs"]:
            rec["load_frac_of_link"] = round(rec["load_gbs"] / link, 4)
        print(json.dumps(rec), flush=True)
        results.append(rec)
        c.close()
    pool.close()
    return results


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--docs", type=int, default=8)
    ap.add_argument("--questions", type=int, default=4)
    ap.add_argument("--doc-len", type=int, default=21613)      # LooGLE average
    ap.add_argument("--order", default="max")
    ap.add_argument("--page-size", type=int, default=1)
    ap.add_argument("--device-tokens", type=int, default=3 * 21613 + 4096)
    ap.add_argument("--max-batch-reqs", type=int, default=4)
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--policies", nargs="+", default=["strata", "fifo"])
    args = ap.parse_args()
    if args.cpu:
        cpu_leg(args)
    else:
        gpu_leg(args)


if __name__ == "__main__":
    main()
