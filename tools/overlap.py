#!/usr/bin/env python
"""Overlap evidence for the per-layer completion events (SURVEY.md §8d "Overlap evidence").

An I/O stream runs strata_load over all layers; a consumer stream, for each layer l, waits on the
layer's event (strata_wait_layer), runs a proxy compute kernel of fixed duration t_c, then a
checksum of layer l.  The measured wall time (first load start -> last checksum) is compared with
the pipeline recurrence (paper_2508_18572_b200.overlap) evaluated on the measured
per-layer load completion times and the measured consumer time per layer; and with the serial
(no overlap) time.  Checksums are compared with the oracle when --check is given.

    python tools/overlap.py [--tokens 8192] [--tc-ratios 0.25,0.5,1,2]
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
from paper_2508_18572_b200.overlap import pipeline_recurrence  # noqa: E402


def _ev():
    return torch.cuda.Event(enable_timing=True)


def measure(tokens=8192, ratios=(0.25, 0.5, 1.0, 2.0), engine=0, num_ctas=0, reps=5, check=False, P=1):
    g = kvgen.geometry("llama8b_32k", P=P)
    q = kvgen.make_requests(kvgen.rng_for(11), [tokens], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    kvgen.fill_random(pool.host, 5)
    reqs = st.Requests.from_kvgen(q)
    io, cons = torch.cuda.Stream(), torch.cuda.Stream()

    # per-layer load time alone
    t = pool.load(reqs, stream=io, engine=engine, num_ctas=num_ctas)
    torch.cuda.synchronize()
    fin = [pool.layer_elapsed_ms(t, l) for l in range(g.L)]
    t_load = fin[-1] / g.L

    # calibrate the proxy compute: torch.cuda._sleep(cycles) is a fixed-duration spin kernel
    def consumer_work(l, cycles):
        torch.cuda._sleep(cycles)
        return k[l].view(torch.int64).sum() + v[l].view(torch.int64).sum()

    def time_consumer(cycles):
        with torch.cuda.stream(cons):
            consumer_work(0, cycles)
            a, b = _ev(), _ev()
            a.record(cons)
            for l in range(g.L):
                consumer_work(l, cycles)
            b.record(cons)
        b.synchronize()
        return a.elapsed_time(b) / g.L

    c1 = time_consumer(100000)
    c2 = time_consumer(200000)
    per_cycle = (c2 - c1) / 100000.0
    base = c1 - 100000 * per_cycle
    out = []
    for ratio in ratios:
        cycles = max(1000, int((ratio * t_load - base) / per_cycle))
        t_c = time_consumer(cycles)
        walls, preds, serials, preds_run, tcs_run, loads = [], [], [], [], [], []
        sums = None
        for _ in range(reps):
            torch.cuda.synchronize()
            start, end = _ev(), _ev()
            start.record(io)
            cons.wait_stream(io)
            ticket = pool.load(reqs, stream=io, engine=engine, num_ctas=num_ctas)
            res = []
            cev = []
            with torch.cuda.stream(cons):
                for l in range(g.L):
                    pool.wait_layer(ticket, l, cons)
                    a, b = _ev(), _ev()
                    a.record(cons)
                    res.append(consumer_work(l, cycles))
                    b.record(cons)
                    cev.append((a, b))
                end.record(cons)
            end.synchronize()
            wall = start.elapsed_time(end)
            lf = [pool.layer_elapsed_ms(ticket, l) for l in range(g.L)]
            tc_run = [a.elapsed_time(b) for a, b in cev]   # consumer time per layer while co-running
            _, pred, _ = pipeline_recurrence([0.0] * g.L, [t_c] * g.L, load_finish=lf)
            _, pred_run, _ = pipeline_recurrence([0.0] * g.L, tc_run, load_finish=lf)
            walls.append(wall)
            preds.append(pred)
            preds_run.append(pred_run)
            tcs_run.append(statistics.mean(tc_run))
            loads.append(lf[-1] / g.L)
            serials.append(lf[-1] + g.L * t_c)
            sums = [int(x) for x in res]
        rec = {"tokens": tokens, "P": P, "layers": g.L, "t_load_ms_per_layer": round(t_load, 4),
               "t_c_ms": round(t_c, 4), "ratio": ratio, "wall_ms": round(statistics.median(walls), 3),
               "recurrence_ms": round(statistics.median(preds), 3),
               "rel_err": round(abs(statistics.median(walls) - statistics.median(preds)) / statistics.median(preds), 4),
               "serial_ms": round(statistics.median(serials), 3),
               "t_c_ms_corun": round(statistics.median(tcs_run), 4),
               "t_load_ms_corun": round(statistics.median(loads), 4),
               "recurrence_corun_ms": round(statistics.median(preds_run), 3),
               "rel_err_corun": round(abs(statistics.median(walls) - statistics.median(preds_run))
                                      / statistics.median(preds_run), 4),
               "overlap_saving": round(1 - statistics.median(walls) / statistics.median(serials), 4)}
        if check:
            import numpy as np

            import oracle
            exp = []
            for l in range(g.L):
                ek = [None] * g.L
                evv = [None] * g.L
                ek[l] = np.zeros(nb, np.uint8)
                evv[l] = np.zeros(nb, np.uint8)
                oracle.load(g, pool.host, ek, evv, q, l, l + 1)
                s = (int(ek[l].view(np.int64).sum()) + int(evv[l].view(np.int64).sum()))
                exp.append(((s + 2**63) % 2**64) - 2**63)
            rec["checksums_match_oracle"] = exp == sums
        out.append(rec)
    pool.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--tc-ratios", default="0.25,0.5,1,2")
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--num-ctas", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    for rec in measure(args.tokens, [float(x) for x in args.tc_ratios.split(",")], args.engine, args.num_ctas,
                       check=args.check):
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
