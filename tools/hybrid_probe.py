#!/usr/bin/env python
"""Would a hybrid engine (most bytes through the SM zero-copy LDG path, the rest through the copy
engines at the same time) keep the link full at low interference?  Probe before building it:
co-run an LDG load (2 CTAs) of a fraction (1-f) of the Llama-8B 32K workload's layers' bytes with a
copy-engine stream moving the other f (contiguous H2D memcpy of the same size), against the
graph-replayed decode proxy of tools/interference.py.  Reports combined GB/s and decode slowdown."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def main():
    g = kvgen.geometry("llama8b_32k")
    hi = "--high-priority-io" in sys.argv        # I/O streams at the highest priority
    lo_p, hi_p = torch.cuda.Stream.priority_range()
    comp = torch.cuda.Stream()
    sa, sb = (torch.cuda.Stream(priority=hi_p), torch.cuda.Stream(priority=hi_p)) if hi else \
        (torch.cuda.Stream(), torch.cuda.Stream())
    kv = [torch.randn(16 * 4096 * 8 * 128 * 2, dtype=torch.bfloat16, device="cuda") for _ in range(32)]

    def decode():
        for t in kv:
            t.sum(dtype=torch.float32)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(comp):
        decode()
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=comp):
            decode()

    def t_decode(reps=10):
        evs = []
        with torch.cuda.stream(comp):
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(comp)
                gr.replay()
                b.record(comp)
                evs.append((a, b))
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in evs)

    alone = t_decode()
    for f in ((0.0, 1.0) if hi else (0.0, 0.1, 0.2, 0.3, 1.0)):
        n_ldg = int(round(32768 * (1 - f) / 64)) * 64
        n_ce = 32768 - n_ldg
        q = kvgen.make_requests(kvgen.rng_for(1), [max(n_ldg, 64)], g.P, g.C, g.num_pages, g.num_chunks)
        nb = g.num_pages * g.P * g.token_bytes
        k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P,
                           chunk_tokens=g.C, k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
        reqs = st.Requests.from_kvgen(q)
        ce_bytes = 2 * n_ce * g.token_bytes            # per layer
        scratch = torch.empty(max(ce_bytes, 16), dtype=torch.uint8, device="cuda")

        def one():
            if n_ldg:
                pool.load(reqs, stream=sa, engine=st.STRATA_ENGINE_LDG)
            if n_ce:
                for _ in range(g.L):
                    st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, scratch.data_ptr(), 0, ce_bytes, sb)
        one()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(sa)
        sb.wait_event(a)
        reps = 4
        for _ in range(reps):
            one()
        ea = torch.cuda.Event()
        ea.record(sb)
        sa.wait_event(ea)
        b.record(sa)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        gbs = 2 * g.L * 32768 * g.token_bytes / (ms / 1e3) / 1e9
        # co-run: keep the I/O busy for the decode measurement
        for _ in range(8):
            one()
        co = t_decode()
        torch.cuda.synchronize()
        print(json.dumps({"ce_fraction": round(n_ce / 32768, 3), "io_high_priority": hi, "load_gbs": round(gbs, 2),
                          "decode_alone_ms": round(alone, 4), "decode_corun_ms": round(co, 4),
                          "decode_slowdown": round(co / alone - 1, 4)}), flush=True)
        pool.close()


if __name__ == "__main__":
    main()
