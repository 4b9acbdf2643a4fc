#!/usr/bin/env python
"""Layer-wise overlapped prefill over the loaded KV (§4.1,
:193 §3.2, fig:stall P:104-111).

A request has `cached` tokens of KV in the host tier and `new` tokens to prefill (Llama-3.1-8B
geometry: 32 layers, 32 query heads, 8 KV heads, d=128, bf16).  Per layer the executor runs the
layer's dense GEMMs for the new tokens and FlashInfer paged prefill attention of the new queries over
the cached pages of the NHD pool (BatchPrefillWithPagedKVCacheWrapper, page size P), after waiting on
that layer's load event (strata_wait_layer).  Measured per load/compute ratio (= cached / new, the
x-axis of fig:stall):

  compute_ms  prefill with the KV already resident (no I/O)
  serial_ms   load every layer first, then prefill
  overlap_ms  layer-wise overlap through the per-layer events
  stall %     (overlap_ms - compute_ms) / overlap_ms   — fig:stall's "I/O stall percentage"

for the library's engines and for the layer-wise per-page cudaMemcpyAsync loader the paper's
SGLang-HiCache baseline uses (events recorded per layer after its copies).
One JSON object per line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402

QO_HEADS = 32
HIDDEN = 4096
GEMMS = [(HIDDEN, 6144), (HIDDEN, HIDDEN), (HIDDEN, 28672), (14336, HIDDEN)]   # qkv, o, gate+up, down


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cached", type=int, default=32768)
    ap.add_argument("--new", default="256,512,1024,2048,4096,8192")
    ap.add_argument("--P", type=int, default=1)
    ap.add_argument("--engines", default="4,1")
    ap.add_argument("--baseline", type=int, default=1, help="also run the layer-wise per-page memcpy loader")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import flashinfer

    g = kvgen.geometry("llama8b_32k", P=args.P)
    q = kvgen.make_requests(kvgen.rng_for(2), [args.cached], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    # finite bf16 payload so attention runs on real numbers
    vals = (torch.randn(g.host_bytes // 2, dtype=torch.float32) * 0.5).to(torch.bfloat16)
    pool.host[:] = vals.view(torch.uint8).numpy()
    del vals
    reqs = st.Requests.from_kvgen(q)
    kc = [t.view(torch.bfloat16).view(g.num_pages, g.P, g.H, g.D) for t in k]
    vc = [t.view(torch.bfloat16).view(g.num_pages, g.P, g.H, g.D) for t in v]
    npages = int(q.dev_pages.size)
    last_len = args.cached - (npages - 1) * g.P
    io, comp = torch.cuda.Stream(), torch.cuda.Stream()
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    weights = [torch.randn(a, b, dtype=torch.bfloat16, device="cuda") * 0.02 for a, b in GEMMS]

    loaders = {}
    for e in [int(x) for x in args.engines.split(",")]:
        name = {1: "ldg", 2: "tma", 3: "tma_bulk", 4: "dma", 0: "default"}[e]
        loaders[f"strata_{name}"] = e
    if args.baseline and (g.P >= 16 or args.baseline > 1):   # 2M copies per load at P=1: seconds
        loaders["memcpy_pages_layerwise"] = -1
    layer_events = [ev() for _ in range(g.L)]

    def issue_load(kind):
        """Enqueue the whole load on `io`; returns a function giving layer l's completion event.

        The per-page baseline issues its copies from a loader thread (as a serving engine's cache
        controller would), so the executor can enqueue layer l as soon as layer l's copies are
        issued instead of after all 2*L*n/P of them."""
        if kind >= 0:
            t = pool.load(reqs, stream=io, engine=kind)
            return lambda l: ("strata", t, l)
        issued = [threading.Event() for _ in range(g.L)]

        def loader():
            for l in range(g.L):
                x = reqs.xfer(l, l + 1, host_lists=True)
                st.strata_baseline_memcpy_pages(pool.handle, x, st.STRATA_H2D, io)
                layer_events[l].record(io)
                issued[l].set()
        th = threading.Thread(target=loader)
        th.start()
        threads.append(th)
        return lambda l: ("event", layer_events[l], l, issued[l])

    def wait(handle):
        if handle[0] == "strata":
            pool.wait_layer(handle[1], handle[2], comp)
        else:
            handle[3].wait()
            comp.wait_event(handle[1])

    threads = []

    for new in [int(x) for x in args.new.split(",")]:
        wrapper = flashinfer.BatchPrefillWithPagedKVCacheWrapper(ws, "NHD")
        qo_indptr = torch.tensor([0, new], dtype=torch.int32, device="cuda")
        kv_indptr = torch.tensor([0, npages], dtype=torch.int32, device="cuda")
        kv_indices = reqs.dev_pages_d
        kv_last = torch.tensor([last_len], dtype=torch.int32, device="cuda")
        wrapper.plan(qo_indptr, kv_indptr, kv_indices, kv_last, QO_HEADS, g.H, g.D, g.P, causal=False,
                     q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        acts = {d: torch.randn(new, d, dtype=torch.bfloat16, device="cuda") for d in (HIDDEN, 14336)}
        qs = torch.randn(new, QO_HEADS, g.D, dtype=torch.bfloat16, device="cuda")

        def layer(l):
            for w in weights:
                torch.matmul(acts[w.shape[0]], w)
            return wrapper.run(qs, (kc[l], vc[l]))

        # warm-up (flashinfer JIT, cuBLAS heuristics) with the KV resident
        pool.load(reqs, stream=io)
        torch.cuda.synchronize()
        with torch.cuda.stream(comp):
            for l in range(g.L):
                layer(l)
        torch.cuda.synchronize()

        def compute_only():
            a, b = ev(), ev()
            with torch.cuda.stream(comp):
                a.record(comp)
                for l in range(g.L):
                    layer(l)
                b.record(comp)
            b.synchronize()
            return a.elapsed_time(b)

        t_comp = statistics.median(compute_only() for _ in range(args.reps))
        for name, kind in loaders.items():
            serial, overlap, loadonly = [], [], []
            for _ in range(args.reps):
                # serial: load everything, then prefill
                torch.cuda.synchronize()
                a, b, c = ev(), ev(), ev()
                a.record(io)
                issue_load(kind)
                for th in threads:      # serial: every copy is issued before the end marker
                    th.join()
                b.record(io)
                comp.wait_stream(io)
                with torch.cuda.stream(comp):
                    for l in range(g.L):
                        layer(l)
                    c.record(comp)
                c.synchronize()
                for th in threads:
                    th.join()
                threads.clear()
                serial.append(a.elapsed_time(c))
                loadonly.append(a.elapsed_time(b))
                # overlap: layer l's prefill waits only for layer l's load
                torch.cuda.synchronize()
                a, c = ev(), ev()
                a.record(io)
                comp.wait_stream(io)
                h = issue_load(kind)
                with torch.cuda.stream(comp):
                    for l in range(g.L):
                        wait(h(l))
                        layer(l)
                    c.record(comp)
                c.synchronize()
                for th in threads:
                    th.join()
                threads.clear()
                overlap.append(a.elapsed_time(c))
            o = statistics.median(overlap)
            print(json.dumps({"cached": args.cached, "new": new, "load_compute_ratio": round(args.cached / new, 2),
                              "P": g.P, "loader": name, "load_ms": round(statistics.median(loadonly), 3),
                              "compute_ms": round(t_comp, 3), "serial_ms": round(statistics.median(serial), 3),
                              "overlap_ms": round(o, 3), "stall_pct": round(100 * max(0.0, o - t_comp) / o, 2),
                              "speedup_vs_serial": round(statistics.median(serial) / o, 3)}), flush=True)
    pool.close()


if __name__ == "__main__":
    main()
