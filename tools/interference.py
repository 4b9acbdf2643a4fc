#!/usr/bin/env python
"""Interference-aware SM quota (§4.2, fig:interference).

The paper co-runs its I/O kernel with a prefill pass (2 requests x 4K) and a decode pass (16 requests
x 4K) on H200 and picks 2 CTAs x 1024 threads for loads (~50 GB/s, < 5 % prefill and < 10 % decode
slowdown) and 1 CTA for backups.  Here the same experiment runs on B200 with synthetic proxies:

  prefill proxy  bf16 GEMMs of a Llama-3.1-8B layer for 2 x 4K tokens (M=8192: QKV 4096x6144,
                 O 4096x4096, gate/up 4096x28672, down 14336x4096) — tensor-core bound;
  decode proxy   a read of 16 x 4K tokens of Llama-8B KV per layer for 32 layers (8 GiB, fp32-
                 accumulated sum) — HBM bound.

For each engine x SM quota (num_ctas) it measures the proxy alone, the I/O alone, and both at once
(I/O on a high-priority stream looping strata_load over the Llama-8B 32K workload), and reports the
proxy slowdown and the co-run I/O bandwidth.  One JSON object per line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def make_prefill():
    M = 8192
    shapes = [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096)]
    xs = {k: torch.randn(M, k, dtype=torch.bfloat16, device="cuda") for k, _ in shapes}
    ws = [torch.randn(k, n, dtype=torch.bfloat16, device="cuda") for k, n in shapes]

    def run():
        for (k, n), w in zip(shapes, ws):
            torch.matmul(xs[k], w)
    return run


def make_decode1():
    # the same 8 GiB HBM read as ONE reduction kernel (no per-layer launches): separates a memory-side
    # slowdown from one in the launch path
    kv = torch.randn(32 * 16 * 4096 * 8 * 128 * 2, dtype=torch.bfloat16, device="cuda")

    def run():
        kv.sum(dtype=torch.float32)
    return run


def make_decode_split(n):
    total = 32 * 16 * 4096 * 8 * 128 * 2
    kv = [torch.randn(total // n, dtype=torch.bfloat16, device="cuda") for _ in range(n)]

    def run():
        for t in kv:
            t.sum(dtype=torch.float32)
    return run


def make_decode():
    # 16 requests x 4096 tokens x 8 heads x 128 dim x bf16 x (K,V) = 256 MiB per layer, 32 layers
    kv = [torch.randn(16 * 4096 * 8 * 128 * 2, dtype=torch.bfloat16, device="cuda")
          for _ in range(32)]

    def run():
        for t in kv:
            t.sum(dtype=torch.float32)
    return run


def _attn_layers(batch=16, ctx=4096, page=16, layers=32):
    """The paper's decode pass (16 requests x 4K) with the real kernel: FlashInfer paged
    decode attention, Llama-3.1-8B heads (32 query / 8 KV heads, d = 128, bf16), page size 16, one
    KV cache per layer (256 MiB each at the defaults), the pages of every request scattered."""
    import flashinfer
    npg = batch * ctx // page
    gen = torch.Generator(device="cuda").manual_seed(7)
    caches = [(torch.randn(npg, page, 8, 128, dtype=torch.bfloat16, device="cuda", generator=gen),
               torch.randn(npg, page, 8, 128, dtype=torch.bfloat16, device="cuda", generator=gen))
              for _ in range(layers)]
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
    indices = torch.randperm(npg, device="cuda", generator=gen).to(torch.int32)
    indptr = torch.arange(0, npg + 1, ctx // page, dtype=torch.int32, device="cuda")
    last = torch.full((batch,), page, dtype=torch.int32, device="cuda")
    w.plan(indptr, indices, last, 32, 8, 128, page, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    q = torch.randn(batch, 32, 128, dtype=torch.bfloat16, device="cuda", generator=gen)
    out = torch.empty_like(q)
    return w, q, out, caches


def make_attn():
    w, q, out, caches = _attn_layers()

    def run():
        for c in caches:
            w.run(q, c, out=out)
    return run


def make_decode_step():
    """A whole Llama-3.1-8B decode step at batch 16 x 4K context, every layer's kernels in order:
    RMSNorm, QKV GEMM, FlashInfer paged decode attention, O GEMM, RMSNorm, gate/up GEMM, SiLU x up,
    down GEMM (random bf16 weights, 14 GiB; KV as in make_attn)."""
    w, q, out, caches = _attn_layers()
    B, Hd = 16, 4096
    gen = torch.Generator(device="cuda").manual_seed(8)
    mk = lambda *s: torch.randn(*s, dtype=torch.bfloat16, device="cuda", generator=gen) * 0.02  # noqa: E731
    layers = [(mk(Hd, 6144), mk(Hd, Hd), mk(Hd, 2 * 14336), mk(14336, Hd), mk(Hd), mk(Hd)) for _ in caches]
    x = torch.randn(B, Hd, dtype=torch.bfloat16, device="cuda", generator=gen)

    def run():
        h = x
        for (wqkv, wo, wgu, wd, n1, n2), c in zip(layers, caches):
            a = torch.nn.functional.rms_norm(h, (Hd,), n1)
            qkv = a @ wqkv
            w.run(qkv[:, :Hd].reshape(B, 32, 128), c, out=out)
            h = h + out.reshape(B, Hd) @ wo
            a = torch.nn.functional.rms_norm(h, (Hd,), n2)
            gu = a @ wgu
            h = h + (torch.nn.functional.silu(gu[:, :14336]) * gu[:, 14336:]) @ wd
        return h
    return run


CLOCKS = []   # (sm MHz, power W) samples of the last time_proxy block


def _sample_clocks(stop):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        while not stop[0]:
            CLOCKS.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                           pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.002)
    except Exception:
        pass


def time_proxy(fn, stream, reps):
    CLOCKS.clear()
    stop = [False]
    th = threading.Thread(target=_sample_clocks, args=(stop,), daemon=True)
    th.start()
    evs = []
    with torch.cuda.stream(stream):
        fn()
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            evs.append((a, b))
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def clock_summary():
    if not CLOCKS:
        return None
    return {"sm_mhz": statistics.median(c for c, _ in CLOCKS), "power_w": round(statistics.median(p for _, p in CLOCKS), 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctas", default="1,2,4,8,16")
    ap.add_argument("--engines", default="1,2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--groups", default="0", help="DMA layer_group values (engine 4 only)")
    ap.add_argument("--ring-smem", default="0",
                    help="ring engine (engine 2) shared-memory budgets per CTA in KiB (0 = all): bounds the host "
                         "bytes in flight (STRATA_RING_SMEM_KB)")
    ap.add_argument("--ring-stage", default="0", help="ring engine piece sizes in KiB (0 = default; STRATA_RING_STAGE_KB)")
    ap.add_argument("--ring-configs", default="",
                    help="explicit ring geometries 'ctas:stage_kb:smem_kb:warps,...' (replaces the engine x ctas grid)")
    ap.add_argument("--env-sets", default="",
                    help="ring loads (engine 2, default quota) under explicit library environments: "
                         "'K=V;K=V,K=V,...' (e.g. STRATA_RING_LOAD_PACE_MBS=48000;STRATA_RING_INFLIGHT_KB=320)")
    ap.add_argument("--memcpy", type=int, default=0, help="also co-run a contiguous cudaMemcpyAsync loop (-1 engine)")
    ap.add_argument("--cooldown", type=float, default=1.0,
                    help="idle seconds before every alone / co-run block (power-state reset for the GEMM proxy)")
    ap.add_argument("--graph", type=int, default=0,
                    help="replay each proxy from a CUDA graph (as serving engines run decode): copy-engine "
                         "traffic delays the per-kernel launch fetches of eager proxies (ce_interference.py)")
    ap.add_argument("--layers", type=int, default=0, help="override L of the Llama-8B load (device-pool footprint)")
    ap.add_argument("--P", type=int, default=1, help="device page size")
    ap.add_argument("--flags", type=int, default=0, help="strata_pool_desc.flags of the host tier (1 = huge pages)")
    ap.add_argument("--tag", default="")
    ap.add_argument("--proxies", default="prefill,decode", help="prefill, decode, decode1 (one-kernel decode), decodeN (N kernels), attn (FlashInfer decode attention), decode_step (a whole Llama-8B decode step)")
    ap.add_argument("--offload", type=int, default=0, help="1: co-run offloads (write-back) instead of loads")
    ap.add_argument("--quota-bracket", type=int, default=0,
                    help="N > 0: also run every proxy bracketed by strata_set_load_quota(N) / (0) on its own "
                         "stream (decode-aware quota: while the proxy runs, running LDG loads take new rows "
                         "on N CTAs only); reported as '<proxy>@qN'")
    args = ap.parse_args()

    g = kvgen.geometry("llama8b_32k", P=args.P, **({"L": args.layers} if args.layers else {}))
    q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks, flags=args.flags)
    reqs = st.Requests.from_kvgen(q)
    bytes_load = 2 * g.L * q.total_tokens * g.token_bytes
    lo, hi = torch.cuda.Stream.priority_range()
    io = torch.cuda.Stream(priority=hi)       # I/O: high priority (its few CTAs get SMs first)
    comp = torch.cuda.Stream(priority=lo)
    makers = {"prefill": make_prefill, "decode": make_decode, "decode1": make_decode1, "attn": make_attn,
              "decode_step": make_decode_step}
    # decodeN: the same 8 GiB HBM read split into N reduction kernels (per-kernel-boundary cost)
    proxies = {name: (makers[name]() if name in makers else make_decode_split(int(name[len("decode"):])))
               for name in args.proxies.split(",")}
    if args.quota_bracket:
        pool.set_load_quota(0, stream=comp)   # loads launched from here on take rows dynamically
        torch.cuda.synchronize()
        qn = args.quota_bracket

        def bracket(fn):
            def run():
                pool.set_load_quota(qn, stream=comp)
                fn()
                pool.set_load_quota(0, stream=comp)
            return run
        proxies.update({f"{name}@q{qn}": bracket(fn) for name, fn in list(proxies.items())})
    if args.graph:
        graphs = {}
        for name, fn in proxies.items():
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(comp):
                fn()
                torch.cuda.synchronize()
                with torch.cuda.graph(gr, stream=comp):
                    fn()
            graphs[name] = gr
        proxies = {name: gr.replay for name, gr in graphs.items()}
    alone = {name: time_proxy(fn, comp, args.reps) for name, fn in proxies.items()}
    print(json.dumps({"kind": "proxy_alone", **{k_: round(v_, 4) for k_, v_ in alone.items()}}), flush=True)

    scratch = torch.empty(bytes_load // g.L, dtype=torch.uint8, device="cuda")

    def make_io(eng, c, G, env):
        for key in ("STRATA_RING_SMEM_KB", "STRATA_RING_STAGE_KB", "STRATA_RING_WARPS", "STRATA_RING_DEBUG",
                    "STRATA_RING_EXCLUSIVE", "STRATA_RING_LOAD_PACE_MBS", "STRATA_RING_INFLIGHT_KB"):
            os.environ.pop(key, None)
        os.environ.update(env)
        if eng < 0:   # contiguous memcpy of the same bytes: 32 copies of one layer's worth
            def run():
                for _ in range(g.L):
                    st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, scratch.data_ptr(), 0, scratch.numel(), io)
            return run
        op = pool.offload if args.offload else pool.load
        return lambda: op(reqs, stream=io, engine=eng, num_ctas=c, layer_group=G)

    configs = []
    for eng in [int(x) for x in args.engines.split(",")]:
        for c in [int(x) for x in args.ctas.split(",")]:
            for G in ([int(x) for x in args.groups.split(",")] if eng == 4 else [0]):
                envs = [{}]
                if eng == 2:
                    envs = [{**({"STRATA_RING_SMEM_KB": str(m)} if int(m) else {}),
                             **({"STRATA_RING_STAGE_KB": str(k_)} if int(k_) else {})}
                            for m in args.ring_smem.split(",") for k_ in args.ring_stage.split(",")]
                for env in envs:
                    configs.append((eng, c, G, env))
    if args.ring_configs:
        configs = []
        for spec in args.ring_configs.split(","):
            f = spec.split(":")
            c, skb, smem, w = (int(x) for x in f[:4])
            env = {"STRATA_RING_STAGE_KB": str(skb), "STRATA_RING_SMEM_KB": str(smem), "STRATA_RING_WARPS": str(w)}
            if len(f) > 4:   # optional 5th field: STRATA_RING_EXCLUSIVE (reserve the SM's shared memory)
                env["STRATA_RING_EXCLUSIVE"] = f[4]
            if len(f) > 5:   # optional 6th field: STRATA_RING_DEBUG bits (A/B only)
                env["STRATA_RING_DEBUG"] = f[5]
            configs.append((2, c, 0, env))
    if args.env_sets:
        configs = [(2, 0, 0, dict(kv.split("=", 1) for kv in item.split(";") if kv))
                   for item in args.env_sets.split(",")]
    if args.memcpy:
        configs.append((-1, 0, 0, {}))
    for eng, c, G, env in configs:
        if True:
            load = make_io(eng, c, G, env)
            # I/O alone
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            load()
            a.record(io)
            for _ in range(3):
                load()
            b.record(io)
            b.synchronize()
            io_alone = 3 * bytes_load / (a.elapsed_time(b) / 1e3) / 1e9
            for name, fn in proxies.items():
                # Alone and co-run measurements alternate (3 rounds, medians): a baseline taken once at
                # the start read up to 13 % slow for the decode proxy (after the GEMM proxy), and two
                # back-to-back GEMM blocks drift with power state, so each co-run gets its own
                # neighbouring alone measurement.
                alone_ms, co_ms, io_cos, clk = [], [], [], []
                for _r in range(3):
                    torch.cuda.synchronize()
                    time.sleep(args.cooldown)
                    alone_ms.append(time_proxy(fn, comp, args.reps))
                    clk.append(("alone", clock_summary()))
                    # keep the I/O stream busy for the whole proxy measurement
                    n_loads = max(2, int(alone_ms[-1] * args.reps / (bytes_load / io_alone / 1e6)) + 2)
                    torch.cuda.synchronize()
                    time.sleep(args.cooldown)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(io)
                    for _ in range(n_loads):
                        load()
                    b.record(io)
                    co_ms.append(time_proxy(fn, comp, args.reps))
                    clk.append(("corun", clock_summary()))
                    b.synchronize()
                    io_cos.append(n_loads * bytes_load / (a.elapsed_time(b) / 1e3) / 1e9)
                al, co = statistics.median(alone_ms), statistics.median(co_ms)
                print(json.dumps({"kind": "corun", "tag": args.tag, "dir": "offload" if args.offload else "load", "L": g.L, "P": g.P, "flags": args.flags,
                                  "graph": args.graph, "engine": eng, "ctas": c, "layer_group": G, "env": env,
                                  "proxy": name, "proxy_alone_ms": round(al, 4), "proxy_corun_ms": round(co, 4),
                                  "slowdown": round(co / al - 1, 4),
                                  "slowdown_rounds": [round(x / y - 1, 4) for x, y in zip(co_ms, alone_ms)],
                                  "io_alone_gbs": round(io_alone, 2),
                                  "io_corun_gbs_upper": round(statistics.median(io_cos), 2),
                                  "clocks": clk}), flush=True)
    pool.close()


if __name__ == "__main__":
    main()
