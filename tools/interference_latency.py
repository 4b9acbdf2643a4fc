#!/usr/bin/env python
"""Device-memory latency beside a running strata_load (interference mechanism).

A single-thread pointer chase over a 512 MiB random cycle of 128-byte slots (> the 126 MB L2, every
step one dependent HBM access) measures loaded HBM latency: alone, beside the default load (ring,
2 CTAs), beside a 1-CTA load, and beside a contiguous copy-engine memcpy; plus the same for an
empty-kernel chain (launch latency).  One JSON object per line.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o tools/probe/libchase.so tools/probe/chase.cu
    python tools/interference_latency.py
"""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    lib = ctypes.CDLL(os.path.join(HERE, "probe", "libchase.so"))
    lib.chase_launch.argtypes = [ctypes.c_void_p, ctypes.c_uint, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_int]
    slots = (512 << 20) // 128
    perm = np.random.default_rng(5).permutation(slots).astype(np.uint32)
    nxt = np.empty(slots, np.uint32)
    nxt[perm] = np.roll(perm, -1)                      # one cycle through every slot
    table = np.zeros((slots, 32), np.uint32)
    table[:, 0] = nxt
    d_next = torch.from_numpy(table.reshape(-1)).cuda()
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    clk = torch.cuda.get_device_properties(0)
    g = kvgen.geometry("llama8b_32k")
    q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    reqs = st.Requests.from_kvgen(q)
    lo, hi = torch.cuda.Stream.priority_range()
    io, probe = torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=lo)
    scratch = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    steps = 20000

    cursor = [1]

    def chase_ns(smem, fresh=False):
        """fresh=False: the same 20000-line path every call (L2-resident after the first: L2-hit
        latency); fresh=True: the next 20000 lines of the 4M-line cycle (HBM-miss latency)."""
        start = int(perm[0])
        if fresh:
            start = int(perm[(cursor[0] * steps) % slots])
            cursor[0] += 1
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(probe)
        lib.chase_launch(d_next.data_ptr(), start, steps, out.data_ptr(), probe.cuda_stream, smem)
        b.record(probe)
        probe.synchronize()
        return a.elapsed_time(b) * 1e6 / steps          # wall ns per dependent access (incl. one launch)

    # a chain of 500 one-element kernels captured in a CUDA graph: device-side launch cadence
    x = torch.zeros(1, device="cuda")
    chain = torch.cuda.CUDAGraph()
    with torch.cuda.stream(probe):
        x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(chain, stream=probe):
            for _ in range(500):
                x.add_(1)

    def empty_chain_us(n=500):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(probe):
            a.record(probe)
            chain.replay()
            b.record(probe)
        b.synchronize()
        return a.elapsed_time(b) * 1e3 / n

    def beside(kind):
        if kind == "alone":
            fn = None
        elif kind == "memcpy":
            fn = lambda: [st.strata_baseline_contiguous(pool.handle, st.STRATA_H2D, scratch.data_ptr(), 0,  # noqa: E731
                                                        scratch.numel(), io) for _ in range(16)]
        else:
            c = {"ring_default": 0, "ring_1cta": 1, "ldg_2cta": 2}[kind]
            eng = st.STRATA_ENGINE_LDG if kind.startswith("ldg") else 0
            fn = lambda: pool.load(reqs, stream=io, num_ctas=c, engine=eng)  # noqa: E731
        res = {"beside": kind, "chase_ns": [], "chase_ns_own_sm": [], "hbm_chase_ns_own_sm": [], "empty_kernel_us": []}
        for _ in range(5):
            if fn:
                for _ in range(3):
                    fn()
            res["chase_ns"].append(chase_ns(0))
            res["chase_ns_own_sm"].append(chase_ns(200 << 10))
            res["hbm_chase_ns_own_sm"].append(chase_ns(200 << 10, fresh=True))
            res["empty_kernel_us"].append(empty_chain_us())
            torch.cuda.synchronize()
        for key in ("chase_ns", "chase_ns_own_sm", "hbm_chase_ns_own_sm", "empty_kernel_us"):
            res[key + "_median"] = round(statistics.median(res[key]), 2)
            res[key] = [round(v, 2) for v in res[key]]
        return res

    chase_ns(0)
    chase_ns(200 << 10)
    for kind in ("alone", "ring_default", "ring_1cta", "memcpy", "ldg_2cta", "alone"):
        print(json.dumps(beside(kind)), flush=True)
    pool.close()


if __name__ == "__main__":
    main()
