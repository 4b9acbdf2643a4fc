#!/usr/bin/env python
"""Host-side cost of one strata_load call (does the calling thread block?): wall time of the call
itself with the GPU idle, then the device time of the load, per engine and copy-stream count."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402


def main():
    g = kvgen.geometry("llama8b_32k")
    chunk_frag = sys.argv[1] if len(sys.argv) > 1 else "perm"
    q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks, chunk_frag=chunk_frag)
    nb = g.num_pages * g.P * g.token_bytes
    k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
    pool = st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                       k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
    reqs = st.Requests.from_kvgen(q)
    io = torch.cuda.Stream()
    for eng in (4, 1):
        pool.load(reqs, stream=io, engine=eng)
        torch.cuda.synchronize()
        for rep in range(3):
            a = torch.cuda.Event(enable_timing=True)
            a.record(io)
            t0 = time.perf_counter()
            t = pool.load(reqs, stream=io, engine=eng)
            t1 = time.perf_counter()
            ms = pool.layer_elapsed_ms(t, g.L - 1)
            print(json.dumps({"engine": eng, "chunk_order": chunk_frag,
                              "strided": os.environ.get("STRATA_DMA_STRIDED", "default"),
                              "copy_streams": os.environ.get("STRATA_COPY_STREAMS", "default"),
                              "call_ms": round((t1 - t0) * 1e3, 3), "device_ms": round(ms, 3)}), flush=True)
            torch.cuda.synchronize()
    pool.close()


if __name__ == "__main__":
    main()
