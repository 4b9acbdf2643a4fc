#!/usr/bin/env python
"""Throughput of the narrow path (R29) on rows that are not 16-byte multiples: 32 layers x 32K tokens
of H x D x e rows, default engine (copy engines + narrow scatter) and the narrow LDG kernel."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402
from kvgen import Geometry  # noqa: E402


def main():
    io = torch.cuda.Stream()
    for H, D, e in ((1, 72, 1), (3, 20, 2), (1, 100, 1), (8, 128, 2)):
        g = Geometry(L=32, H=H, D=D, e=e, P=1, C=64, num_pages=40960, num_chunks=640)
        q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks)
        nb = g.num_pages * g.P * g.token_bytes
        k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
        pool = st.HostPool(num_layers=g.L, num_heads=H, head_dim=D, elem_bytes=e, page_size=1, chunk_tokens=64,
                           k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks)
        reqs = st.Requests.from_kvgen(q)
        nbytes = 2 * g.L * 32768 * g.token_bytes
        quotas = [int(x) for x in os.environ.get("NARROW_CTAS", "0").split(",")]
        for eng, c in [(0, 0)] + [(1, c) for c in quotas]:
            for d, fn in (("load", pool.load), ("offload", pool.offload)):
                fn(reqs, stream=io, engine=eng, num_ctas=c)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(io)
                for _ in range(3):
                    fn(reqs, stream=io, engine=eng, num_ctas=c)
                b.record(io)
                b.synchronize()
                print(json.dumps({"row_bytes": g.token_bytes, "engine": {0: "default", 1: "ldg"}[eng], "ctas": c,
                                  "dir": d,
                                  "used": pool.counters()["last_engine"],
                                  "gbs": round(3 * nbytes / (a.elapsed_time(b) / 1e3) / 1e9, 2)}), flush=True)
        pool.close()


if __name__ == "__main__":
    main()
