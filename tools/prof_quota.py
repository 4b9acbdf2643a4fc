#!/usr/bin/env python
"""One Llama-8B 32K P=1 load through ldg_quota_kernel (the decode-aware-quota variant of the fused
LDG load: dynamic row-group assignment), cap lifted, for an ncu --set full capture:

    ncu --set full -k regex:ldg_quota_kernel -c 1 -o out python tools/prof_quota.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2508_18572_b200 as st  # noqa: E402

g = kvgen.geometry("llama8b_32k")
q = kvgen.make_requests(kvgen.rng_for(1), [32768], g.P, g.C, g.num_pages, g.num_chunks)
nb = g.num_pages * g.P * g.token_bytes
k = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
v = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(g.L)]
with st.HostPool(num_layers=g.L, num_heads=g.H, head_dim=g.D, elem_bytes=g.e, page_size=g.P, chunk_tokens=g.C,
                 k_ptrs=k, v_ptrs=v, num_pages=g.num_pages, num_chunks=g.num_chunks) as pool:
    kvgen.fill_random(pool.host, 1)
    reqs = st.Requests.from_kvgen(q)
    io = torch.cuda.Stream()
    pool.set_load_quota(0, stream=io)
    for _ in range(2):
        pool.load(reqs, stream=io)
    torch.cuda.synchronize()
    print("engine", pool.counters()["last_engine"])
