#!/usr/bin/env python
"""Disk -> host prefetch latency, page-first vs layer-first (§5.3.4, fig:disk:
"loading 8192 tokens from disk" with page size 32; page-first up to 4x lower latency).

Llama-3.1-8B geometry (32 layers x 8 KV heads x 128 x bf16 = 4 KiB per token per layer) with host
chunks of C = 32 tokens, so one page-first chunk is 4 MiB (one read) and a layer-first chunk is 32
reads of 128 KiB (SPEC.md:177-178 sizes).  Writes a file of `--chunks` chunks with the library's
writeback, then times prefetches of the 8192-token (256-chunk) set with O_DIRECT for several I/O
thread counts.  One JSON object per line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import kvgen  # noqa: E402
from paper_2508_18572_b200 import _lib  # noqa: E402
from paper_2508_18572_b200 import disk as sd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default=".")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--C", type=int, default=32)
    ap.add_argument("--chunks", type=int, default=1024, help="disk tier capacity (chunks)")
    ap.add_argument("--threads", default="1,4,16")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    L, tok_layer = 32, 4096
    cb = L * args.C * tok_layer
    need = -(-args.tokens // args.C)
    host = sd.aligned_empty(need * cb)
    kvgen.fill_random(host, 4)
    rng = kvgen.rng_for(8)
    dsel = rng.permutation(args.chunks)[:need]
    for layout, name in ((sd.STRATA_DISK_PAGE_FIRST, "page_first"), (sd.STRATA_DISK_LAYER_FIRST, "layer_first")):
        path = os.path.join(args.dir, f"strata_disk_{name}.bin")
        o_direct = True
        try:
            tier = sd.DiskTier(path, cb, L, args.chunks, layout=layout, o_direct=True, io_threads=16)
        except _lib.StrataError:
            o_direct = False
            tier = sd.DiskTier(path, cb, L, args.chunks, layout=layout, o_direct=False, io_threads=16)
        assert tier.wait(tier.writeback(host, range(need), dsel))[0] == 0
        tier.close()
        for nt in [int(x) for x in args.threads.split(",")]:
            tier = sd.DiskTier(path, cb, L, args.chunks, layout=layout, o_direct=o_direct, create=False, io_threads=nt)
            back = sd.aligned_empty(need * cb)
            ts = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                rc, done, _ = tier.wait(tier.prefetch(back, dsel, range(need)))
                ts.append(time.perf_counter() - t0)
                assert rc == 0 and done == need
            assert np.array_equal(back, host)
            t = statistics.median(ts)
            reads = need * (1 if layout == sd.STRATA_DISK_PAGE_FIRST else L)
            print(json.dumps({"layout": name, "tokens": args.tokens, "C": args.C, "chunks": need,
                              "bytes": int(need * cb), "reads": reads, "read_bytes": cb // (1 if layout == 0 else L),
                              "io_threads": nt, "o_direct": o_direct, "ms": round(t * 1e3, 2),
                              "gbs": round(need * cb / t / 1e9, 3)}), flush=True)
            tier.close()
        os.remove(path)


if __name__ == "__main__":
    main()
