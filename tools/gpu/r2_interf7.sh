#!/bin/bash
# Round 2: decode slowdown vs the number of kernels the same 8 GiB HBM read is split into
# (4 / 32 / 128 / 512 kernels), under the ring default, the 1-CTA point and a contiguous memcpy;
# graph-replayed and eager.
O=gpurun_out/r2_interf7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/interference.py --proxies decode4,decode32,decode128,decode512 --ring-configs 2:16:128:7:0:0,1:16:112:7:0:0 --memcpy 1 --reps 10 --tag split_eager > $O/interf.jsonl 2> $O/interf.err
timeout 1500 python tools/interference.py --proxies decode4,decode32,decode128,decode512 --ring-configs 2:16:128:7:0:0 --reps 10 --graph 1 --tag split_graph >> $O/interf.jsonl 2>> $O/interf.err
python - <<'PY'
import json
for l in open("gpurun_out/r2_interf7/interf.jsonl"):
    d=json.loads(l)
    if d["kind"]!="corun": print(l.strip()); continue
    print(d["tag"], d["engine"], d["ctas"], d["proxy"], d["proxy_alone_ms"], d["proxy_corun_ms"], d["slowdown"], d["io_alone_gbs"])
PY
tail -3 $O/interf.err
