#!/bin/bash
# Round 2: interference mechanism: one-kernel decode (decode1) vs 32-launch decode; evict-first L2
# policy on the ring's host reads (STRATA_RING_DEBUG=2); contiguous copy-engine memcpy.
O=gpurun_out/r2_interf6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python tools/interference.py --proxies decode,decode1 --ring-configs 2:16:128:7:0:0,2:16:128:7:0:2,1:16:112:7:0:0 --memcpy 1 --reps 10 --tag mech6 > $O/interf.jsonl 2> $O/interf.err
timeout 600 python tools/interference.py --proxies decode,decode1 --engines 1 --ctas 2 --reps 10 --graph 1 --tag mech6_graph >> $O/interf.jsonl 2>> $O/interf.err
python - <<'PY'
import json
for l in open("gpurun_out/r2_interf6/interf.jsonl"):
    d=json.loads(l)
    if d["kind"]!="corun": print(l.strip()); continue
    print(d["tag"], d["engine"], d["ctas"], d["env"], d["proxy"], d["slowdown"], d["io_alone_gbs"], d["io_corun_gbs_upper"])
PY
tail -3 $O/interf.err
