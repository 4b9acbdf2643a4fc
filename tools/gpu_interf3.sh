#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python tools/interference.py --graph 1 --engines 1,4 --ctas 1,2,8 --memcpy 1 > gpurun_out/interference_graph2.jsonl 2> gpurun_out/interf.err; echo "graph rc=$?"
timeout 1200 python tools/interference.py --graph 0 --engines 1,4 --ctas 1,2,8 --memcpy 1 > gpurun_out/interference_eager2.jsonl 2>> gpurun_out/interf.err; echo "eager rc=$?"
python - <<'PY'
import json
for f in ("interference_graph2", "interference_eager2"):
    for l in open(f"gpurun_out/{f}.jsonl"):
        d = json.loads(l)
        if d["kind"] == "corun":
            print(f, d["engine"], d["ctas"], d["proxy"], d["proxy_alone_ms"], d["proxy_corun_ms"], d["slowdown"], d["io_alone_gbs"])
PY
