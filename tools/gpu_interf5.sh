#!/bin/bash
timeout 1500 python tools/interference.py --graph 1 --engines 1,4 --ctas 1,2 --memcpy 1 --cooldown 1.0 > gpurun_out/interference_cool.jsonl 2> gpurun_out/interf.err; echo "rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/interference_cool.jsonl"):
    d = json.loads(l)
    if d["kind"] == "corun":
        print(d["engine"], d["ctas"], d["proxy"], d["proxy_alone_ms"], d["proxy_corun_ms"], d["slowdown"], d["slowdown_rounds"])
PY
