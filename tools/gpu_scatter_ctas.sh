#!/bin/bash
# DMA scatter quota: throughput vs interference (cool-down method), to pick the default.
mkdir -p gpurun_out/sc
for c in 1 2 4 8 16; do python bench.py --no-cpu-baseline --num-ctas $c --steps 10 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.read());print('ctas=$c',d['value'],[round(x,2) for x in d['per_layer_ms_last_step'][:3]])"; done
timeout 1500 python tools/interference.py --graph 1 --engines 4 --ctas 2,4,8 > gpurun_out/sc/interf.jsonl 2> gpurun_out/sc/err; echo "rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/sc/interf.jsonl"):
    d = json.loads(l)
    if d["kind"] == "corun":
        print(d["engine"], d["ctas"], d["proxy"], d["slowdown"], d["slowdown_rounds"], d["io_alone_gbs"])
PY
