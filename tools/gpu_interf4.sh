#!/bin/bash
timeout 1200 python tools/interference.py --graph 1 --engines 1,4 --ctas 2 --memcpy 1 > gpurun_out/interference_clk.jsonl 2> gpurun_out/interf.err; echo "rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/interference_clk.jsonl"):
    d = json.loads(l)
    if d["kind"] == "corun":
        print(d["engine"], d["ctas"], d["proxy"], d["slowdown"], d["slowdown_rounds"], [(k, c["sm_mhz"] if c else None, c["power_w"] if c else None) for k, c in d["clocks"]])
PY
