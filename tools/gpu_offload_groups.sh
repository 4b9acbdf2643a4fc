#!/bin/bash
mkdir -p gpurun_out/og
for cfg in deepseek_v3_mla llama70b_tp8_shared llama70b_tp8 llama8b_32k; do
  timeout 900 python tools/sweep.py --config $cfg --pages 1 --ctas 0 --engines 4 --groups 1,2,4,8 --baselines 0 > gpurun_out/og/$cfg.jsonl 2>/dev/null
  python - <<PY
import json
for l in open("gpurun_out/og/$cfg.jsonl"):
    d = json.loads(l)
    if d["dir"] == "d2h": print("$cfg", "G", d["layer_group"], d["gbs"])
PY
done
