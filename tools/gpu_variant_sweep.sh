#!/bin/bash
mkdir -p gpurun_out/vs
timeout 1200 python tools/sweep.py --config deepseek_v3_mla --pages 1,16,64 --ctas 0 --engines 4,1 --baselines 0 > gpurun_out/vs/mla.jsonl 2>/dev/null; echo "mla rc=$?"
timeout 1200 python tools/sweep.py --config llama70b_tp8_shared --pages 1,16,64 --ctas 0 --engines 4,1 --baselines 0 > gpurun_out/vs/shared.jsonl 2>/dev/null; echo "shared rc=$?"
python bench.py --no-cpu-baseline --config qwen14b_batch8 --page-size 16 --steps 4 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.read());print('qwen P16',d['value'])"
python - <<'PY'
import json
for f in ("mla", "shared"):
    for l in open(f"gpurun_out/vs/{f}.jsonl"):
        d = json.loads(l)
        print(f, d["P"], d["engine"], d["dir"], d["gbs"])
PY
