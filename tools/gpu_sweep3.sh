#!/bin/bash
# fig:loading with the current defaults: GB/s vs page size 1-64 for every engine at its default SM
# quota, the per-page / batched DMA baselines and the contiguous roofline; churn fragmentation.
mkdir -p gpurun_out/sweep3
timeout 2400 python tools/sweep.py --pages 1,2,4,8,16,32,64 --ctas 0 --engines 1,2,4 --baselines 1 > gpurun_out/sweep3/llama_pages.jsonl 2> gpurun_out/sweep3/err; echo "llama rc=$?"
timeout 1200 python tools/sweep.py --pages 1,16 --ctas 0 --engines 1,4 --baselines 0 --frag churn > gpurun_out/sweep3/llama_churn.jsonl 2>> gpurun_out/sweep3/err; echo "churn rc=$?"
timeout 1800 python tools/sweep.py --config llama70b_tp8 --pages 1,16,64 --ctas 0 --engines 1,4 --baselines 0 > gpurun_out/sweep3/70b_pages.jsonl 2>> gpurun_out/sweep3/err; echo "70b rc=$?"
python - <<'PY'
import json
for f in ("llama_pages", "llama_churn", "70b_pages"):
    for l in open(f"gpurun_out/sweep3/{f}.jsonl"):
        d = json.loads(l)
        print(f, d["P"], d["method"], d["dir"], d.get("engine"), d["gbs"])
PY
