#!/bin/bash
# warp-specialised TMA offload: parity, then SM-quota sweep vs LDG (both directions reported).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --pages 1 --ctas 1,2,4,8 --engines 1,2 --baselines 0 > gpurun_out/sw_off_llama.jsonl 2> gpurun_out/sw_off.err; echo "sweep llama rc=$?"
timeout 900 python tools/sweep.py --config llama70b_tp8 --pages 1 --ctas 1,2,4,8 --engines 1,2 --baselines 0 > gpurun_out/sw_off_70b.jsonl 2>> gpurun_out/sw_off.err; echo "sweep 70b rc=$?"
grep d2h gpurun_out/sw_off_llama.jsonl gpurun_out/sw_off_70b.jsonl | python -c "
import sys,json
for l in sys.stdin:
    f,j=l.split(':',1); d=json.loads(j); print(f.split('/')[-1], d['engine'], d['ctas'], d.get('gbs'))"
