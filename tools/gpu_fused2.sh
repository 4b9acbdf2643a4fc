#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for rep in a b; do for f in 1 0; do
  STRATA_LDG_FUSED=$f timeout 600 python tools/sweep.py --config llama8b_32k --pages 1 --ctas 1,2,4 --engines 1 --baselines 0 --tag fused$f$rep > gpurun_out/fused2_llama_$f$rep.jsonl 2>&1
done; done
for f in 1 0; do
  STRATA_LDG_FUSED=$f timeout 600 python tools/sweep.py --config llama70b_tp8 --pages 1 --ctas 1,2,4 --engines 1 --baselines 0 --tag fused$f > gpurun_out/fused2_70b_$f.jsonl 2>&1
  STRATA_LDG_FUSED=$f timeout 600 python tools/latency.py --engines 1 --reps 50 > gpurun_out/fused2_latency_$f.jsonl 2>&1
done
for f in gpurun_out/fused2_*.jsonl; do echo $f; grep -h '"gbs"' $f | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['dir'], d['ctas'], d['gbs'])"; done
