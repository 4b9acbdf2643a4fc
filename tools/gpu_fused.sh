#!/bin/bash
# Fused (one launch for all layers) vs per-layer LDG: parity suite, A/B sweeps, latency, overlap.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for f in 1 0; do
  STRATA_LDG_FUSED=$f timeout 600 python tools/sweep.py --config llama8b_32k --pages 1 --ctas 1,2,4 --engines 1 --baselines 0 --tag fused$f > gpurun_out/fused_ab_llama_$f.jsonl 2>&1
  STRATA_LDG_FUSED=$f timeout 600 python tools/sweep.py --config llama70b_tp8 --pages 1 --ctas 1,2,4 --engines 1 --baselines 0 --tag fused$f > gpurun_out/fused_ab_70b_$f.jsonl 2>&1
  STRATA_LDG_FUSED=$f timeout 600 python tools/latency.py --engines 1 --reps 50 > gpurun_out/fused_latency_$f.jsonl 2>&1
done
STRATA_LDG_FUSED=1 timeout 600 python tools/sweep.py --config llama8b_32k --pages 1 --ctas 1,2,4 --engines 1 --baselines 0 --tag fused1b > gpurun_out/fused_ab_llama_1b.jsonl 2>&1
STRATA_LDG_FUSED=0 timeout 600 python tools/sweep.py --config llama8b_32k --pages 1 --ctas 1,2,4 --engines 1 --baselines 0 --tag fused0b > gpurun_out/fused_ab_llama_0b.jsonl 2>&1
timeout 600 python tools/overlap.py > gpurun_out/overlap_fused.jsonl 2>&1
grep -h gbs gpurun_out/fused_ab_*.jsonl | head -40
cat gpurun_out/fused_latency_*.jsonl
