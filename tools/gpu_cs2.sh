#!/bin/bash
# copy streams 1 vs 4 across configs and directions; small-load LDG planning (tiny).
mkdir -p gpurun_out/cs
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m "not slow" > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/pytest_parity.log
for n in 1 4; do
  for cfg in "llama8b_32k --page-size 16" "llama70b_tp8" "qwen14b_batch8 --steps 4" "deepseek_v3_mla" "llama70b_tp8_shared"; do
    tag=$(echo $cfg | tr ' ' '_' | tr -d '-')
    STRATA_COPY_STREAMS=$n python bench.py --no-cpu-baseline --steps 8 --config $cfg > gpurun_out/cs/b_${tag}_cs$n.json 2>> gpurun_out/cs/err
    python -c "import json;d=json.load(open('gpurun_out/cs/b_${tag}_cs$n.json'));print('$tag cs=$n',d['value'],d['step_stats_rank0']['median_ms'])"
  done
  STRATA_COPY_STREAMS=$n timeout 600 python tools/sweep.py --pages 1 --ctas 8 --engines 4 --baselines 0 > gpurun_out/cs/sweep_dma_cs$n.jsonl 2>> gpurun_out/cs/err
  STRATA_COPY_STREAMS=$n timeout 600 python tools/sweep.py --config llama70b_tp8 --pages 1 --ctas 8 --engines 4 --baselines 0 > gpurun_out/cs/sweep70_dma_cs$n.jsonl 2>> gpurun_out/cs/err
  STRATA_COPY_STREAMS=$n timeout 600 python tools/bidir.py > gpurun_out/cs/bidir_cs$n.jsonl 2>> gpurun_out/cs/err
done
grep -h d2h gpurun_out/cs/sweep*_cs*.jsonl | cut -c1-250
python bench.py --no-cpu-baseline --config tiny --steps 50 > gpurun_out/bench_tiny.json 2>> gpurun_out/cs/err; cut -c1-200 gpurun_out/bench_tiny.json
python tools/latency.py > gpurun_out/latency.jsonl 2>> gpurun_out/cs/err; head -4 gpurun_out/latency.jsonl
