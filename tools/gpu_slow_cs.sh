#!/bin/bash
# full-size slow parity (incl. MLA and shared-tier configs) + copy-stream count A/B with the piece barrier.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m "gpu and slow" -q -x > gpurun_out/pytest_gpu_slow.log 2>&1; echo "slow rc=$?"; tail -3 gpurun_out/pytest_gpu_slow.log
for n in 1 2 3 4 6 8; do
  STRATA_COPY_STREAMS=$n python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cs$n.json 2>> gpurun_out/bench_cs.err
  python -c "import json;d=json.load(open('gpurun_out/bench_cs$n.json'));print('streams=$n',d['value'],d['step_stats_rank0']['median_ms'],[round(x,2) for x in d['per_layer_ms_last_step'][:3]])"
done
