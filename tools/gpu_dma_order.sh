#!/bin/bash
# A/B of the DMA piece barrier (STRATA_DMA_ORDERED): bench throughput, per-layer event spacing, and
# the layer-wise prefill stall it feeds (tools/prefill_overlap.py).
mkdir -p gpurun_out
for o in 0 1; do
  STRATA_DMA_ORDERED=$o python bench.py --no-cpu-baseline > gpurun_out/bench_ordered$o.json 2>> gpurun_out/bench_order.err
  echo "ordered=$o rc=$?"; cut -c1-200 gpurun_out/bench_ordered$o.json
  STRATA_DMA_ORDERED=$o python bench.py --no-cpu-baseline --config llama70b_tp8 --steps 5 > gpurun_out/bench70_ordered$o.json 2>> gpurun_out/bench_order.err
  STRATA_DMA_ORDERED=$o python tools/prefill_overlap.py --engines 4 --baseline 0 --new 512,1024,2048,4096 > gpurun_out/prefill_ordered$o.jsonl 2>> gpurun_out/bench_order.err
  echo "prefill rc=$?"
done
