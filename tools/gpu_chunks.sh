#!/bin/bash
# host chunk size C (the transfer unit of the page-first tier) vs throughput and host submission cost
mkdir -p gpurun_out/chunks
for C in 8 16 32 64 128 256; do
  for e in 0 1; do
    python bench.py --no-cpu-baseline --steps 10 --chunk-tokens $C --engine $e > gpurun_out/chunks/c${C}_e$e.json 2>> gpurun_out/chunks/err
    python -c "import json;d=json.load(open('gpurun_out/chunks/c${C}_e$e.json'));print('C=$C',d['engine'],d['value'],d['step_stats_rank0']['median_ms'],d['host_submit_ms_per_step'])"
  done
done
