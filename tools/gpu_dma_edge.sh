#!/bin/bash
# DMA piece schedule: edge split (first/last layer in smaller pieces) A/B; fused-LDG last-layer event;
# parity of the DMA schedules.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dma or tiny or layer_events" > gpurun_out/pytest_dma.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dma.log
for e in 1 4; do
  STRATA_DMA_EDGE_SPLIT=$e python bench.py --no-cpu-baseline > gpurun_out/bench_edge$e.json 2>> gpurun_out/bench_edge.err
  echo "edge=$e rc=$?"; cut -c1-160 gpurun_out/bench_edge$e.json
  STRATA_DMA_EDGE_SPLIT=$e python bench.py --no-cpu-baseline --config llama70b_tp8 --steps 8 > gpurun_out/bench70_edge$e.json 2>> gpurun_out/bench_edge.err
done
python bench.py --no-cpu-baseline --config tiny --steps 50 > gpurun_out/bench_tiny.json 2>> gpurun_out/bench_edge.err; cut -c1-160 gpurun_out/bench_tiny.json
python bench.py --no-cpu-baseline --engine 1 > gpurun_out/bench_ldg.json 2>> gpurun_out/bench_edge.err; cut -c1-160 gpurun_out/bench_ldg.json
python tools/latency.py > gpurun_out/latency.jsonl 2>> gpurun_out/bench_edge.err; echo "latency rc=$?"
