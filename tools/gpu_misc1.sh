#!/bin/bash
# bubble filling with graph-replayed decode; MLA layer groups.
mkdir -p gpurun_out
timeout 900 python tools/bubble_fill.py --graph 1 > gpurun_out/bubble_fill_graph.jsonl 2> gpurun_out/bubble_fill_graph.err; echo "bubble rc=$?"; cut -c1-400 gpurun_out/bubble_fill_graph.jsonl
for G in 1 2 4; do
python bench.py --config deepseek_v3_mla --no-cpu-baseline --layer-group $G --steps 10 > gpurun_out/bench_mla_g$G.json 2>> gpurun_out/bench_g.err; echo "mla G=$G rc=$?"; cut -c1-110 gpurun_out/bench_mla_g$G.json
done
