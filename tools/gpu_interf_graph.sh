#!/bin/bash
# Copy-engine interference: eager vs CUDA-graph proxies; engines x quota with graph-replayed proxies.
mkdir -p gpurun_out
timeout 600 python tools/ce_interference.py > gpurun_out/ce_interference2.jsonl 2> gpurun_out/ce_interference2.err; echo "ce rc=$?"; grep -v '"l2"' gpurun_out/ce_interference2.jsonl | cut -c1-220
timeout 900 python tools/interference.py --graph 1 --engines 1,4 --ctas 1,2,8 --memcpy 1 > gpurun_out/interference_graph.jsonl 2> gpurun_out/interference_graph.err; echo "interf rc=$?"; cut -c1-260 gpurun_out/interference_graph.jsonl
