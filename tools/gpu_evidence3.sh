#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/pcie_counters.py > gpurun_out/pcie_counters.jsonl 2> gpurun_out/pcie_counters.err; echo "pcie rc=$?"; cat gpurun_out/pcie_counters.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ldg -s 4 -c 1 \
    -o gpurun_out/prof_dma_scatter3 -f python tools/prof_one.py --engine 4 --layers 3 --reps 1 > gpurun_out/ncu_dma3.log 2>&1; echo "ncu dma rc=$?"
