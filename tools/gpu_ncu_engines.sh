#!/bin/bash
mkdir -p gpurun_out/ncu2
O=gpurun_out/ncu2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ldg_fused -s 1 -c 1 \
    -o $O/ldg_fused -f python tools/prof_one.py --engine 1 --layers 4 > $O/ldg.log 2>&1; echo "ldg rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tma_ws -s 2 -c 1 \
    -o $O/tma_ws -f python tools/prof_one.py --engine 2 --layers 3 > $O/tma.log 2>&1; echo "tma rc=$?"
ls -la $O
