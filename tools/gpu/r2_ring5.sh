#!/bin/bash
# Round 2: ring v4 (warp-per-piece, W | S): sweep, ncu 1-CTA, GPU fast suite.
O=gpurun_out/r2_ring5; mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python tools/ring_sweep.py --ctas 1,2 --warps 2,4,8 --gather-warps 2,4,8 --stage-kb 16,24,32,48 > $O/ring_sweep.jsonl 2> $O/ring_sweep.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ring_load -c 1 -o $O/ring_load_1cta \
  python tools/prof_one.py --engine 2 --ctas 1 --layers 4 --reps 1 > $O/ncu1.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/smoke.log; tail -3 $O/ring_sweep.err; tail -4 $O/pytest_gpu.log
