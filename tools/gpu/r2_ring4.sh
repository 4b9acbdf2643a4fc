#!/bin/bash
# Round 2: ring v3 (warp-owned rows): sweep, ncu 1-CTA, GPU fast suite, slow full-size + slot race.
O=gpurun_out/r2_ring4; mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python tools/ring_sweep.py --ctas 1,2 --warps 4,8,16 --gather-warps 4,8,16 --stage-kb 16,32,64 > $O/ring_sweep.jsonl 2> $O/ring_sweep.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ring_load -c 1 -o $O/ring_load_1cta \
  python tools/prof_one.py --engine 2 --ctas 1 --layers 4 --reps 1 > $O/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ring_offload -c 1 -o $O/ring_offload_1cta \
  python tools/prof_one.py --engine 2 --ctas 1 --layers 4 --reps 1 --dir d2h > $O/ncu2.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1500 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fullsize.py -x -q --timeout 900 > $O/pytest_slow.log 2>&1; echo "pytest rc=$?" >> $O/pytest_slow.log
tail -2 $O/smoke.log; tail -3 $O/ring_sweep.err; tail -4 $O/pytest_gpu.log; tail -15 $O/pytest_slow.log
