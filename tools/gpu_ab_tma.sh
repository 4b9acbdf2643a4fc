#!/bin/bash
# A: per-thread arrivals on both barriers; B: per-thread on `full`, per-warp on `empty`.
mkdir -p gpurun_out/abtma
D=paper_2508_18572_b200
for v in A B A B; do
  cp $D/libstrata_$v.so $D/libstrata.so
  for c in 2 4; do python bench.py --no-cpu-baseline --engine 2 --num-ctas $c --steps 10 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.read());print('$v ctas=$c',d['value'])"; done
done
cp $D/libstrata_B.so $D/libstrata.so
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny_load_offload or special_float" > gpurun_out/abtma/racecheck_B.log 2>&1; echo "racecheck B rc=$?"; grep -E "SUMMARY" gpurun_out/abtma/racecheck_B.log | tail -1
