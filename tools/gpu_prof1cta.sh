#!/bin/bash
# ncu of the single-CTA regime of each engine (why one SM does not reach the probe's 42-46 GB/s)
mkdir -p gpurun_out
python tools/sweep.py --pages 1 --ctas 1,2 --engines 1 --baselines 0 --threads 1024 --tag t1024 > gpurun_out/sweep_t1024.jsonl 2>&1 &
wait
for cfg in "1 512" "1 1024" "2 0" "3 0"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"(tma|ldg)" -s 1 -c 1 \
    -o gpurun_out/prof1_e$1_t$2 -f python tools/prof_one.py --engine $1 --ctas 1 --threads $2 --layers 2 > gpurun_out/ncu1_e$1_t$2.log 2>&1
  echo "ncu e$1 t$2 rc=$?"
done
