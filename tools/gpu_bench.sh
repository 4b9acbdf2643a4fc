#!/bin/bash
# Bench + sweep + ncu evidence under gpurun (one GPU).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
python bench.py --engine 1 --no-cpu-baseline > gpurun_out/bench_ldg.json 2>> gpurun_out/bench.err; echo "bench ldg rc=$?"
python bench.py --page-size 16 --no-cpu-baseline > gpurun_out/bench_p16.json 2>> gpurun_out/bench.err; echo "bench p16 rc=$?"
timeout 900 python tools/sweep.py --pages 1,16,64 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
for eng in 2 1; do
  for dir in h2d d2h; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"(tma|ldg)_kernel" -s 2 -c 1 \
      -o gpurun_out/prof_e${eng}_${dir} -f python tools/prof_one.py --engine $eng --dir $dir > gpurun_out/ncu_e${eng}_${dir}.log 2>&1
    echo "ncu full e$eng $dir rc=$?"
  done
done
