#!/bin/bash
# Round-end evidence: smoke, default bench (+variants), bidirectional mixes, launch list + ncu of the default path.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench.json
python bench.py --page-size 16 --no-cpu-baseline > gpurun_out/bench_p16.json 2>> gpurun_out/bench.err; echo "bench p16 rc=$?"
python bench.py --config llama70b_tp8 --no-cpu-baseline --steps 10 > gpurun_out/bench_70b.json 2>> gpurun_out/bench.err; echo "bench 70b rc=$?"
python bench.py --config qwen14b_batch8 --no-cpu-baseline --steps 5 > gpurun_out/bench_qwen.json 2>> gpurun_out/bench.err; echo "bench qwen rc=$?"
python bench.py --config tiny --no-cpu-baseline --steps 50 > gpurun_out/bench_tiny.json 2>> gpurun_out/bench.err; echo "bench tiny rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "bench ref rc=$?"
python tools/bidir.py > gpurun_out/bidir.jsonl 2>&1; echo "bidir rc=$?"
python tools/bidir.py --offload-engine 1 > gpurun_out/bidir_ldg_off.jsonl 2>&1; echo "bidir2 rc=$?"
python tools/bidir.py --load-engine 2 --offload-engine 4 > gpurun_out/bidir_tma_dma.jsonl 2>&1; echo "bidir3 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ldg -s 1 -c 1 \
    -o gpurun_out/prof_dma_scatter -f python tools/prof_one.py --engine 4 --layers 2 > gpurun_out/ncu_dma.log 2>&1; echo "ncu dma rc=$?"
