#!/bin/bash
# Round-end evidence with the current defaults (one copy stream, edge pieces): tests, bench lines,
# launch list, interference / overlap / bubble filling with graph-replayed decode.
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 1800 python -m pytest tests -m "gpu and slow" -q -x > $O/pytest_gpu_slow.log 2>&1; echo "pytest slow rc=$?"; tail -1 $O/pytest_gpu_slow.log
for r in 1 2 3; do python bench.py > $O/bench_rep$r.json 2>> $O/err; echo "bench rep$r rc=$?"; cut -c1-140 $O/bench_rep$r.json; done
python bench.py --page-size 16 --no-cpu-baseline > $O/bench_p16.json 2>> $O/err
python bench.py --config llama70b_tp8 --no-cpu-baseline --steps 10 > $O/bench_70b_tp8.json 2>> $O/err
python bench.py --config qwen14b_batch8 --no-cpu-baseline --steps 5 > $O/bench_qwen14b.json 2>> $O/err
python bench.py --config tiny --no-cpu-baseline --steps 50 > $O/bench_tiny.json 2>> $O/err
python bench.py --config deepseek_v3_mla > $O/bench_mla.json 2>> $O/err
python bench.py --config llama70b_tp8_shared --no-cpu-baseline --steps 10 > $O/bench_70b_shared.json 2>> $O/err
python bench.py --engine 1 --no-cpu-baseline > $O/bench_engine_ldg.json 2>> $O/err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_oracle.json 2>> $O/err
for f in $O/bench_*.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f',d['value'],d.get('frac_of_link'),d.get('engine'))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 python tools/interference.py --graph 1 --engines 1,4 --ctas 1,2,8 --memcpy 1 > $O/interference_graph.jsonl 2>> $O/err; echo "interf rc=$?"
timeout 900 python tools/bubble_fill.py --graph 1 > $O/bubble_fill_graph.jsonl 2>> $O/err; echo "bubble rc=$?"
timeout 900 python tools/prefill_overlap.py --engines 4,1 --baseline 0 > $O/prefill_p1.jsonl 2>> $O/err; echo "prefill rc=$?"
timeout 600 python tools/bidir.py > $O/bidir.jsonl 2>> $O/err; echo "bidir rc=$?"
