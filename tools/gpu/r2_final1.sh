#!/bin/bash
# Round 2: full verification of the current tree: build, smoke, bench (default), whole GPU suite,
# ncu launch list of the bench and ncu --set full of the load + offload kernels.
O=gpurun_out/r2_final1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_load -s 1 -c 1 -o $O/ncu_ring_load_32L python tools/prof_one.py --layers 32 --engine 2 --reps 2 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_offload -s 1 -c 1 -o $O/ncu_ring_offload_32L python tools/prof_one.py --layers 32 --engine 2 --reps 2 --dir d2h > $O/ncu_full_off.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q --timeout 1200 > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
tail -1 $O/build.log; tail -2 $O/smoke.log; tail -1 $O/bench.err; python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['frac_of_link'], d['offload'], d['gpu_launches'], d['clocks'], d.get('interference'))"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -5
