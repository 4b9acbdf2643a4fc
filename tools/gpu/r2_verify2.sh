#!/bin/bash
# Round 2 (re-entry): verify the committed tree on B200: smoke, bench (default ring), launch list,
# ncu --set full of the fused ring load (traffic for roofline), fast + slow GPU suites.
O=gpurun_out/r2_verify2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_load -s 1 -c 1 -o $O/ncu_ring_load_32L python tools/prof_one.py --layers 32 --engine 2 --reps 2 > $O/ncu_full.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_offload -s 1 -c 1 -o $O/ncu_ring_offload_32L python tools/prof_one.py --layers 32 --engine 2 --reps 2 --dir d2h > $O/ncu_full_off.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full_off.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_fast.log 2>&1; echo "pytest rc=$?" >> $O/pytest_fast.log
timeout 2400 python -m pytest tests -m "gpu and slow" -q -s --timeout 1200 > $O/pytest_slow.log 2>&1; echo "pytest rc=$?" >> $O/pytest_slow.log
tail -2 $O/build.log; tail -2 $O/smoke.log; tail -2 $O/bench.err; head -c 1200 $O/bench.json; echo; tail -3 $O/ncu_full.log; tail -3 $O/pytest_fast.log; grep -E "slowdown|passed|failed|FAILED" $O/pytest_slow.log | tail -20
