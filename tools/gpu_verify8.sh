#!/bin/bash
# Re-verification of the current tree after a container restore: smoke, every GPU test, the default
# bench, the reference arm, the launch list of the default bench.
O=gpurun_out/verify8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_all.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cut -c1-200 $O/bench.json
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>> $O/bench.err; cut -c1-200 $O/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-extras > $O/ncu_bench.log 2>&1; echo "ncu list rc=$?"
