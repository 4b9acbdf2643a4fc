#!/bin/bash
# End-of-session check with the final code: smoke, every GPU test (incl. full-size), default bench
# twice, the reference arm, the launch list of the default bench.
mkdir -p gpurun_out/final3
O=gpurun_out/final3
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu_all.log
for r in 1 2; do python bench.py > $O/bench_rep$r.json 2>> $O/err; echo "bench rc=$?"; cut -c1-140 $O/bench_rep$r.json; done
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>> $O/err; cut -c1-140 $O/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu list rc=$?"
