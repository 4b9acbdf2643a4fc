#!/bin/bash
# Final (static LDG body restored): smoke, default bench, the prefill overlap test 3x, the GPU suite.
O=gpurun_out/final6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['frac_of_link'], d['engine'], d['other_engines_gbs'], d['interference'])"
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_prefill.py -m gpu -q -p no:cacheprovider > $O/prefill_$i.log 2>&1; echo "prefill $i rc=$?"; tail -1 $O/prefill_$i.log; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > $O/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_all.log
grep -E "^FAILED|slowdown|uncapped|beside the offload" $O/pytest_gpu_all.log | head -30
