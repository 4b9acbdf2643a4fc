#!/bin/bash
# End-of-round check of the final tree: smoke, the whole GPU suite as the driver runs it (-x), bench.
O=gpurun_out/final7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_all.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['frac_of_link'], d['engine'], d['e2e'], d['interference'])"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>> $O/bench.err; cut -c1-120 $O/bench_reference.json
