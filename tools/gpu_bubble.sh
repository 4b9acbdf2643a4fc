#!/bin/bash
O=gpurun_out/bubble; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_prefill.py -m gpu -q -s -p no:cacheprovider > $O/run_$i.log 2>&1; echo "run $i rc=$? $(tail -1 $O/run_$i.log)"; grep "load beside decode" $O/run_$i.log; done
timeout 1500 python -m pytest tests/test_gpu_quota.py tests/test_gpu_stress.py -x -q -m gpu -p no:cacheprovider > $O/rest.log 2>&1; echo "rest rc=$? $(tail -1 $O/rest.log)"
