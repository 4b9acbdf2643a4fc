#!/bin/bash
# Round 2: defaults fixed (ring 2 CTAs, 16 KiB pieces, 224 KiB in flight): bench, fast + slow GPU suites.
O=gpurun_out/r2_verify1; mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_fast.log 2>&1; echo "pytest rc=$?" >> $O/pytest_fast.log
timeout 2400 python -m pytest tests/test_gpu_fused.py tests/test_gpu_prefill.py tests/test_gpu_interference.py tests/test_gpu_fullsize.py -q -s --timeout 1200 > $O/pytest_slow.log 2>&1; echo "pytest rc=$?" >> $O/pytest_slow.log
tail -2 $O/smoke.log; tail -2 $O/bench.err; tail -3 $O/pytest_fast.log; grep -E "slowdown|passed|failed|FAILED" $O/pytest_slow.log | tail -20
