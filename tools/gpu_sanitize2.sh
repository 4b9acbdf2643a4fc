#!/bin/bash
mkdir -p gpurun_out/sanitize
S=gpurun_out/sanitize
K="tiny_load_offload or special_float"
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -q -x -k "$K" > $S/racecheck2.log 2>&1; echo "racecheck rc=$?"; grep -E "SUMMARY|passed|failed" $S/racecheck2.log | tail -2
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -q -x -k "$K" > $S/synccheck2.log 2>&1; echo "synccheck rc=$?"; grep -E "SUMMARY|passed|failed" $S/synccheck2.log | tail -2
STRATA_DMA_NO_BATCH=1 timeout 1200 compute-sanitizer --tool initcheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -q -x -k "$K" > $S/initcheck_nobatch.log 2>&1; echo "initcheck no-batch rc=$?"; grep -E "SUMMARY|passed|failed" $S/initcheck_nobatch.log | tail -2
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrent.py -q -x -k "$K or in_flight" > $S/memcheck2.log 2>&1; echo "memcheck rc=$?"; grep -E "SUMMARY|passed|failed" $S/memcheck2.log | tail -2
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --engine 2 > gpurun_out/bench_tma.json 2>/dev/null; cut -c1-120 gpurun_out/bench_tma.json
