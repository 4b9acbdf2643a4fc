#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_concurrent.py -q -x > gpurun_out/pytest_conc.log 2>&1; echo "conc rc=$?"; tail -3 gpurun_out/pytest_conc.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python tools/bidir.py > gpurun_out/bidir.jsonl 2> gpurun_out/bidir.err; echo "bidir rc=$?"; cut -c1-250 gpurun_out/bidir.jsonl
timeout 600 python tools/bidir.py --offload-engine 1 > gpurun_out/bidir_ldg_off.jsonl 2>> gpurun_out/bidir.err; echo "bidir2 rc=$?"; cut -c1-250 gpurun_out/bidir_ldg_off.jsonl
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>/dev/null; cut -c1-150 gpurun_out/bench.json
