#!/bin/bash
# head slices / head-major host tiers (R28): parity, regression of the rest, shared-tier bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_heads.py -q -x > gpurun_out/pytest_heads.log 2>&1; echo "pytest heads rc=$?"; tail -15 gpurun_out/pytest_heads.log
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py --config llama70b_tp8_shared --no-cpu-baseline --steps 10 > gpurun_out/bench_70b_shared.json 2> gpurun_out/bench_heads.err; echo "bench shared rc=$?"; cut -c1-200 gpurun_out/bench_70b_shared.json
python bench.py --config llama70b_tp8_shared --no-cpu-baseline --steps 10 --engine 1 > gpurun_out/bench_70b_shared_ldg.json 2>> gpurun_out/bench_heads.err; echo "bench shared ldg rc=$?"
python bench.py --config llama70b_tp8 --no-cpu-baseline --steps 10 > gpurun_out/bench_70b.json 2>> gpurun_out/bench_heads.err; echo "bench 70b rc=$?"; cut -c1-200 gpurun_out/bench_70b.json
python bench.py > gpurun_out/bench.json 2>> gpurun_out/bench_heads.err; echo "bench rc=$?"; cut -c1-200 gpurun_out/bench.json
