#!/bin/bash
# GPU test pass under gpurun: smoke, fast parity tests, then the full-size configs.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest fast rc=$?" | tee -a gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
if [ "$1" == "slow" ]; then
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/pytest_gpu_slow.log 2>&1; echo "pytest slow rc=$?" | tee -a gpurun_out/pytest_gpu_slow.log
tail -15 gpurun_out/pytest_gpu_slow.log
fi
