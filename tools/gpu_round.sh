#!/bin/bash
# generic GPU pass: fast GPU tests, then the named extras
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
./tools/probe/tma_probe > gpurun_out/tma_probe.jsonl 2>&1; echo "tma_probe rc=$?"
python tools/sweep.py --pages 1 --ctas 1,2,4,8 --engines 1,4 --baselines 0 > gpurun_out/sweep_ldg32.jsonl 2>&1; echo "sweep rc=$?"
