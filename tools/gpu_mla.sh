#!/bin/bash
# Single-buffer (MLA latent) pools: parity + bench of the DeepSeek-V3 latent geometry.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mla.py -q -x > gpurun_out/pytest_mla.log 2>&1; echo "pytest mla rc=$?"; tail -3 gpurun_out/pytest_mla.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_graph.py -q -x -m "not slow" > gpurun_out/pytest_parity.log 2>&1; echo "pytest parity rc=$?"; tail -2 gpurun_out/pytest_parity.log
python bench.py --config deepseek_v3_mla --no-cpu-baseline > gpurun_out/bench_mla.json 2> gpurun_out/bench_mla.err; echo "bench mla rc=$?"; cut -c1-300 gpurun_out/bench_mla.json
python bench.py --config deepseek_v3_mla --no-cpu-baseline --engine 1 > gpurun_out/bench_mla_ldg.json 2>> gpurun_out/bench_mla.err; echo "bench mla ldg rc=$?"
python bench.py --config deepseek_v3_mla --no-cpu-baseline --page-size 64 > gpurun_out/bench_mla_p64.json 2>> gpurun_out/bench_mla.err; echo "bench mla p64 rc=$?"
python bench.py --no-cpu-baseline --config tiny --steps 50 > gpurun_out/bench_tiny.json 2>> gpurun_out/bench_mla.err; cut -c1-200 gpurun_out/bench_tiny.json
