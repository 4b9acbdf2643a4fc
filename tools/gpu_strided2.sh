#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --config llama70b_tp8_shared --chunk-frag identity --steps 8 > gpurun_out/bench_shared_ident.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_shared_ident.json'));print('shared ident',d['value'],d['host_submit_ms_per_step'])"
