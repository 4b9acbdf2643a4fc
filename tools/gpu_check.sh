#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for e in 4 1; do timeout 600 python tools/overlap.py --engine $e --tokens 32768 --check >> gpurun_out/overlap.jsonl 2>> gpurun_out/overlap.err; echo "overlap e=$e rc=$?"; done; cut -c1-300 gpurun_out/overlap.jsonl | head
