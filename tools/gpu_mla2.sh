#!/bin/bash
# magic-number row division (non-power-of-two rows): MLA parity + LDG/TMA bench; copy-engine interference diagnosis.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mla.py tests/test_gpu_parity.py -q -x -m "not slow" > gpurun_out/pytest_mla2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_mla2.log
python bench.py --config deepseek_v3_mla --no-cpu-baseline --engine 1 > gpurun_out/bench_mla_ldg2.json 2> gpurun_out/bench_mla2.err; echo "bench mla ldg rc=$?"; cut -c1-120 gpurun_out/bench_mla_ldg2.json
python bench.py --config deepseek_v3_mla > gpurun_out/bench_mla2.json 2>> gpurun_out/bench_mla2.err; echo "bench mla rc=$?"
timeout 600 python tools/ce_interference.py > gpurun_out/ce_interference.jsonl 2> gpurun_out/ce_interference.err; echo "ce_interference rc=$?"; cat gpurun_out/ce_interference.jsonl
