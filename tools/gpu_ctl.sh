#!/bin/bash
# NEXT-4 on the GPU: control-plane-driven load/write-back parity, then the serving-loop replay.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ctl.py -q -x > gpurun_out/pytest_ctl.log 2>&1
timeout 900 python tools/ctl_bench.py --order max > gpurun_out/ctl_bench_max.jsonl 2> gpurun_out/ctl_bench_max.err
timeout 900 python tools/ctl_bench.py --order min > gpurun_out/ctl_bench_min.jsonl 2> gpurun_out/ctl_bench_min.err
timeout 600 python tools/ctl_bench.py --order max --page-size 16 --policies strata > gpurun_out/ctl_bench_p16.jsonl 2> gpurun_out/ctl_bench_p16.err
timeout 600 python tools/ctl_bench.py --cpu > gpurun_out/ctl_bench_cpu.jsonl 2>&1
tail -3 gpurun_out/pytest_ctl.log
cat gpurun_out/ctl_bench_*.jsonl
