#!/bin/bash
# Round 2: ring geometry vs interference (decode / prefill proxies, cool-down method) and throughput.
O=gpurun_out/r2_interf2; mkdir -p $O
timeout 1500 python tools/interference.py --reps 20 --ring-configs 2:32:0:8,2:16:64:4,2:16:80:4,2:16:112:6,3:16:64:4,4:16:48:2,4:16:64:3,1:16:128:7,2:8:48:4,3:8:40:4,4:8:32:3 > $O/interference_ring_geom.jsonl 2> $O/interference.err
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q -s --timeout 900 > $O/pytest_prefill.log 2>&1; echo "pytest rc=$?" >> $O/pytest_prefill.log
tail -3 $O/interference.err; tail -5 $O/pytest_prefill.log
