#!/bin/bash
# Round 2: ring engine v2 (index lookahead 4, cp.async offload gather): sweep with parity, then the fast GPU suite.
O=gpurun_out/r2_ring2; mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 700 python tools/ring_sweep.py --ctas 1,2 --stage-kb 16,32,64 > $O/ring_sweep.jsonl 2> $O/ring_sweep.err; echo "sweep rc=$?" >> $O/ring_sweep.err
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/smoke.log; tail -3 $O/ring_sweep.err; tail -30 $O/pytest_gpu.log
