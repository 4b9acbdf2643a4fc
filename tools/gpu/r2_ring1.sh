#!/bin/bash
# Round 2: first hardware pass of the ring engine: smoke, ring geometry sweep (with parity checks), GPU test suite.
O=gpurun_out/r2_ring1; mkdir -p $O
nvidia-smi -q | grep -iE "Link Gen|Link Width|Product Name" | head -8 > $O/box.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python tools/ring_sweep.py > $O/ring_sweep.jsonl 2> $O/ring_sweep.err; echo "sweep rc=$?" >> $O/ring_sweep.err
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -5 $O/smoke.log; tail -3 $O/ring_sweep.err; tail -30 $O/pytest_gpu.log
