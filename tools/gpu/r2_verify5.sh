#!/bin/bash
# Round 2: whole -m gpu suite in one process (as the driver runs it) after the registration fallback
# + per-test collection; captured-op external events test; box memory facts.
O=gpurun_out/r2_verify5; mkdir -p $O
(free -g; ulimit -l; cat /proc/meminfo | head -5; nproc; ls /sys/devices/system/node/ | grep node) > $O/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_graph.py -q --timeout 300 > $O/pytest_graph.log 2>&1; echo "rc=$?" >> $O/pytest_graph.log
(while true; do grep -E "MemAvailable|Mlocked" /proc/meminfo | tr '\n' ' '; echo; sleep 10; done) > $O/mem_trace.txt 2>&1 &
MT=$!
timeout 3000 python -m pytest tests -m gpu -q --timeout 1200 > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
kill $MT
cat $O/box.txt; tail -3 $O/pytest_graph.log; grep -E "passed|failed|FAILED|Error" $O/pytest_all.log | tail -10; sort -t: -k2 -n $O/mem_trace.txt | head -3
