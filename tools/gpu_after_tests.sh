#!/bin/bash
# Does the link slow down after the full-size tests free tens of GiB of pinned memory?
mkdir -p gpurun_out/after
O=gpurun_out/after
python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.read());print('before', d['value'], d['roofline']['peak'], d['step_stats_rank0']['cv'], d['clocks'].get('pcie_link'))"
timeout 1800 python -m pytest tests -m "gpu and slow" -q -x > $O/slow.log 2>&1; echo "slow rc=$?"
for i in 1 2 3 4; do
  date +%T; grep -E "MemFree|Dirty|Writeback:|AnonHugePages" /proc/meminfo | tr '\n' ' '; echo
  python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.read());print('after', d['value'], d['roofline']['peak'], d['step_stats_rank0']['cv'], d['clocks'].get('pcie_link'), d['remeasured'])"
  sleep 20
done
