#!/bin/bash
O=gpurun_out/prof_quota; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/prof_quota.py > $O/plain.log 2>&1; echo "plain rc=$?"; cat $O/plain.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ldg_quota_kernel -c 1 -o $O/ncu_ldg_quota_32L \
  python tools/prof_quota.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
