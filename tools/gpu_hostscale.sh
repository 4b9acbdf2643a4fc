#!/bin/bash
# Host-pool scale sweep: the same 32K-token load drawn from 2 / 8 / 32 / 70 GiB host
# tiers, 4 KiB pages (flags 0) vs transparent huge pages (flags 1).
mkdir -p gpurun_out
for fl in 0 1; do for hc in 256 1024 4096 8960; do
  python tools/sweep.py --pages 1 --ctas 2 --engines 1,4 --baselines 0 --host-chunks $hc --flags $fl --tag scale > gpurun_out/hs_${fl}_${hc}.jsonl 2>&1
  grep -h AnonHugePages /proc/meminfo
done; done
cat gpurun_out/hs_*.jsonl > gpurun_out/host_scale.jsonl
