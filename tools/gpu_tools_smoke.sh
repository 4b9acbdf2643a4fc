#!/bin/bash
# every measurement tool still runs against the final library (short settings)
mkdir -p gpurun_out/tools
O=gpurun_out/tools
timeout 900 python tools/ctl_bench.py --order max > $O/ctl_bench.jsonl 2> $O/ctl.err; echo "ctl_bench rc=$?"; cut -c1-200 $O/ctl_bench.jsonl | tail -3
timeout 600 python tools/disk_bench.py --threads 4 --reps 2 > $O/disk_bench.jsonl 2> $O/disk.err; echo "disk_bench rc=$?"; cut -c1-200 $O/disk_bench.jsonl
timeout 600 python tools/latency.py --reps 20 > $O/latency.jsonl 2> $O/lat.err; echo "latency rc=$?"
timeout 600 python tools/pcie_counters.py --ops 4 --engines 4,1 > $O/pcie.jsonl 2> $O/pcie.err; echo "pcie rc=$?"
timeout 600 python tools/sweep.py --pages 16 --ctas 0 --engines 4 --baselines 0 --config deepseek_v3_mla > $O/sweep_mla.jsonl 2> $O/sw.err; echo "sweep mla rc=$?"; cut -c1-200 $O/sweep_mla.jsonl
