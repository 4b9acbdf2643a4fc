#!/bin/bash
# Box probe: hardware facts + link ceilings. Run under gpurun from the repo root.
mkdir -p gpurun_out
{
nvidia-smi -q | grep -E -A3 -i "Product Name|PCIe Generation|Link Width|Max|Current" | head -60
nvidia-smi topo -m
lscpu | head -30
numactl -H 2>/dev/null || echo "no numactl"
cat /proc/meminfo | grep -i -E "huge|MemTotal"
cat /sys/kernel/mm/transparent_hugepage/enabled
nproc
nvidia-smi --query-gpu=index,pci.bus_id,clocks.sm,clocks.max.sm --format=csv
} > gpurun_out/probe_box.txt 2>&1
timeout 600 ./tools/probe/probe > gpurun_out/probe.jsonl 2> gpurun_out/probe.err
echo "probe exit $?"
tail -3 gpurun_out/probe.jsonl
