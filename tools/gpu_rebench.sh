#!/bin/bash
mkdir -p gpurun_out/rebench
nvidia-smi topo -m > gpurun_out/rebench/topo.txt 2>&1; nvidia-smi --query-gpu=index,name,utilization.gpu,pcie.link.gen.current,pcie.link.width.current --format=csv >> gpurun_out/rebench/topo.txt 2>&1
uptime >> gpurun_out/rebench/topo.txt
for r in 1 2 3; do python bench.py --no-cpu-baseline > gpurun_out/rebench/b$r.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/rebench/b$r.json'));print(d['value'],d['roofline']['peak'],d['step_stats_rank0']['median_ms'],d['step_stats_rank0']['cv'])"; done
cat gpurun_out/rebench/topo.txt | tail -8
