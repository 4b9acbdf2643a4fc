#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -c 60 --csv --log-file gpurun_out/tiny_launches.csv \
    python bench.py --config tiny --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tiny_ncu.log 2>&1; echo "rc=$?"
for c in 2 4 8 16; do python bench.py --config tiny --no-cpu-baseline --steps 50 --num-ctas $c > gpurun_out/tiny_c$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/tiny_c$c.json'));print('ctas=$c',d['value'],d['ms_per_step'],d['per_layer_ms_last_step'])"; done
STRATA_LDG_FUSED=0 python bench.py --config tiny --no-cpu-baseline --steps 50 > gpurun_out/tiny_unfused.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/tiny_unfused.json'));print('unfused',d['value'],d['ms_per_step'],d['per_layer_ms_last_step'])"
