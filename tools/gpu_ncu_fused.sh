#!/bin/bash
# ncu: fused vs per-layer LDG kernel at 1 and 2 CTAs (Llama-8B 32K, 4 layers)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for mode in force 0; do for c in 1 2; do
  STRATA_LDG_FUSED=$mode timeout 600 ncu --set full --clock-control none --import-source on -k regex:ldg -c 1 \
    -o gpurun_out/ncu_fused_${mode}_c$c python tools/prof_one.py --engine 1 --ctas $c --layers 4 --reps 1 > gpurun_out/ncu_fused_${mode}_c$c.log 2>&1
done; done
ls -la gpurun_out/*.ncu-rep
