#!/bin/bash
# Evidence refresh after the DMA schedule / MLA / head-slice changes: smoke, PCIe counters,
# launch list of the default bench, ncu --set full of the DMA scatter and of the MLA LDG kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python tools/pcie_counters.py > gpurun_out/pcie_counters.jsonl 2> gpurun_out/pcie_counters.err; echo "pcie rc=$?"; cat gpurun_out/pcie_counters.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ldg -s 2 -c 1 \
    -o gpurun_out/prof_dma_scatter2 -f python tools/prof_one.py --engine 4 --layers 3 > gpurun_out/ncu_dma.log 2>&1; echo "ncu dma rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ldg -s 1 -c 1 \
    -o gpurun_out/prof_mla_ldg -f python tools/prof_one.py --config deepseek_v3_mla --engine 1 --layers 2 > gpurun_out/ncu_mla.log 2>&1; echo "ncu mla rc=$?"
ls -la gpurun_out/*.ncu-rep
