#!/bin/bash
# Round 2: ring bulk-store variant vs st.global; 70B quotas; ncu 1-CTA both variants; fast tests.
O=gpurun_out/r2_ring6; mkdir -p $O
timeout 900 python tools/ring_sweep.py --configs llama8b_32k:1,llama8b_32k:16 --ctas 1,2 --warps 4,8 --gather-warps 4 --stage-kb 16,32 --bulk-store 0,1 --dirs load > $O/ring_sweep.jsonl 2> $O/ring_sweep.err
timeout 900 python tools/ring_sweep.py --configs llama70b_tp8:1,llama70b_tp8:16 --ctas 2,3,4 --warps 4,8 --gather-warps 2,4,8 --stage-kb 16 --bulk-store 0,1 >> $O/ring_sweep.jsonl 2>> $O/ring_sweep.err
for bs in 0 1; do
STRATA_RING_BULK_STORE=$bs timeout 300 ncu --set full --clock-control none --import-source on -k regex:ring_load -c 1 -o $O/ring_load_1cta_bs$bs \
  python tools/prof_one.py --engine 2 --ctas 1 --layers 4 --reps 1 > $O/ncu_bs$bs.log 2>&1
done
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
STRATA_RING_BULK_STORE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_heads.py -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_gpu_bulk.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_bulk.log
tail -3 $O/ring_sweep.err; tail -4 $O/pytest_gpu.log; tail -4 $O/pytest_gpu_bulk.log
