#!/bin/bash
# Round 2: what bounds the ring engine at ONE CTA (host page size / chunk order / page order), ncu of the
# 1-CTA load kernel, and the slow full-size + slot-race tests.
O=gpurun_out/r2_ring3; mkdir -p $O
S="timeout 300 python tools/ring_sweep.py --configs llama8b_32k:1 --ctas 1 --warps 8 --gather-warps 8 --stage-kb 32,64"
$S --tag base > $O/one_cta.jsonl 2>>$O/err.txt
$S --tag chunks_identity --chunk-frag identity >> $O/one_cta.jsonl 2>>$O/err.txt
$S --tag pages_identity --frag identity >> $O/one_cta.jsonl 2>>$O/err.txt
$S --tag thp --flags 1 >> $O/one_cta.jsonl 2>>$O/err.txt
$S --tag cudahostalloc --flags 16 >> $O/one_cta.jsonl 2>>$O/err.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ring_load -c 1 -o $O/ring_load_1cta \
  python tools/prof_one.py --engine 2 --ctas 1 --layers 4 --reps 1 > $O/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ring_offload -c 1 -o $O/ring_offload_1cta \
  python tools/prof_one.py --engine 2 --ctas 1 --layers 4 --reps 1 --dir d2h > $O/ncu2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fullsize.py -x -q --timeout 900 > $O/pytest_slow.log 2>&1; echo "pytest rc=$?" >> $O/pytest_slow.log
tail -3 $O/err.txt; tail -20 $O/pytest_slow.log
