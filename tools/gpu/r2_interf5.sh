#!/bin/bash
# Round 2: exclusive-SM ring CTAs vs shared ones (interference), and the bubble-fill scheduling test.
O=gpurun_out/r2_interf5; mkdir -p $O
I="timeout 1200 python tools/interference.py --reps 20"
$I --ring-configs 2:16:112:6:0,2:16:112:6:1,2:16:128:7:1,2:16:144:8:1,2:8:112:6:1,1:16:128:7:1,2:16:96:5:1 --tag excl > $O/interf.jsonl 2>> $O/err.txt
$I --engines 1 --ctas 1,2 --tag ldg >> $O/interf.jsonl 2>> $O/err.txt
for ex in 0 1; do
STRATA_RING_INFLIGHT_KB=96 STRATA_RING_EXCLUSIVE=$ex timeout 600 python -m pytest tests/test_gpu_prefill.py -k bubble -x -q -s --timeout 600 > $O/bubble_excl$ex.log 2>&1; echo "rc=$?" >> $O/bubble_excl$ex.log
done
tail -3 $O/err.txt; tail -3 $O/bubble_excl0.log; tail -3 $O/bubble_excl1.log
