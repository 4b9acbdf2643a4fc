#!/bin/bash
# Round 2: what makes an I/O kernel slow a co-running HBM-bound decode?  (device-pool footprint, host
# page size, page writes, page size) at one ring geometry; LDG reference.
O=gpurun_out/r2_interf3; mkdir -p $O
R="2:16:112:6,2:16:144:8,2:16:0:7"
I="timeout 900 python tools/interference.py --reps 20"
$I --ring-configs $R --tag base > $O/interf.jsonl 2>> $O/err.txt
$I --ring-configs $R --layers 4 --tag L4 >> $O/interf.jsonl 2>> $O/err.txt
$I --ring-configs $R --flags 1 --tag thp >> $O/interf.jsonl 2>> $O/err.txt
$I --ring-configs 2:16:112:6:1,2:16:0:7:1 --tag nostore >> $O/interf.jsonl 2>> $O/err.txt
$I --ring-configs $R --P 16 --tag P16 >> $O/interf.jsonl 2>> $O/err.txt
$I --engines 1 --ctas 2 --tag ldg >> $O/interf.jsonl 2>> $O/err.txt
$I --engines 1 --ctas 2 --flags 1 --tag ldg_thp >> $O/interf.jsonl 2>> $O/err.txt
$I --engines 1 --ctas 2 --layers 4 --tag ldg_L4 >> $O/interf.jsonl 2>> $O/err.txt
tail -3 $O/err.txt
