#!/bin/bash
# Round 2: the knee of the throughput / decode-interference frontier (ring geometries vs LDG).
O=gpurun_out/r2_interf4; mkdir -p $O
I="timeout 1200 python tools/interference.py --reps 20"
$I --ring-configs 2:8:112:6,2:8:128:7,2:16:128:7,3:16:80:4,4:8:64:6,2:32:112:3,2:16:96:5,3:8:64:7 --tag knee > $O/interf.jsonl 2>> $O/err.txt
$I --engines 1 --ctas 2 --tag ldg >> $O/interf.jsonl 2>> $O/err.txt
tail -3 $O/err.txt
