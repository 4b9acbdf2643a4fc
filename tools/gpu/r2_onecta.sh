#!/bin/bash
# Round 2: what bounds ONE ring CTA? page-table locality (device TLB), pool size, scatter warps.
O=gpurun_out/r2_onecta; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
S="timeout 600 python tools/ring_sweep.py --configs llama8b_32k:1 --dirs load --ctas 1 --reps 3"
$S --warps 8,12,16 --stage-kb 8,16 --inflight-kb 224,448 --tag perm > $O/sweep.jsonl 2> $O/sweep.err
$S --warps 8 --stage-kb 16 --inflight-kb 224,448 --frag identity --tag pages_identity >> $O/sweep.jsonl 2>> $O/sweep.err
$S --warps 8 --stage-kb 16 --inflight-kb 224,448 --chunk-frag identity --tag chunks_identity >> $O/sweep.jsonl 2>> $O/sweep.err
$S --warps 8 --stage-kb 16 --inflight-kb 224,448 --layers 4 --tag L4 >> $O/sweep.jsonl 2>> $O/sweep.err
python -c "
import json
for l in open('$O/sweep.jsonl'):
    d=json.loads(l)
    if d['kind']=='ring': print(d['tag'], d['L'], d['warps'], d['stage_kb'], d['inflight_kb'], d['gbs'], d['parity'])
"; tail -3 $O/sweep.err
