#!/bin/bash
O=gpurun_out/r2_probe4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o tools/probe/libchase.so tools/probe/chase.cu >> $O/build.log 2>&1
timeout 600 python tools/interference_latency.py > $O/latency.jsonl 2> $O/latency.err
timeout 900 python tools/ring_sweep.py --configs llama8b_32k:1,llama8b_32k:16 --dirs offload --ctas 2,3,4 --gather-warps 8 --stage-kb 16 --reps 3 > $O/sweep_off.jsonl 2> $O/sweep.err
python -c "
import json
for l in open('$O/latency.jsonl'):
    d=json.loads(l); print(d['beside'], {k:v for k,v in d.items() if k.endswith('median')})
"; tail -3 $O/latency.err; cat $O/sweep_off.jsonl | cut -c1-330
