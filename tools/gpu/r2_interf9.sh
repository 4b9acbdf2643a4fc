#!/bin/bash
# Round 2: interference of the offload (write-back) at its default quota (4 CTAs) and at 1 / 2 CTAs.
O=gpurun_out/r2_interf9; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python tools/interference.py --offload 1 --proxies prefill,decode4,decode32 --engines 2 --ctas 0,1,2 --reps 10 --tag offload > $O/interf.jsonl 2> $O/interf.err
python -c "
import json
for l in open('$O/interf.jsonl'):
    d=json.loads(l)
    if d['kind']=='corun': print(d['tag'], d['ctas'], d['proxy'], d['slowdown'], d['io_alone_gbs'], d['io_corun_gbs_upper'])
"; tail -3 $O/interf.err
