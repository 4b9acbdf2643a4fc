#!/bin/bash
# Round 2: the copy-engine path with G layers per copy run (fewer, larger copies: 256 KiB x G) —
# its rate and interference.
O=gpurun_out/r2_interf10; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/interference.py --proxies prefill,decode4,decode32 --engines 4 --ctas 0 --groups 2,4,8,32 --reps 10 --tag dma_groups > $O/interf.jsonl 2> $O/interf.err
timeout 300 python tools/submit_probe.py --engines 4 > $O/submit.jsonl 2>> $O/interf.err
python -c "
import json
for l in open('$O/interf.jsonl'):
    d=json.loads(l)
    if d['kind']=='corun': print(d['tag'], d['layer_group'], d['proxy'], d['slowdown'], d['io_alone_gbs'], d['io_corun_gbs_upper'])
"; cut -c1-300 $O/submit.jsonl; tail -3 $O/interf.err
