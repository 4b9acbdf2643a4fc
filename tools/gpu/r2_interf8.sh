#!/bin/bash
# Round 2: copy-engine path (DMA engine, one cudaMemcpyAsync per chunk-layer run) interference vs its
# rate, set by the number of copy streams; the ring at the same rates for comparison.
O=gpurun_out/r2_interf8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for CS in 1 2 3 4 8; do
  STRATA_COPY_STREAMS=$CS timeout 900 python tools/interference.py --proxies decode4,decode32,prefill --engines 4 --ctas 0 --reps 10 --tag dma_cs$CS >> $O/interf.jsonl 2>> $O/interf.err
done
python -c "
import json
for l in open('$O/interf.jsonl'):
    d=json.loads(l)
    if d['kind']=='corun': print(d['tag'], d['proxy'], d['slowdown'], d['io_alone_gbs'], d['io_corun_gbs_upper'])
"; tail -3 $O/interf.err
