#!/bin/bash
# Round 2: does an L2 prefetch of the host runs (cp.async.bulk.prefetch.L2) lift the SM zero-copy plateau?
O=gpurun_out/r2_prefetch; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for D in 0 4; do
  STRATA_RING_DEBUG=$D timeout 600 python tools/ring_sweep.py --configs llama8b_32k:1 --dirs load --ctas 1,2,4 --warps 8 --stage-kb 16 --inflight-kb 0,448 --reps 3 --tag dbg$D >> $O/sweep.jsonl 2>> $O/sweep.err
  STRATA_RING_DEBUG=$D timeout 600 python tools/ring_sweep.py --configs llama8b_32k:1 --dirs load --ctas 2 --warps 8 --stage-kb 16 --reps 3 --chunk-frag identity --frag identity --tag dbg${D}_contig >> $O/sweep.jsonl 2>> $O/sweep.err
done
python -c "
import json
for l in open('$O/sweep.jsonl'):
    d=json.loads(l)
    if d['kind']=='ring': print(d['tag'], d['ctas'], d['inflight_kb'], d['gbs'], d['frac_link'], d['parity'])
    else: print(d)
"; tail -3 $O/sweep.err
