#!/bin/bash
# Round 2: offload yields to running ring loads (STRATA_OFFLOAD_YIELD = K: at most K+1 incomplete host
# stores per offload CTA while a load runs): solo rates unchanged? overlap rates?
O=gpurun_out/r2_bidir3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for K in -1 0 1 2; do
  STRATA_OFFLOAD_YIELD=$K timeout 600 python tools/bidir.py --config llama8b_32k --reps 3 --grid 0:0:0:0 > $O/bidir_8b_k$K.jsonl 2>> $O/bidir.err
done
STRATA_OFFLOAD_YIELD=1 timeout 600 python tools/bidir.py --config llama70b_tp8 --reps 3 --grid 0:0:0:0 > $O/bidir_70b_k1.jsonl 2>> $O/bidir.err
STRATA_OFFLOAD_YIELD=0 timeout 600 python tools/bidir.py --config llama70b_tp8 --reps 3 --grid 0:0:0:0 > $O/bidir_70b_k0.jsonl 2>> $O/bidir.err
for f in $O/bidir_*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); print(' ', d.get('mode'), d.get('load_gbs'), d.get('offload_gbs'), d.get('overlap_gbs'))
"; done; tail -3 $O/bidir.err
