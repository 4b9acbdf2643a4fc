#!/bin/bash
# Round 2: offload paced to a share of the link while ring loads run (STRATA_OFFLOAD_SHARE_GBS)
O=gpurun_out/r2_bidir4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for S in 0 8 16 24 32; do
  STRATA_OFFLOAD_SHARE_GBS=$S timeout 600 python tools/bidir.py --config llama8b_32k --reps 3 --grid 0:0:0:0 > $O/bidir_8b_s$S.jsonl 2>> $O/bidir.err
done
STRATA_OFFLOAD_SHARE_GBS=16 timeout 600 python tools/bidir.py --config llama70b_tp8 --reps 3 --grid 0:0:0:0 > $O/bidir_70b_s16.jsonl 2>> $O/bidir.err
for f in $O/bidir_*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); print(' ', d.get('mode'), d.get('load_gbs'), d.get('offload_gbs'), d.get('load_ms'), d.get('offload_ms'), d.get('overlap_gbs'))
"; done; tail -3 $O/bidir.err
