#!/bin/bash
# Round 2: offload pacing default (16 GB/s while ring loads run): bidir at defaults, concurrent tests, bench.
O=gpurun_out/r2_verify7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/bidir.py --config llama8b_32k --reps 3 > $O/bidir_8b.jsonl 2> $O/bidir.err
timeout 600 python tools/bidir.py --config llama70b_tp8 --reps 3 >> $O/bidir_70b.jsonl 2>> $O/bidir.err
timeout 900 python -m pytest tests/test_gpu_concurrent.py tests/test_gpu_stress.py -q -s --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
for f in $O/bidir_*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); print(' ', d.get('mode'), d.get('load_gbs'), d.get('offload_gbs'), d.get('overlap_gbs'))
"; done; grep -E "alone|passed|failed|FAILED" $O/pytest.log | tail -5; tail -1 $O/bench.err; python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['frac_of_link'], d['offload'], d.get('interference'))"
