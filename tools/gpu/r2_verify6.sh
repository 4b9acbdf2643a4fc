#!/bin/bash
# Round 2: offload default 4 CTAs, bench with the page-size sweep + per-page baseline at P=32,
# bidirectional load+offload on the ring, whole GPU suite.
O=gpurun_out/r2_verify6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python tools/bidir.py > $O/bidir.jsonl 2> $O/bidir.err
timeout 600 python tools/bidir.py --config llama8b_32k >> $O/bidir.jsonl 2>> $O/bidir.err
timeout 3000 python -m pytest tests -m gpu -q --timeout 1200 > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
tail -2 $O/smoke.log; tail -2 $O/bench.err; python -c "
import json
d=json.load(open('$O/bench.json'))
print(d['value'], d['frac_of_link'], d['offload'], d['page_size_sweep'], d.get('per_page_memcpy_baseline_P32'), d.get('interference'), d['roofline']['traffic'])
"; cat $O/bidir.jsonl | cut -c1-400; grep -E "slowdown|passed|failed|FAILED" $O/pytest_all.log | tail -12
