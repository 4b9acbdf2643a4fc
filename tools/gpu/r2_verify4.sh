#!/bin/bash
# Round 2: after the planning changes (short-row in-flight, W/S, small-op re-plan, narrow 4-byte ->
# LDG, offload quota for short rows): bench with the interference extra, narrow probe, whole GPU suite.
O=gpurun_out/r2_verify4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --config deepseek_v3_mla --no-cpu-baseline > $O/bench_mla.json 2> $O/bench_mla.err
timeout 600 python tools/narrow_probe.py > $O/narrow.jsonl 2> $O/narrow.err
timeout 3000 python -m pytest tests -m gpu -q --timeout 1200 > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
tail -2 $O/smoke.log; tail -2 $O/bench.err; python -c "
import json
for f in ('bench','bench_mla'):
    d=json.load(open('$O/'+f+'.json'))
    print(f, d['value'], d['frac_of_link'], d['offload'], d.get('interference'), d['host_submit_ms_per_step'], d['gpu_launches'])
"; cat $O/narrow.jsonl | cut -c1-200; grep -E "slowdown|passed|failed|FAILED|Error" $O/pytest_all.log | tail -20
