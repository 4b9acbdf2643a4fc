#!/bin/bash
# Round 2: short-row in-flight default (320 KiB), W/S planning fix, small-op re-plan, graph-replay
# bench extra: every bench config + the fast GPU suite.
O=gpurun_out/r2_verify3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in llama8b_32k tiny llama70b_tp8 deepseek_v3_mla llama70b_tp8_shared; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python tools/ring_sweep.py --configs llama70b_tp8:1,deepseek_v3_mla:1,llama8b_32k:1 --dirs load,offload --ctas 0 --warps 8 --gather-warps 8 --stage-kb 16 --reps 5 > $O/sweep_default.jsonl 2> $O/sweep.err
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q --timeout 300 > $O/pytest_fast.log 2>&1; echo "pytest rc=$?" >> $O/pytest_fast.log
for c in llama8b_32k tiny llama70b_tp8 deepseek_v3_mla llama70b_tp8_shared; do python -c "
import json
d=json.load(open('$O/bench_$c.json'))
print('$c', d['value'], d['ms_per_step'], d['frac_of_link'], d['engine'], 'off', d.get('offload',{}).get('value'), d.get('offload',{}).get('frac_of_d2h_link'), 'p16', d.get('page_size_16',{}).get('value'), d.get('page_size_16',{}).get('frac_of_link'), d.get('other_engines_gbs'), d.get('graph_replay'), d['host_submit_ms_per_step'])
" || tail -3 $O/bench_$c.err; done
cat $O/sweep_default.jsonl | cut -c1-330; tail -3 $O/pytest_fast.log
