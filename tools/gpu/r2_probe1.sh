#!/bin/bash
# Round 2: host cost of back-to-back calls (does strata_load block the caller?), the other bench
# configs on the ring default, narrow rows.
O=gpurun_out/r2_probe1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/submit_probe.py --engines 2,1,4 > $O/submit.jsonl 2> $O/submit.err
STRATA_LDG_FUSED=0 timeout 300 python tools/submit_probe.py --engines 2,1 >> $O/submit.jsonl 2>> $O/submit.err
timeout 300 python tools/submit_probe.py --config tiny --engines 2,1 --n 20 >> $O/submit.jsonl 2>> $O/submit.err
for c in tiny llama70b_tp8 deepseek_v3_mla; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config qwen14b_batch8 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_qwen14b_batch8.json 2> $O/bench_qwen14b_batch8.err
timeout 600 python tools/narrow_probe.py > $O/narrow.jsonl 2> $O/narrow.err
cat $O/submit.jsonl | cut -c1-400; for c in tiny llama70b_tp8 deepseek_v3_mla qwen14b_batch8; do head -c 700 $O/bench_$c.json; echo; tail -2 $O/bench_$c.err; done; cat $O/narrow.jsonl | cut -c1-300
