#!/bin/bash
# NEXT-4 replay (fixed host seeding, pipelined scheduler) + NEXT-2 bubble filling.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for o in max min random; do
  timeout 900 python tools/ctl_bench.py --order $o > gpurun_out/ctl_bench_$o.jsonl 2> gpurun_out/ctl_bench_$o.err
done
timeout 600 python tools/ctl_bench.py --order max --page-size 16 > gpurun_out/ctl_bench_p16.jsonl 2> gpurun_out/ctl_bench_p16.err
timeout 900 python tools/bubble_fill.py > gpurun_out/bubble_fill.jsonl 2> gpurun_out/bubble_fill.err
cat gpurun_out/ctl_bench_*.jsonl gpurun_out/bubble_fill.jsonl
tail -5 gpurun_out/bubble_fill.err
