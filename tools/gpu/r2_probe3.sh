#!/bin/bash
O=gpurun_out/r2_probe3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o tools/probe/libchase.so tools/probe/chase.cu >> $O/build.log 2>&1
timeout 600 python tools/interference_latency.py > $O/latency.jsonl 2> $O/latency.err
timeout 1500 python tools/ring_sweep.py --configs qwen14b_batch8:1 --dirs offload --ctas 0,2,3,4 --gather-warps 8 --stage-kb 16,32 --reps 2 > $O/sweep_qwen_off.jsonl 2> $O/sweep_qwen.err
cat $O/latency.jsonl; tail -3 $O/latency.err; cat $O/sweep_qwen_off.jsonl | cut -c1-330; tail -3 $O/sweep_qwen.err
