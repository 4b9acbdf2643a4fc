#!/bin/bash
# Round 2: device-memory latency and launch latency beside the load (interference mechanism);
# Qwen-14B batch quota sweep (its offload sits at 0.88 of the link).
O=gpurun_out/r2_probe2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o tools/probe/libchase.so tools/probe/chase.cu >> $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_gpu_concurrent.py -q --timeout 300 > $O/pytest_graph.log 2>&1; echo "rc=$?" >> $O/pytest_graph.log
timeout 600 python tools/interference_latency.py > $O/latency.jsonl 2> $O/latency.err
timeout 1500 python tools/ring_sweep.py --configs qwen14b_batch8:1 --dirs load,offload --ctas 0,2,3,4 --warps 8 --gather-warps 8 --stage-kb 16 --reps 2 > $O/sweep_qwen.jsonl 2> $O/sweep_qwen.err
tail -3 $O/pytest_graph.log; cat $O/latency.jsonl; tail -3 $O/latency.err; cat $O/sweep_qwen.jsonl | cut -c1-330; tail -3 $O/sweep_qwen.err
