#!/bin/bash
# Round 2: first bench.py run of the zero-copy default; 1-CTA fused vs per-layer; interference sweep;
# NEXT-1 / NEXT-2 tests; bench N=2 flow in shared-GPU test mode.
O=gpurun_out/r2_eval1; mkdir -p $O
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/clocks_start.csv
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 300 python bench.py --config tiny --no-cpu-baseline > $O/bench_tiny.json 2> $O/bench_tiny.err
timeout 600 python bench.py --config llama70b_tp8 --no-cpu-baseline > $O/bench_70b.json 2> $O/bench_70b.err
S="timeout 300 python tools/ring_sweep.py --configs llama8b_32k:1 --ctas 1,2 --warps 8 --gather-warps 4 --stage-kb 32"
$S --layers 4 --tag fused_L4 > $O/fused_vs_layer.jsonl 2>> $O/sweep.err
$S --tag fused_L32 >> $O/fused_vs_layer.jsonl 2>> $O/sweep.err
STRATA_LDG_FUSED=0 $S --tag perlayer_L32 >> $O/fused_vs_layer.jsonl 2>> $O/sweep.err
timeout 900 python tools/interference.py --engines 2 --ctas 1,2,4 --ring-smem 0,96 --reps 20 > $O/interference_ring.jsonl 2> $O/interference.err
timeout 600 python tools/interference.py --engines 1,4 --ctas 2 --reps 20 >> $O/interference_ring.jsonl 2>> $O/interference.err
STRATA_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-extras > $O/bench_n2_share.json 2> $O/bench_n2_share.err; echo "n2 rc=$?" >> $O/bench_n2_share.err
timeout 1500 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_interference.py -x -q -s --timeout 900 > $O/pytest_next.log 2>&1; echo "pytest rc=$?" >> $O/pytest_next.log
tail -2 $O/bench.err; cat $O/bench.json | head -c 1500; echo; tail -3 $O/interference.err; tail -15 $O/pytest_next.log; tail -3 $O/bench_n2_share.err
