#!/bin/bash
# The N=8 torchrun flow of bench.py end to end in test mode (all ranks on cuda:0, gloo for the
# barrier / max reduction): orchestration check only — eight ranks share one GPU and one link.
mkdir -p gpurun_out
STRATA_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
   --master-port 29544 bench.py --gpus 8 --steps 4 --warmup 3 > gpurun_out/bench_8ranks_testmode.json 2> gpurun_out/bench_8ranks.err; echo "rc=$?"
cut -c1-400 gpurun_out/bench_8ranks_testmode.json; grep -iE "error|Traceback" gpurun_out/bench_8ranks.err | head -5
