#!/bin/bash
# Two ranks (test mode: both on cuda:0, gloo) sharing ONE host tier file in /dev/shm, each moving its head.
mkdir -p gpurun_out
df -h /dev/shm | tee gpurun_out/devshm.txt; free -g | tee -a gpurun_out/devshm.txt
STRATA_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29533 bench.py --gpus 2 --config llama70b_tp8_shared --steps 5 --warmup 3 \
   > gpurun_out/bench_shared_2ranks_testmode.json 2> gpurun_out/bench_shared_2ranks.err; echo "rc=$?"
cut -c1-300 gpurun_out/bench_shared_2ranks_testmode.json; tail -5 gpurun_out/bench_shared_2ranks.err
ls /dev/shm | head
