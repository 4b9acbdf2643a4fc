#!/bin/bash
# The N>1 bench flow (torchrun, 2 ranks) on a one-GPU box in the shared-GPU test mode, final tree.
O=gpurun_out/n2check; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
STRATA_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_n2.json 2> $O/bench_n2.err; echo "n2 rc=$?"; cut -c1-300 $O/bench_n2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $O/ref_n2.json 2> $O/ref_n2.err; echo "ref n2 rc=$?"; wc -l $O/ref_n2.json
