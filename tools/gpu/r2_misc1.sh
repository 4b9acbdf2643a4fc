#!/bin/bash
# Round 2: bench N=2 flow in shared-GPU test mode (new extras), copy-engine path interference at its
# current rate vs the ring at a similar rate.
O=gpurun_out/r2_misc1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
STRATA_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_n2_share.json 2> $O/bench_n2_share.err; echo "n2 rc=$?" >> $O/bench_n2_share.err
timeout 900 python tools/interference.py --proxies decode4,decode32 --engines 4 --ctas 0 --reps 10 --tag dma_percopy > $O/interf_dma.jsonl 2> $O/interf.err
timeout 900 python tools/interference.py --proxies decode4,decode32 --ring-configs 1:16:112:7:0:0,2:16:80:4:0:0 --reps 10 --tag ring_low > $O/interf_ring_low.jsonl 2>> $O/interf.err
tail -2 $O/bench_n2_share.err; python -c "
import json; d=json.load(open('$O/bench_n2_share.json')); print({k: d.get(k) for k in ('value','n_gpus','per_rank','page_size_sweep','shared_gpu_test_mode')})"
for f in $O/interf_*.jsonl; do python -c "
import json
for l in open('$f'):
    d=json.loads(l)
    if d['kind']=='corun': print(d['tag'], d['engine'], d['ctas'], d['proxy'], d['slowdown'], d['io_alone_gbs'], d['io_corun_gbs_upper'])
"; done; tail -3 $O/interf.err
