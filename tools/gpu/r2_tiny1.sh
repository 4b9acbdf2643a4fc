#!/bin/bash
# Round 2: small-operation latency (tiny config): ring geometry sweep + bench + ncu of the tiny kernel.
O=gpurun_out/r2_tiny1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python bench.py --config tiny --no-cpu-baseline > $O/bench_tiny.json 2> $O/bench_tiny.err
timeout 600 python tools/ring_sweep.py --configs tiny:16 --dirs load,offload --ctas 0,8,16,32,64 --warps 2,4 --gather-warps 2,4 --stage-kb 4,8,16 --inflight-kb 0,4096 --reps 30 > $O/sweep_tiny.jsonl 2> $O/sweep.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_tiny.csv python bench.py --config tiny --steps 5 --warmup 3 --no-extras --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ring_load -s 3 -c 1 -o $O/ncu_tiny python tools/prof_one.py --config tiny --P 16 --layers 2 --engine 0 --reps 5 > $O/ncu_full.log 2>&1
timeout 900 python -m pytest tests/test_gpu_heads.py tests/test_gpu_parity.py -x -q --timeout 600 -k "shared_tier_outlives or tiny or small or fuzz" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
head -c 600 $O/bench_tiny.json; echo; python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/r2_tiny1/sweep_tiny.jsonl") if '"ring"' in l]
for d in ("load","offload"):
    rs=sorted([r for r in rows if r["dir"]==d], key=lambda r: r["us"])[:8]
    for r in rs: print(d, r["ctas"], r["warps"], r["stage_kb"], r["inflight_kb"], r["us"], r["gbs"], r["parity"])
PY
tail -3 $O/pytest.log
