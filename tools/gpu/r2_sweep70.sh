#!/bin/bash
# Round 2: ring geometry vs bytes in flight on the small-row (70B TP=8, 256 B) and MLA (1152 B) configs.
O=gpurun_out/r2_sweep70; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/ring_sweep.py --configs llama70b_tp8:1,deepseek_v3_mla:1 --dirs load --ctas 0,2,3,4,8 --warps 8 --stage-kb 8,16,32 --inflight-kb 0,256,320,448 --reps 3 > $O/sweep_load.jsonl 2> $O/sweep.err
timeout 600 python tools/ring_sweep.py --configs llama70b_tp8:1,deepseek_v3_mla:1 --dirs offload --ctas 0,2,4 --gather-warps 8 --stage-kb 8,16,32 --inflight-kb 0,256,448 --reps 3 > $O/sweep_off.jsonl 2>> $O/sweep.err
python - <<'PY'
import json
for f in ("sweep_load","sweep_off"):
    rows=[json.loads(l) for l in open(f"gpurun_out/r2_sweep70/{f}.jsonl") if '"ring"' in l]
    for cfg in ("llama70b_tp8","deepseek_v3_mla"):
        rs=sorted([r for r in rows if r["config"]==cfg], key=lambda r: -r["gbs"])
        print(f, cfg, "best:")
        for r in rs[:6]: print("  ", r["ctas"], r["stage_kb"], r["inflight_kb"], r["gbs"], r["frac_link"], r["parity"])
        print("   default:", [ (r["stage_kb"], r["gbs"]) for r in rs if r["ctas"]==0 and r["inflight_kb"]==0])
PY
