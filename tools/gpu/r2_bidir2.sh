#!/bin/bash
# Round 2: load + offload frontier: offload CTAs x bytes in flight (solo and beside a load)
O=gpurun_out/r2_bidir2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
G="0:0:4:64,0:0:4:128,0:0:4:160,0:0:4:192,0:320:4:128,0:320:4:160,0:0:2:128,0:0:8:128,0:0:8:192"
timeout 900 python tools/bidir.py --config llama8b_32k --reps 3 --grid $G > $O/bidir_8b.jsonl 2> $O/bidir.err
timeout 900 python tools/ring_sweep.py --configs llama8b_32k:1,llama70b_tp8:1 --dirs offload --ctas 2,4,8 --gather-warps 8 --stage-kb 16 --inflight-kb 64,128,160,192,0 --reps 3 > $O/sweep_off.jsonl 2> $O/sweep.err
python - <<'PY'
import json
for l in open("gpurun_out/r2_bidir2/bidir_8b.jsonl"):
    d=json.loads(l)
    print(d.get("mode"), d.get("load_ctas"), d.get("load_inflight_kib"), d.get("offload_ctas"), d.get("offload_inflight_kib"), d.get("load_gbs"), d.get("offload_gbs"), d.get("overlap_gbs"))
for l in open("gpurun_out/r2_bidir2/sweep_off.jsonl"):
    d=json.loads(l)
    if d["kind"]=="ring": print(d["config"], d["ctas"], d["inflight_kb"], d["gbs"], d["frac_link"])
PY
tail -3 $O/bidir.err
