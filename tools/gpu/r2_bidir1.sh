#!/bin/bash
# Round 2: load + offload at once — operating points (load starved by the offload's posted writes?)
O=gpurun_out/r2_bidir1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
G="0:0:0:0,0:448:0:0,0:896:0:0,0:0:1:0,0:0:2:0,0:0:1:64,0:0:2:96,0:0:4:96,0:448:1:0,0:448:2:96,4:448:1:64,0:0:1:32"
timeout 900 python tools/bidir.py --config llama8b_32k --reps 3 --grid $G > $O/bidir_8b.jsonl 2> $O/bidir.err
timeout 900 python tools/bidir.py --config llama70b_tp8 --reps 3 --grid 0:0:0:0,0:448:1:0,0:0:1:64,0:448:2:96 > $O/bidir_70b.jsonl 2>> $O/bidir.err
python - <<'PY'
import json
for f in ("bidir_8b","bidir_70b"):
    for l in open(f"gpurun_out/r2_bidir1/{f}.jsonl"):
        d=json.loads(l)
        print(f, d.get("mode"), d.get("load_ctas"), d.get("load_inflight_kib"), d.get("offload_ctas"), d.get("offload_inflight_kib"), d.get("load_gbs"), d.get("offload_gbs"), d.get("overlap_gbs"))
PY
tail -3 $O/bidir.err
