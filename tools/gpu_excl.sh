#!/bin/bash
# A/B: does issuing the ring's host reads as one cp.async.bulk per 2 KiB row (or smaller pieces)
# instead of one per 16 KiB piece interfere less with decode at the same load rate?
O=gpurun_out/excl; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/interference.py --proxies attn,decode,decode_step --reps 10 --tag excl --env-sets \
"STRATA_RING_INFLIGHT_KB=224,STRATA_RING_EXCLUSIVE=1,STRATA_RING_EXCLUSIVE=1;STRATA_RING_WARPS=15" \
  > $O/excl.jsonl 2> $O/excl.err; echo "rc=$?"; tail -2 $O/excl.err
python - <<'PY'
import json
for l in open("gpurun_out/excl/excl.jsonl"):
    d = json.loads(l)
    if d.get("kind") == "corun":
        print(d["env"], d["proxy"], d["slowdown"], d["io_alone_gbs"], d["io_corun_gbs_upper"])
PY
