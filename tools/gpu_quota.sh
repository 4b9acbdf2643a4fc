#!/bin/bash
# Decode-aware quota (strata_set_load_quota): parity / cap tests, then the co-run with and without the
# quota bracketing the decode-side proxies (INTERF=1).
O=gpurun_out/quota; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_quota.py tests/test_gpu_fused.py tests/test_gpu_concurrent.py -m gpu -q -x -s -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log; grep -E "uncapped|beside the offload" $O/pytest.log
if [ "${INTERF:-1}" = 1 ]; then
  timeout 1500 python tools/interference.py --engines 1 --ctas 0 --proxies attn,decode_step,decode,prefill --quota-bracket 1 \
      --reps 10 --tag quota > $O/quota.jsonl 2> $O/quota.err; echo "interf rc=$?"; tail -2 $O/quota.err
fi
