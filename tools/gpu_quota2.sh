#!/bin/bash
O=gpurun_out/quota2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests/test_gpu_quota.py tests/test_gpu_fused.py tests/test_gpu_graph.py tests/test_gpu_concurrent.py tests/test_gpu_parity.py -m gpu -q -x -s -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log; grep -E "uncapped" $O/pytest.log
python bench.py --no-extras > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cut -c1-200 $O/bench.json
