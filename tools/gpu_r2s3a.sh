#!/bin/bash
# LDG loads in the running-load counter + NEXT-1 attention-decode operating points
O=gpurun_out/s3a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests/test_gpu_concurrent.py tests/test_gpu_interference.py tests/test_gpu_fused.py tests/test_gpu_graph.py tests/test_gpu_parity.py -m gpu -q -x -s -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
grep -E "slowdown|beside the offload" $O/pytest.log | head -40
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['frac_of_link'], d['interference'])"
