#!/bin/bash
# the layer-wise prefill overlap test, repeated (flake check after preallocating the outputs)
O=gpurun_out/prefill_loop; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2 3 4 5 6; do timeout 600 python -m pytest tests/test_gpu_prefill.py -m gpu -q -p no:cacheprovider -s > $O/prefill_$i.log 2>&1; echo "run $i rc=$? $(tail -1 $O/prefill_$i.log)"; done
