#!/bin/bash
# Last check of the final tree: smoke + the whole GPU suite exactly as the driver runs it.
O=gpurun_out/final8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2700 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_all.log
