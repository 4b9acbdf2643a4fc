#!/bin/bash
# compute-sanitizer over small parity cases of every engine: memcheck (out-of-bounds / misaligned
# accesses, incl. host-mapped memory), racecheck and synccheck (shared-memory rings of the TMA
# engines, mbarrier use), initcheck.
mkdir -p gpurun_out/sanitize
S=gpurun_out/sanitize
K="tiny_load_offload or special_float or fuzz_load and (0 or 1 or 2 or 3)"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
     python -m pytest tests/test_gpu_parity.py -q -x -k "tiny_load_offload or special_float" > $S/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $S/$tool.log | tail -3
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 99 --target-processes all \
   python -m pytest tests/test_gpu_mla.py tests/test_gpu_heads.py -q -x -k "small or latent_small" > $S/memcheck_variants.log 2>&1
echo "memcheck variants rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $S/memcheck_variants.log | tail -3
