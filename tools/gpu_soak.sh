#!/bin/bash
# soak: the stress suite over 6 fresh seed bases (9000 cases)
for b in 100000 200000 300000 400000 500000 600000; do
  STRESS_SEED_BASE=$b timeout 900 python -m pytest tests/test_gpu_stress.py -q -x -p no:cacheprovider 2>&1 | tail -1
done
