#!/bin/bash
mkdir -p gpurun_out
for n in 1 4; do STRATA_COPY_STREAMS=$n python tools/submit_probe.py; done 2>&1 | tee gpurun_out/submit_probe.jsonl
