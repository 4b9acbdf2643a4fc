#!/bin/bash
mkdir -p gpurun_out/strided
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dma or tiny" > gpurun_out/strided/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/strided/pytest.log
for s in 1 0; do
  STRATA_DMA_STRIDED=$s python bench.py --no-cpu-baseline --chunk-frag identity > gpurun_out/strided/bench_ident_s$s.json 2>> gpurun_out/strided/err
  python -c "import json;d=json.load(open('gpurun_out/strided/bench_ident_s$s.json'));print('identity strided=$s',d['value'],d['step_stats_rank0']['median_ms'],d['host_submit_ms_per_step'])"
done
python bench.py --no-cpu-baseline > gpurun_out/strided/bench_perm.json 2>> gpurun_out/strided/err
python -c "import json;d=json.load(open('gpurun_out/strided/bench_perm.json'));print('perm',d['value'],d['step_stats_rank0']['median_ms'],d['host_submit_ms_per_step'])"
python bench.py --no-cpu-baseline --config llama70b_tp8 --chunk-frag identity --steps 8 > gpurun_out/strided/bench70_ident.json 2>> gpurun_out/strided/err
python -c "import json;d=json.load(open('gpurun_out/strided/bench70_ident.json'));print('70b ident',d['value'],d['host_submit_ms_per_step'])"
for s in 1 0; do STRATA_DMA_STRIDED=$s python tools/submit_probe.py identity > gpurun_out/strided/submit_s$s.jsonl 2>&1; head -1 gpurun_out/strided/submit_s$s.jsonl; done
