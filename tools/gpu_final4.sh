#!/bin/bash
# Final verification of the round with the LDG default for large loads: smoke, every GPU test, the
# default bench (+ reference arm), the other bench configs, the ncu launch list, and one ncu --set full
# capture of the bench's dominant kernel (ldg_fused_kernel, one 32-layer launch).
O=gpurun_out/final4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cut -c1-160 $O/bench.json
for c in qwen14b_batch8 llama70b_tp8 deepseek_v3_mla; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; echo "bench $c rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ldg_fused_kernel -c 1 -o $O/ncu_ldg_fused_32L \
    python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/ncu_ldg_fused_32L.ncu-rep --page details --csv > $O/ncu_ldg_fused_32L.details.csv 2>/dev/null
ncu -i $O/ncu_ldg_fused_32L.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active > $O/ncu_ldg_fused_32L.raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu list rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>> $O/bench.err; cut -c1-120 $O/bench_reference.json
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_all.log
