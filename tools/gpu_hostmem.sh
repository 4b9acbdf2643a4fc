mkdir -p gpurun_out
for fl in 0 1 16; do for cf in perm identity; do
python tools/sweep.py --pages 1 --ctas 1,2,4 --engines 1,3 --baselines 0 --flags $fl --chunk-frag $cf > gpurun_out/sweep_host_f${fl}_${cf}.jsonl 2>&1
done; done
grep -h AnonHuge /proc/meminfo
python tools/interference.py > gpurun_out/interference.jsonl 2>&1; echo interf rc=$?
