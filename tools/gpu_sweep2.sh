#!/bin/bash
mkdir -p gpurun_out
python tools/sweep.py --config llama8b_32k --pages 1,16,64 --ctas 1,2,4,8,32 --engines 1,4 --baselines 0 > gpurun_out/sw2_llama.jsonl 2>&1; echo "llama rc=$?"
python tools/sweep.py --config llama70b_tp8 --pages 1,16 --ctas 1,2,4,8,32 --engines 1,4 --baselines 1 > gpurun_out/sw2_70b.jsonl 2>&1; echo "70b rc=$?"
python tools/sweep.py --config tiny --pages 16 --ctas 0,1,2,4,8 --engines 0,1,2,4 --baselines 1 > gpurun_out/sw2_tiny.jsonl 2>&1; echo "tiny rc=$?"
python tools/sweep.py --config qwen14b_batch8 --pages 1 --ctas 2,8 --engines 1,4 --baselines 0 > gpurun_out/sw2_qwen.jsonl 2>&1; echo "qwen rc=$?"
python tools/interference.py --engines 1,4 --ctas 1,2,4,8 > gpurun_out/interference2.jsonl 2>&1; echo "interf rc=$?"
python tools/bidir.py > gpurun_out/bidir.jsonl 2>&1; echo "bidir rc=$?"
