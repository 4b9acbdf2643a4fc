#!/bin/bash
# NEXT-1 with real decode kernels: FlashInfer paged decode attention (the paper's 16 x 4K decode pass)
# and a whole Llama-8B decode step, beside the default load, one-CTA ring, LDG 2 CTAs, the copy-engine
# path and a contiguous memcpy.
O=gpurun_out/interf_real; mkdir -p $O
timeout 1500 python tools/interference.py --engines 2,1 --ctas 0,1,2 --proxies attn,decode_step,decode,decode4 \
    --reps 10 --memcpy 1 --tag real > $O/interf_real.jsonl 2> $O/interf_real.err; echo "interf rc=$?"
tail -3 $O/interf_real.err
