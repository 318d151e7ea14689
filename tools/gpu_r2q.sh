#!/bin/bash
# Round-2 pass Q: the P = 8 points of the in-process cfg-5 slice at 16K (LLaMA-7B width).
O=gpurun_out
mkdir -p $O
timeout 1500 python tools/pipeline_inproc.py --model llama-7b --layers-per-stage 1 \
   --sweep 16384:1:8,16384:2:8,16384:4:8,16384:8:8,16384:16:8 --dump-after 1400 > $O/r2q_cfg5_p8.txt 2>&1; echo "rc=$?"
grep -c '^{' $O/r2q_cfg5_p8.txt
