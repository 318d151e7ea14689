#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "attention" > gpurun_out/r2_fused_kernels.log 2>&1
echo "kernel tests rc=$?"
for shape in "6674 26094 32 80" "10170 0 32 80"; do
  for w in bwd bwd-split; do timeout 300 python tools/attn_clock.py $w $shape; done
done > gpurun_out/r2_fused_clock.txt 2>&1
python tools/attn_once.py --variant prof 6674 26094 32 80 > gpurun_out/r2_trace.txt 2>&1
