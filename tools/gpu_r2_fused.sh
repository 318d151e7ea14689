#!/bin/bash
# Fused attention backward bring-up: L2 reduce microbenchmark, kernel parity (fused vs split vs
# fp64), hd-128 long-shape parity, the LLaMA loss sanity test, and fused-vs-split timing.
mkdir -p gpurun_out
./tools/micro/red_bench > gpurun_out/r2_red_bench.txt 2>&1; echo "red_bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "attention" > gpurun_out/r2_fused_kernels.log 2>&1
echo "kernel tests rc=$?"
timeout 600 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -k "cfg3_shape or memorisation or cfg2_shape" > gpurun_out/r2_fused_engine.log 2>&1
echo "engine tests rc=$?"
for shape in "10170 0 32 80" "6674 26094 32 80" "8496 10170 32 80"; do
  for w in bwd bwd-split; do timeout 300 python tools/attn_clock.py $w $shape; done
done > gpurun_out/r2_fused_clock.txt 2>&1
echo "clock rc=$?"
