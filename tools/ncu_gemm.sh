#!/bin/bash
# ncu --set full of the tcgen05 GEMM in its three engine roles at cfg-2 shapes (one launch each, after 3 warm-ups)
O=gpurun_out
mkdir -p $O
for c in mlp_down_fwd qkv_dgrad mlp_up_wgrad o_wgrad; do
  SP_GEMM_ONLY=$c SP_GEMM_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc \
    --launch-skip 3 -c 1 -o $O/r2y_gemm_$c -f python tools/gemm_tail_ab.py > $O/r2y_ncu_gemm_$c.log 2>&1
  echo "ncu $c rc=$?"
done
python tools/ncu_summary.py $O/r2y_gemm_*.ncu-rep > $O/r2y_ncu_gemm_summary.txt 2>&1
cat $O/r2y_ncu_gemm_summary.txt | head -80
