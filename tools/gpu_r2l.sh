#!/bin/bash
# Round-2 pass L: dK/dV softmax warps split by block parity (variant dkvpar): parity, then A/B.
O=gpurun_out
mkdir -p $O
S=$O/r2l_summary.txt
: > $S
timeout 600 python tools/attn_variant_check.py dkvpar > $O/r2l_check_dkvpar.txt 2>&1; echo "check dkvpar rc=$?" >> $S
tail -1 $O/r2l_check_dkvpar.txt >> $S
for rep in 1 2 3; do
  for v in "" "--variant dkvpar"; do
    timeout 300 python tools/attn_clock.py $v bwd 6674 26094 32 80 >> $O/r2l_attn_ab.txt 2>&1
    timeout 300 python tools/attn_clock.py $v bwd 10170 0 32 80 >> $O/r2l_attn_ab.txt 2>&1
  done
done; echo "ab rc=$?" >> $S
cat $O/r2l_attn_ab.txt >> $S
KERNELS="attn_bwd_dkv" timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dkv -c 1 -o $O/r2l_dkvpar -f \
   python tools/attn_once.py --variant dkvpar > $O/r2l_ncu.log 2>&1; echo "ncu rc=$?" >> $S
cat $S
