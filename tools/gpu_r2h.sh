#!/bin/bash
# Round-2 pass H: per-tile MMA-issuing warps in the forward (variant tilew): parity, then A/B.
O=gpurun_out
mkdir -p $O
S=$O/r2h_summary.txt
: > $S
timeout 600 python tools/attn_variant_check.py tilew > $O/r2h_check_tilew.txt 2>&1; echo "check tilew rc=$?" >> $S
tail -1 $O/r2h_check_tilew.txt >> $S
for rep in 1 2 3; do
  for v in "" "--variant tilew"; do
    timeout 300 python tools/attn_clock.py $v fwd 6674 26094 32 80 >> $O/r2h_attn_ab.txt 2>&1
    timeout 300 python tools/attn_clock.py $v fwd 10170 0 32 80 >> $O/r2h_attn_ab.txt 2>&1
    timeout 300 python tools/attn_clock.py $v fwd 6229 59307 32 128 >> $O/r2h_attn_ab.txt 2>&1
  done
done; echo "ab rc=$?" >> $S
cat $O/r2h_attn_ab.txt >> $S
cat $S
