#!/bin/bash
# Round-2 pass F: P-in-shared-memory forward variant: parity vs fp64, then sustained-clock A/B.
O=gpurun_out
mkdir -p $O
S=$O/r2f_summary.txt
: > $S
timeout 600 python tools/attn_variant_check.py psmem > $O/r2f_check_psmem.txt 2>&1; echo "check psmem rc=$?" >> $S
tail -1 $O/r2f_check_psmem.txt >> $S
for rep in 1 2 3; do
  for v in "" "--variant psmem"; do
    timeout 300 python tools/attn_clock.py $v fwd 6674 26094 32 80 >> $O/r2f_attn_ab.txt 2>&1
    timeout 300 python tools/attn_clock.py $v fwd 10170 0 32 80 >> $O/r2f_attn_ab.txt 2>&1
  done
done; echo "ab rc=$?" >> $S
cat $O/r2f_attn_ab.txt >> $S
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_ps -c 1 -o $O/r2f_attn_fwd_ps -f \
   python tools/attn_once.py --variant psmem > $O/r2f_ncu_fwd_ps.log 2>&1; echo "ncu rc=$?" >> $S
cat $S
