#!/bin/bash
# Final-code evidence: CUPTI step profile and the ncu launch list of a (1-micro-batch) bench step
O=gpurun_out
mkdir -p $O
S=$O/r2fin_summary.txt
: > $S
timeout 600 python tools/profile_step.py > $O/r2fin_step_profile.txt 2>&1; echo "profile rc=$?" >> $S
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2fin_launches.csv \
   python bench.py --steps 1 --warmup 1 --micro 1 --graph 0 --no-cpu-baseline > $O/r2fin_ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> $S
python tools/launch_shares.py $O/r2fin_launches.csv > $O/r2fin_launch_shares.txt 2>&1
head -14 $O/r2fin_step_profile.txt >> $S
head -12 $O/r2fin_launch_shares.txt >> $S
cat $S
