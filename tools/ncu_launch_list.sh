#!/bin/bash
# ncu launch list (device time of every kernel, cold-cache, serialised) of one
# timed bench step: skip the warm-up step's launches, capture the next step's.
TAG=${1:-r1}
N=${2:-24961}   # launches per step (bench.py "gpu_launches" / steps)
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none -s $((N + 250)) -c $N --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "ncu rc=$?"
python tools/launch_shares.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_shares.txt 2>&1
cat gpurun_out/${TAG}_launch_shares.txt
