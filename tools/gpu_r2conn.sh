#!/bin/bash
# Same-box A/B: CUDA_DEVICE_MAX_CONNECTIONS 32 vs the default (8), alternating
O=gpurun_out
mkdir -p $O
S=$O/r2conn_summary.txt
: > $S
for i in 1 2; do
  for c in 32 default; do
    if [ $c = default ]; then unset CUDA_DEVICE_MAX_CONNECTIONS; else export CUDA_DEVICE_MAX_CONNECTIONS=$c; fi
    timeout 900 python bench.py --no-cpu-baseline > $O/r2conn_${c}_$i.json 2> $O/r2conn_${c}_$i.err
    python -c "import json;d=json.load(open('$O/r2conn_${c}_$i.json'));print('conn=$c', round(d['value']),round(d['e2e']['value']),round(d['ms_per_step'],1),d['clocks']['sm_mhz'])" >> $S
  done
done
unset CUDA_DEVICE_MAX_CONNECTIONS
cat $S
