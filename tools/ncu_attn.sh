#!/bin/bash
# ncu --set full of the attention kernels at one shape: tools/ncu_attn.sh TAG [n q_off H hd]
TAG=$1; shift
for k in ${KERNELS:-attn_bwd_dkv attn_bwd_dq attn_fwd_tc}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_$k -f \
   python tools/attn_once.py "$@" > gpurun_out/${TAG}_ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
