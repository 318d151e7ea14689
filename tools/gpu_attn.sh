#!/bin/bash
# Attention iteration loop on one GPU: parity, microbench, ncu captures of the three kernels.
TAG=${1:-attn}
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" > $O/${TAG}_summary.txt
tail -3 $O/${TAG}_pytest.log >> $O/${TAG}_summary.txt
timeout 300 python tools/kernel_bench.py --attn-only > $O/${TAG}_kbench.jsonl 2>&1; echo "kbench rc=$?" >> $O/${TAG}_summary.txt
cat $O/${TAG}_kbench.jsonl >> $O/${TAG}_summary.txt
if [ "${NCU:-1}" = "1" ]; then
for k in attn_bwd_dkv attn_bwd_dq attn_fwd_tc; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/${TAG}_$k -f \
   python tools/attn_once.py > $O/${TAG}_ncu_$k.log 2>&1; echo "ncu $k rc=$?" >> $O/${TAG}_summary.txt
done
fi
cat $O/${TAG}_summary.txt
