#!/bin/bash
# Round-2 pass O: norm kernels with the gain / dgain in registers: parity + HBM bench + ncu.
O=gpurun_out
mkdir -p $O
S=$O/r2o_summary.txt
: > $S
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -p no:cacheprovider -k "norm or tiny_gpt or llama or cfg2_shape or recompute" > $O/r2o_pytest.log 2>&1; echo "pytest rc=$?" >> $S
tail -2 $O/r2o_pytest.log >> $S
timeout 300 python tools/elem_bench.py > $O/r2o_elem.jsonl 2>&1
timeout 300 python tools/elem_bench.py 8192 4096 11008 >> $O/r2o_elem.jsonl 2>&1; echo "elem rc=$?" >> $S
cat $O/r2o_elem.jsonl >> $S
for k in norm_fwd_rows_k norm_bwd_rows_k; do
  timeout 300 ncu --set full --clock-control none -k regex:$k -c 1 -o $O/r2o_ncu_$k -f python tools/norm_once.py 10170 2560 > $O/r2o_ncu_$k.log 2>&1; echo "ncu $k rc=$?" >> $S
done
cat $S
