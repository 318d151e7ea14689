#!/bin/bash
# Round-2 pass E: full GPU suite (streaming norm kernels, GEMM tail split, owned-slot transport),
# elementwise HBM bench, attention softmax exp-split variants at sustained clocks, bench.
O=gpurun_out
mkdir -p $O
S=$O/r2e_summary.txt
: > $S
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2e_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/r2e_pytest_gpu.log >> $S
timeout 300 python tools/elem_bench.py > $O/r2e_elem.jsonl 2>&1; echo "elem rc=$?" >> $S
timeout 300 python tools/elem_bench.py 8192 4096 11008 >> $O/r2e_elem.jsonl 2>&1
for rep in 1 2; do
  for v in "" "--variant dq1" "--variant dq2" "--variant dkv1"; do
    timeout 300 python tools/attn_clock.py $v bwd 6674 26094 32 80 >> $O/r2e_attn_ab.txt 2>&1
  done
  for v in "" "--variant fwd3" "--variant fwd1"; do
    timeout 300 python tools/attn_clock.py $v fwd 6674 26094 32 80 >> $O/r2e_attn_ab.txt 2>&1
  done
done; echo "attn ab rc=$?" >> $S
timeout 900 python bench.py > $O/r2e_bench.json 2> $O/r2e_bench.err; echo "bench rc=$?" >> $S
# in-process pipeline hang bisection (GPU utilisation sampled alongside)
for cfg in "--P 4 --layers-per-stage 1 --seq 4096 --micro 8" "--P 2 --layers-per-stage 2 --seq 32768 --micro 4" \
           "--P 4 --layers-per-stage 1 --seq 16384 --micro 8" "--P 4 --layers-per-stage 2 --seq 32768 --micro 8"; do
  tag=$(echo $cfg | tr -d ' -')
  (for i in $(seq 1 40); do nvidia-smi --query-gpu=utilization.gpu,power.draw,memory.used --format=csv,noheader; sleep 5; done) > $O/r2e_smi_$tag.txt 2>&1 &
  SMI=$!
  timeout 240 python tools/pipeline_inproc.py $cfg --kinds seq1f1b --dump-after 200 > $O/r2e_pipe_$tag.txt 2>&1; echo "pipe $tag rc=$?" >> $S
  kill $SMI 2>/dev/null
done
cat $S
