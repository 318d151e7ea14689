#!/bin/bash
# Round-2 pass C: GPU suite, elementwise HBM bench (paired-warp norm), attention clocks,
# in-process pipeline memory (small, then P=4 cfg-2 width), loss held-out check, bench.
O=gpurun_out
mkdir -p $O
S=$O/r2c_summary.txt
: > $S
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/r2c_pytest_gpu.log >> $S
timeout 300 python tools/elem_bench.py > $O/r2c_elem.jsonl 2>&1; echo "elem rc=$?" >> $S
timeout 300 python tools/elem_bench.py 8192 4096 11008 >> $O/r2c_elem.jsonl 2>&1
for w in "bwd 6674 26094 32 80" "bwd 10170 0 32 80" "fwd 6674 26094 32 80"; do
  timeout 300 python tools/attn_clock.py $w >> $O/r2c_attn_clock.txt 2>&1
done; echo "attn_clock rc=$?" >> $S
timeout 300 python tools/pipeline_inproc.py --P 2 --layers-per-stage 1 --seq 4096 --micro 4 --dump-after 200 > $O/r2c_pipeline_small.txt 2>&1; echo "pipeline small rc=$?" >> $S
timeout 900 python tools/pipeline_inproc.py --P 4 --layers-per-stage 2 --dump-after 420 > $O/r2c_pipeline_p4.txt 2>&1; echo "pipeline p4 rc=$?" >> $S
timeout 600 python tools/loss_curve.py cfg3-stage 6 > $O/r2c_loss_cfg3.txt 2>&1; echo "loss rc=$?" >> $S
timeout 900 python bench.py > $O/r2c_bench.json 2> $O/r2c_bench.err; echo "bench rc=$?" >> $S
for sel in 96-160-3-80-0-dtype1 200-57-2-128-0-dtype1 700-1111-2-80-0-dtype1; do
  timeout 300 compute-sanitizer --tool synccheck --print-limit 3 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider \
     -k "test_attention_fwd_bwd and $sel" > $O/r2c_synccheck_$sel.log 2>&1; echo "synccheck $sel rc=$?" >> $S
done
cat $S
