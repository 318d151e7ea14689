#!/bin/bash
# Round-2 pass B: loss sanity (eager vs graph) at the stage workloads, in-process P=4 pipeline
# memory/bubble (Seq1F1B vs 1F1B), compute-sanitizer, cfg-2 bench with the offline-placed arena.
O=gpurun_out
mkdir -p $O
S=$O/r2b_summary.txt
: > $S
timeout 900 python tools/loss_curve.py cfg3-stage 6 > $O/r2b_loss_cfg3.txt 2>&1; echo "loss cfg3 rc=$?" >> $S
timeout 600 python tools/loss_curve.py cfg3-stage 6 1 > $O/r2b_loss_cfg3_l1.txt 2>&1; echo "loss cfg3 l1 rc=$?" >> $S
timeout 900 python tools/loss_curve.py cfg4-stage 5 > $O/r2b_loss_cfg4.txt 2>&1; echo "loss cfg4 rc=$?" >> $S
timeout 900 python tools/loss_curve.py cfg2 5 4 > $O/r2b_loss_cfg2_l4.txt 2>&1; echo "loss cfg2 rc=$?" >> $S
timeout 1500 python tools/pipeline_inproc.py --P 4 --layers-per-stage 2 > $O/r2b_pipeline_p4.txt 2>&1; echo "pipeline p4 rc=$?" >> $S
timeout 900 python bench.py > $O/r2b_bench.json 2> $O/r2b_bench.err; echo "bench rc=$?" >> $S
bash tools/sanitize.sh r2b >> $S 2>&1
cat $S
