#!/bin/bash
# Round-2 pass K: GPU suite, Seq1F1B vs 1F1B executed with P stages in one process (1-CTA GEMMs
# there), bench line.
O=gpurun_out
mkdir -p $O
S=$O/r2k_summary.txt
: > $S
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2k_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/r2k_pytest_gpu.log >> $S
timeout 1200 python tools/pipeline_inproc.py --P 4 --layers-per-stage 2 --seq 32768 --micro 8 --dump-after 1100 > $O/r2k_pipeline_p4.txt 2>&1; echo "pipeline p4 rc=$?" >> $S
timeout 1200 python tools/pipeline_inproc.py --P 8 --layers-per-stage 1 --seq 32768 --micro 16 --dump-after 1100 > $O/r2k_pipeline_p8.txt 2>&1; echo "pipeline p8 rc=$?" >> $S
timeout 900 python bench.py > $O/r2k_bench.json 2> $O/r2k_bench.err; echo "bench rc=$?" >> $S
cat $S
