#!/bin/bash
# Round-2 pass D: GEMM tail split (tests + A/B), multi-rank tests + in-process P=4 pipeline with
# owned staging slots, bench, step profile, ncu launch list of a 1-micro-batch step, ncu --set
# full of the attention kernels at the cfg-2 long shape.
O=gpurun_out
mkdir -p $O
S=$O/r2d_summary.txt
: > $S
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py -q -p no:cacheprovider -k "gemm or multirank or unmatched or interleaved_table" > $O/r2d_pytest.log 2>&1; echo "pytest gemm+multirank rc=$?" >> $S
tail -2 $O/r2d_pytest.log >> $S
SP_GEMM_TAIL_SPLIT=0 timeout 300 python tools/gemm_tail_ab.py 0 > $O/r2d_gemm_tail.jsonl 2>&1
timeout 300 python tools/gemm_tail_ab.py 1 >> $O/r2d_gemm_tail.jsonl 2>&1; echo "gemm ab rc=$?" >> $S
timeout 900 python tools/pipeline_inproc.py --P 4 --layers-per-stage 2 --dump-after 600 > $O/r2d_pipeline_p4.txt 2>&1; echo "pipeline p4 rc=$?" >> $S
timeout 900 python bench.py > $O/r2d_bench.json 2> $O/r2d_bench.err; echo "bench rc=$?" >> $S
timeout 600 python tools/profile_step.py > $O/r2d_step_profile.txt 2>&1; echo "profile rc=$?" >> $S
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2d_launches.csv \
   python bench.py --steps 1 --warmup 1 --micro 1 --graph 0 --no-cpu-baseline > $O/r2d_ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> $S
KERNELS="attn_bwd_dkv attn_bwd_dq attn_fwd_tc" timeout 1500 bash tools/ncu_attn.sh r2d >> $S 2>&1
cat $S
