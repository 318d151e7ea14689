#!/bin/bash
# Round-2 pass R: (1) is the concurrent 2-CTA GEMM hang a hardware-queue false dependency?
# (CUDA_DEVICE_MAX_CONNECTIONS=32), (2) compute-sanitizer on the reworked norm kernels.
O=gpurun_out
mkdir -p $O
S=$O/r2r_summary.txt
: > $S
try() {  # tag env...
  local tag=$1; shift
  local ok=0 hung=0
  for attempt in 1 2 3 4 5 6; do
    env "$@" timeout 60 python tools/pipeline_inproc.py --P 3 --layers-per-stage 1 --seq 4096 --micro 6 --kinds seq1f1b --dump-after 55 > $O/r2r_${tag}_$attempt.txt 2>&1
    if [ $? = 0 ]; then ok=$((ok+1)); else hung=$((hung+1)); fi
  done
  echo "$tag: ok $ok hung $hung" >> $S
}
try conn32_2cta CUDA_DEVICE_MAX_CONNECTIONS=32 SP_GEMM_CTA=2 SP_WGRAD_STREAM=0 SP_ATTN_BWD_CONCURRENT=0
try conn1_2cta CUDA_DEVICE_MAX_CONNECTIONS=1 SP_GEMM_CTA=2 SP_WGRAD_STREAM=0 SP_ATTN_BWD_CONCURRENT=0
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider \
     -k "test_norm_fwd_bwd and (301-2560 or 64-4096 or 9-5120)" > $O/r2r_sanitize_norm_$tool.log 2>&1; echo "norm $tool rc=$?" >> $S
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $O/r2r_sanitize_norm_$tool.log | tail -2 >> $S
done
cat $S
