#!/bin/bash
# Round-2 evidence pass: cfg-3 / cfg-4 single-stage benches (cwp vs even) and ncu --set full
# captures of the elementwise kernels and the forward GEMMs inside one cfg-2 micro-batch.
mkdir -p gpurun_out
for w in "cfg3-stage --partition cwp" "cfg3-stage --partition even" "cfg4-stage --partition cwp"; do
  tag=$(echo $w | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$tag.log 2>&1
  echo "bench $w rc=$?"
done
B="python bench.py --micro 1 --steps 1 --warmup 0 --graph 0 --no-cpu-baseline"
for k in norm_fwd_vec_k norm_bwd_pair_k norm_apply_vec_k act_fwd_vec_k act_bwd_vec_k ce_k assemble_dqkv_vec_k attn_prep_k adamw_k; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -c 1 -o gpurun_out/r2_ncu_$k -f $B > gpurun_out/r2_ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
timeout 900 ncu --set full --clock-control none -k regex:gemm_tc2_k -c 4 -o gpurun_out/r2_ncu_gemm_fwd -f $B > gpurun_out/r2_ncu_gemm.log 2>&1
echo "ncu gemm rc=$?"
