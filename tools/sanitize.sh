#!/bin/bash
# compute-sanitizer passes over the hand-written kernels at small shapes (under gpurun):
# memcheck (out-of-bounds / misaligned global + shared accesses, incl. the KV-slab rows the
# QKV epilogue writes and the dK/dV TMA reduce-add targets), racecheck (shared-memory
# hazards), synccheck (barrier misuse). Logs -> gpurun_out/<TAG>_sanitize_*.log
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
CS="compute-sanitizer --error-exitcode 9 --print-limit 50"
K='tests/test_gpu_kernels.py'
SEL='77-0-2-64-0-dtype1 or 96-160-3-80-0-dtype1 or 200-57-2-128-0-dtype1'
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool python -m pytest $K -q -p no:cacheprovider -x \
     -k "test_attention_fwd_bwd and ($SEL)" > $O/${TAG}_sanitize_attn_$tool.log 2>&1
  echo "attention $tool rc=$?"
  timeout 1200 $CS --tool $tool python -m pytest $K -q -p no:cacheprovider -x \
     -k "test_tcgen05_gemm_layouts and (304-520-200 or 128-256-64)" > $O/${TAG}_sanitize_gemm_$tool.log 2>&1
  echo "gemm $tool rc=$?"
  timeout 1200 $CS --tool $tool python -m pytest $K -q -p no:cacheprovider -x \
     -k "test_norm_fwd_bwd and 301-2560 or test_activation_fwd_bwd and 129-10240" > $O/${TAG}_sanitize_elem_$tool.log 2>&1
  echo "elementwise $tool rc=$?"
done
timeout 1800 $CS --tool memcheck python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -x \
   -k "test_bf16_production_tiny_gpt" > $O/${TAG}_sanitize_engine_memcheck.log 2>&1
echo "engine bf16 memcheck rc=$?"
