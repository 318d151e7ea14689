#!/bin/bash
# Same-box A/B of the fused GeLU-backward GEMM epilogue (SP_FUSE_GELU_BWD=1 vs 0), alternating
O=gpurun_out
mkdir -p $O
S=$O/r2ab_summary.txt
: > $S
for i in 1 2; do
  for f in 1 0; do
    SP_FUSE_GELU_BWD=$f timeout 900 python bench.py --no-cpu-baseline > $O/r2ab_f${f}_$i.json 2> $O/r2ab_f${f}_$i.err
    python -c "import json;d=json.load(open('$O/r2ab_f${f}_$i.json'));c=d['roofline']['classes'];print('fuse=$f', round(d['value']),round(d['e2e']['value']),round(d['ms_per_step'],1),d['clocks']['sm_mhz'],round(c['gemm_tcgen05']['ms']),round(c['gemm_tcgen05']['tflops']))" >> $S
  done
done
cat $S
