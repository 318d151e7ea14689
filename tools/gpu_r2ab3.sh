#!/bin/bash
# GPU suite, then same-box A/B of the fused GeLU forward (up-projection epilogue writes g) vs the elementwise kernel
O=gpurun_out
mkdir -p $O
S=$O/r2ab3_summary.txt
: > $S
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2ab3_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -1 $O/r2ab3_pytest_gpu.log >> $S
for i in 1 2; do
  for f in 1 0; do
    SP_FUSE_GELU_FWD=$f timeout 900 python bench.py --no-cpu-baseline > $O/r2ab3_f${f}_$i.json 2> $O/r2ab3_f${f}_$i.err
    python -c "import json;d=json.load(open('$O/r2ab3_f${f}_$i.json'));c=d['roofline']['classes'];print('fuse=$f', round(d['value']),round(d['e2e']['value']),round(d['ms_per_step'],1),d['clocks']['sm_mhz'],round(c['gemm_tcgen05']['ms']),round(c['gemm_tcgen05']['tflops']),d['loss'])" >> $S
  done
done
cat $S
