#!/bin/bash
# Verification final HEAD: smoke, GPU suite, two bench lines
O=gpurun_out
mkdir -p $O
S=$O/r2z9_summary.txt
: > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2z9_smoke.log 2>&1; echo "smoke rc=$?" >> $S
tail -1 $O/r2z9_smoke.log >> $S
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2z9_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -1 $O/r2z9_pytest_gpu.log >> $S
for i in 1 2; do
  timeout 900 python bench.py > $O/r2z9_bench_$i.json 2> $O/r2z9_bench_$i.err; echo "bench $i rc=$?" >> $S
  python -c "import json;d=json.load(open('$O/r2z9_bench_$i.json'));print(round(d['value']),round(d['e2e']['value']),round(d['ms_per_step'],1),d['clocks']['sm_mhz'],d['roofline']['classes']['gemm_tcgen05']['tflops'])" >> $S
done
cat $S
