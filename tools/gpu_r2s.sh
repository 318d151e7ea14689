#!/bin/bash
# Round-2 final verification of HEAD: smoke, GPU suite, two bench lines (run-to-run spread).
O=gpurun_out
mkdir -p $O
S=$O/r2s_summary.txt
: > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s_smoke.log 2>&1; echo "smoke rc=$?" >> $S
tail -3 $O/r2s_smoke.log >> $S
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2s_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/r2s_pytest_gpu.log >> $S
for i in 1 2; do
  timeout 900 python bench.py > $O/r2s_bench_$i.json 2> $O/r2s_bench_$i.err; echo "bench $i rc=$?" >> $S
done
cat $S
