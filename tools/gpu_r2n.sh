#!/bin/bash
# Round-2 pass N: GPU suite (recompute-MLP test), cfg-2 bench, cfg-4 stage with and without the
# MLP recompute, smoke.
O=gpurun_out
mkdir -p $O
S=$O/r2n_summary.txt
: > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2n_smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2n_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/r2n_pytest_gpu.log >> $S
timeout 900 python bench.py > $O/r2n_bench.json 2> $O/r2n_bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --workload cfg4-stage --steps 3 --warmup 3 --no-cpu-baseline > $O/r2n_cfg4.json 2> $O/r2n_cfg4.err; echo "cfg4 rc=$?" >> $S
timeout 900 python bench.py --workload cfg4-stage --recompute-mlp --steps 3 --warmup 3 --no-cpu-baseline > $O/r2n_cfg4_rc.json 2> $O/r2n_cfg4_rc.err; echo "cfg4 recompute rc=$?" >> $S
cat $S
