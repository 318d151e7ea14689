#!/bin/bash
# Round-2 GPU pass: smoke, GPU parity suite, cfg-2 bench line, then (EVIDENCE=1) the
# cfg-3/cfg-4 stage benches and elementwise/GEMM ncu captures of tools/gpu_r2_evidence.sh.
# Usage (under gpurun): bash tools/gpu_r2.sh TAG
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
S=$O/${TAG}_summary.txt
: > $S
nvidia-smi > $O/${TAG}_nvsmi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $S
if [ "${TESTS:-1}" = 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
  tail -5 $O/${TAG}_pytest_gpu.log >> $S
fi
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?" >> $S
if [ "${EVIDENCE:-0}" = 1 ]; then bash tools/gpu_r2_evidence.sh >> $S 2>&1; fi
cat $S
