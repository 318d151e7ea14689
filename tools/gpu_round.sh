#!/bin/bash
# One GPU session: parity tests, bench line, kernel microbench, ncu launch list + full capture.
# Usage (under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/${TAG}_nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_summary.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_summary.txt
tail -3 $O/${TAG}_pytest_gpu.log >> $O/${TAG}_summary.txt
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?" >> $O/${TAG}_summary.txt
timeout 600 python tools/kernel_bench.py --attn > $O/${TAG}_kernel_bench.jsonl 2>&1; echo "kbench rc=$?" >> $O/${TAG}_summary.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/${TAG}_ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> $O/${TAG}_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dkv -c 1 -o $O/${TAG}_attn_bwd_dkv -f \
   python tools/attn_once.py > $O/${TAG}_ncu_dkv.log 2>&1; echo "ncu-dkv rc=$?" >> $O/${TAG}_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tc -c 1 -o $O/${TAG}_attn_fwd -f \
   python tools/attn_once.py > $O/${TAG}_ncu_fwd.log 2>&1; echo "ncu-fwd rc=$?" >> $O/${TAG}_summary.txt
cat $O/${TAG}_summary.txt
