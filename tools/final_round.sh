#!/bin/bash
# End-of-round GPU evidence: smoke, full GPU parity suite, bench line, per-step kernel profile
# (torch.profiler/CUPTI, real concurrency), ncu launch list of a 1-micro-batch bench step, and
# ncu --set full captures of the three attention kernels + the bench GEMM at the cfg-2 shapes.
# Usage (under gpurun): bash tools/final_round.sh TAG
TAG=${1:-r1f}
O=gpurun_out
mkdir -p $O
S=$O/${TAG}_summary.txt
: > $S
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1800 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/${TAG}_pytest_gpu.log >> $S
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?" >> $S
timeout 600 python tools/profile_step.py > $O/${TAG}_step_profile.txt 2>&1; echo "profile rc=$?" >> $S
KERNELS="attn_bwd_dkv attn_bwd_dq attn_fwd_tc" timeout 1500 bash tools/ncu_attn.sh ${TAG} >> $S 2>&1
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
   python bench.py --steps 1 --warmup 1 --micro 1 --no-cpu-baseline > $O/${TAG}_ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> $S
cat $S
