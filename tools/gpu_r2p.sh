#!/bin/bash
# Round-2 pass P (final evidence): smoke, GPU suite, cfg-2 bench, cfg-3 stage bench, step profile,
# ncu launch list + attention ncu, cfg-5 memory sweep executed in-process (LLaMA-7B width).
O=gpurun_out
mkdir -p $O
S=$O/r2p_summary.txt
: > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2p_smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2p_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/r2p_pytest_gpu.log >> $S
timeout 900 python bench.py > $O/r2p_bench.json 2> $O/r2p_bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --workload cfg3-stage --steps 3 --warmup 3 --no-cpu-baseline > $O/r2p_cfg3.json 2> $O/r2p_cfg3.err; echo "cfg3 rc=$?" >> $S
timeout 600 python tools/profile_step.py > $O/r2p_step_profile.txt 2>&1; echo "profile rc=$?" >> $S
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2p_launches.csv \
   python bench.py --steps 1 --warmup 1 --micro 1 --graph 0 --no-cpu-baseline > $O/r2p_ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> $S
KERNELS="attn_bwd_dkv attn_bwd_dq attn_fwd_tc" timeout 1500 bash tools/ncu_attn.sh r2p >> $S 2>&1
timeout 1800 python tools/pipeline_inproc.py --model llama-7b --layers-per-stage 1 \
   --sweep 32768:1:4,32768:2:4,32768:4:4,32768:8:4,32768:16:4,32768:1:8,32768:4:8,32768:16:8 --dump-after 1700 \
   > $O/r2p_cfg5_sweep.txt 2>&1; echo "cfg5 sweep rc=$?" >> $S
cat $S
