#!/bin/bash
# Round-2 verification after the IPC transport: smoke, GPU suite, bench N=1, and the bench's
# N=2 path under torchrun with both ranks on the one GPU (--transport ipc; functional check).
O=gpurun_out
mkdir -p $O
S=$O/r2t_summary.txt
: > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2t_smoke.log 2>&1; echo "smoke rc=$?" >> $S
tail -3 $O/r2t_smoke.log >> $S
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2t_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $O/r2t_pytest_gpu.log >> $S
SP_P2P_WATCHDOG_S=240 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --transport ipc --steps 2 --warmup 3 > $O/r2t_bench_n2.json 2> $O/r2t_bench_n2.err
echo "bench n2 rc=$?" >> $S
tail -c 600 $O/r2t_bench_n2.err >> $S
timeout 900 python bench.py > $O/r2t_bench_1.json 2> $O/r2t_bench_1.err; echo "bench rc=$?" >> $S
cat $S
