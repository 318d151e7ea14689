#!/bin/bash
# IPC transport diagnosis on one B200 (several processes share the GPU)
O=gpurun_out
mkdir -p $O
export SP_P2P_WATCHDOG_S=30
timeout 200 python tools/ipc_debug.py --P 2 --k 1 --kind 1f1b --steps 2 > $O/ipcdbg_a.txt 2>&1; echo "a rc=$?" >> $O/ipcdbg_a.txt
grep -v "^  File" $O/ipcdbg_a.txt | head -30
if grep -q "^ok" $O/ipcdbg_a.txt; then
  timeout 200 python tools/ipc_debug.py --P 4 --k 4 --steps 3 --bf16 > $O/ipcdbg_b.txt 2>&1; echo "b rc=$?" >> $O/ipcdbg_b.txt
  grep -v "^  File" $O/ipcdbg_b.txt | head -30
  timeout 900 python -m pytest tests/test_gpu_multiprocess_ipc.py -x -q -p no:cacheprovider > $O/r2u_ipc.log 2>&1; tail -15 $O/r2u_ipc.log
fi
