#!/bin/bash
# Round-2 pass G: which kernel hangs in the in-process 4-stage pipeline (cuda-gdb attach).
O=gpurun_out
mkdir -p $O
S=$O/r2g_summary.txt
: > $S
run_probe() {  # tag, args...
  local tag=$1; shift
  python tools/pipeline_inproc.py "$@" --kinds seq1f1b --dump-after 100 > $O/r2g_$tag.txt 2>&1 &
  local pid=$!
  for i in $(seq 1 24); do sleep 5; kill -0 $pid 2>/dev/null || break; done
  if kill -0 $pid 2>/dev/null; then
    echo "$tag: still running after 120 s -> cuda-gdb" >> $S
    timeout 120 cuda-gdb -p $pid -batch -ex "info cuda kernels" -ex "info cuda devices" > $O/r2g_gdb_$tag.txt 2>&1
    head -40 $O/r2g_gdb_$tag.txt >> $S
    kill -9 $pid 2>/dev/null
    sleep 5
  else
    wait $pid; echo "$tag: finished rc=$?" >> $S
  fi
}
run_probe tiny_p4 --model tiny --P 4 --layers-per-stage 1 --seq 4096 --micro 8
run_probe gpt_p3 --P 3 --layers-per-stage 1 --seq 4096 --micro 6
run_probe gpt_p4 --P 4 --layers-per-stage 1 --seq 4096 --micro 8
timeout 300 python tools/elem_bench.py > $O/r2g_elem.jsonl 2>&1
SP_FLUSH=write timeout 300 python tools/elem_bench.py >> $O/r2g_elem.jsonl 2>&1
timeout 300 python tools/elem_bench.py 8192 4096 11008 >> $O/r2g_elem.jsonl 2>&1; echo "elem rc=$?" >> $S
cat $S
