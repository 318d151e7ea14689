#!/bin/bash
# Stage benches after the GEMM raster: cfg-3 (cwp and even), cfg-4 (with and without the MLP recompute)
O=gpurun_out
mkdir -p $O
: > $O/r2v_stage.jsonl
timeout 900 python bench.py --workload cfg3-stage --no-cpu-baseline >> $O/r2v_stage.jsonl 2> $O/r2v_stage_1.err; echo "cfg3 cwp rc=$?"
timeout 900 python bench.py --workload cfg3-stage --partition even --no-cpu-baseline >> $O/r2v_stage.jsonl 2> $O/r2v_stage_2.err; echo "cfg3 even rc=$?"
timeout 900 python bench.py --workload cfg4-stage --no-cpu-baseline >> $O/r2v_stage.jsonl 2> $O/r2v_stage_3.err; echo "cfg4 rc=$?"
timeout 900 python bench.py --workload cfg4-stage --recompute-mlp --no-cpu-baseline >> $O/r2v_stage.jsonl 2> $O/r2v_stage_4.err; echo "cfg4 recompute rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r2v_stage.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); c = d["config"]
        print(c.get("workload")[:40], c.get("partition_mode"), c.get("recompute"), round(d["value"]), round(d["tflops_per_gpu"]), d["clocks"]["sm_mhz"])
PY
