#!/bin/bash
# GEMM raster A/B (grouped 8 m-blocks vs m-fastest) on one box, interleaved; GEMM parity tests; DRAM bytes under ncu
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -p no:cacheprovider -k "gemm" > $O/r2z_pytest.log 2>&1; tail -2 $O/r2z_pytest.log
for i in 1 2; do
  python tools/gemm_tail_ab.py grouped >> $O/r2z_gemm_ab.jsonl 2>&1
  python tools/gemm_tail_ab.py --variant mfast >> $O/r2z_gemm_ab.jsonl 2>&1
done
SP_GEMM_ONLY=mlp_down_fwd SP_GEMM_REPS=1 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc \
    --launch-skip 3 -c 1 python tools/gemm_tail_ab.py grouped > $O/r2z_ncu_dram.txt 2>&1
SP_GEMM_ONLY=mlp_down_fwd SP_GEMM_REPS=1 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc \
    --launch-skip 3 -c 1 python tools/gemm_tail_ab.py --variant mfast >> $O/r2z_ncu_dram.txt 2>&1
grep -E "dram__bytes|duration" $O/r2z_ncu_dram.txt
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/r2z_gemm_ab.jsonl"):
    if l.startswith("{"):
        j = json.loads(l); d[(j["gemm"], j["tag"])].append(j["ms"])
for (g, t), v in sorted(d.items()):
    print(f"{g:16s} {t:8s} " + " ".join(f"{x:.4f}" for x in v))
PY
