#!/bin/bash
# GEMM raster group-size sweep (4 / 8 / 16 m-blocks per group), interleaved on one box
O=gpurun_out
mkdir -p $O
: > $O/r2z2_gemm_ab.jsonl
for i in 1 2; do
  python tools/gemm_tail_ab.py g8 >> $O/r2z2_gemm_ab.jsonl 2>&1
  python tools/gemm_tail_ab.py --variant g4 >> $O/r2z2_gemm_ab.jsonl 2>&1
  python tools/gemm_tail_ab.py --variant g16 >> $O/r2z2_gemm_ab.jsonl 2>&1
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/r2z2_gemm_ab.jsonl"):
    if l.startswith("{"):
        j = json.loads(l); d[(j["gemm"], j["tag"])].append(j["ms"])
for (g, t), v in sorted(d.items()):
    print(f"{g:16s} {t:8s} " + " ".join(f"{x:.4f}" for x in v))
PY
