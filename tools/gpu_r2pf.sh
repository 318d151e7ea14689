#!/bin/bash
# weight-gradient epilogue prefetch: GEMM tests, then isolated A/B vs the per-chunk loads (variant), interleaved
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -p no:cacheprovider -k "gemm or engine_step or zero_bubble" > $O/r2pf_pytest.log 2>&1; tail -2 $O/r2pf_pytest.log
: > $O/r2pf_ab.jsonl
for i in 1 2; do
  python tools/gemm_tail_ab.py prefetch >> $O/r2pf_ab.jsonl 2>&1
  python tools/gemm_tail_ab.py --variant noprefetch >> $O/r2pf_ab.jsonl 2>&1
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/r2pf_ab.jsonl"):
    if l.startswith("{"):
        j = json.loads(l); d[(j["gemm"], j["tag"])].append(j["ms"])
for (g, t), v in sorted(d.items()):
    if "wgrad" in g:
        print(f"{g:16s} {t:10s} " + " ".join(f"{x:.4f}" for x in v))
PY
