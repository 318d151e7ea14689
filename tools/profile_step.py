#!/usr/bin/env python
"""Kernel-time breakdown of ONE bench step (cfg-2 workload at P=1) via torch.profiler /
CUPTI: real (non-serialised) per-kernel durations, grouped by kernel name, plus the
device-idle time between kernels. tools/profile_step.py [--seq 32768 --micro 8 --k 4]."""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2406_03488_b200 import engine as E  # noqa: E402
from paper_2406_03488_b200 import planner as pl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--micro", type=int, default=8)
ap.add_argument("--k", type=int, default=4)
a = ap.parse_args()
W = bench.WORKLOADS["cfg2"]
preset, ov = bench.scenario_overrides("cfg2", 1, a.micro, a.k, a.seq)
cfg = pl.preset_scenario(preset)
for key, v in ov:
    pl.apply_scenario_override(cfg, key, str(v))
model = E.ModelConfig(family=W["family"], dtype=E.BF16, vocab=W["V"], hidden=W["h"], layers=W["L"], heads=W["H"],
                      head_dim=W["hd"], ffn=W["F"], max_seq=a.seq, seed=42, lr=1e-4, weight_decay=0.0)
part = pl.cwp_partition(cfg)
eng = E.Engine(cfg, "seq1f1b", part, model)
tok = np.random.default_rng(1234).integers(0, model.vocab, size=(cfg.micro_batches, cfg.seq_len + 1)).astype(np.int32)
eng.step(tok)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    rep = eng.step(tok)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs], key=lambda x: x[0])
by = defaultdict(lambda: [0.0, 0])
for s, e, n in kern:
    key = n.replace("void ", "").replace("spk::(anonymous namespace)::", "").replace("spk::<unnamed>::", "")
    key = key.split("(")[0]
    by[key][0] += (e - s) / 1e3
    by[key][1] += 1
span = (kern[-1][1] - kern[0][0]) / 1e3
busy, last = 0.0, kern[0][0]
for s, e, _ in kern:
    busy += max(0, e - max(s, last)) / 1e3
    last = max(last, e)
print(f"step (engine) {rep.step_ms:.1f} ms; profiled span {span:.1f} ms; GPU busy {busy:.1f} ms; idle {span - busy:.1f} ms;"
      f" {len(kern)} kernels")
for k, (ms, n) in sorted(by.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{ms:10.1f} ms {100 * ms / span:5.1f}% {n:6d}  {k[:110]}")
