#!/usr/bin/env python
"""Loss per AdamW step of a bench workload on one fixed synthetic batch, eager vs CUDA-graph
replay: tools/loss_curve.py [workload] [steps] [layers]. A sanity probe for the training loop
(a causal model on uniform random tokens can only memorise, so the loss stays near ln V)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2406_03488_b200 import engine as E  # noqa: E402
from paper_2406_03488_b200 import planner as pl  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "cfg3-stage"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
W = bench.WORKLOADS[w]
layers = int(sys.argv[3]) if len(sys.argv) > 3 else (W["stage_layers"] or W["L"])
preset, ov = bench.scenario_overrides(w, 1, 2, W["k"], W["seq"])
full = pl.preset_scenario(preset)
for k, v in ov:
    pl.apply_scenario_override(full, k, str(v))
lengths = pl.cwp_partition(full).lengths
for graph in (False, True):
    model = E.ModelConfig(family=W["family"], dtype=E.BF16, vocab=W["V"], hidden=W["h"], layers=layers, heads=W["H"],
                          head_dim=W["hd"], ffn=W["F"], max_seq=W["seq"], seed=42, lr=1e-4, weight_decay=0.0)
    cfg = pl.ScenarioConfig(pipeline_size=1, micro_batches=2, segments=W["k"], seq_len=W["seq"], layers=layers,
                            hidden_dim=W["h"], param_count=model.param_count())
    eng = E.Engine(cfg, "seq1f1b", pl.make_partition(lengths, cfg), model)
    tok = np.random.default_rng(1234).integers(0, W["V"], size=(2, W["seq"] + 1)).astype(np.int32)
    losses = []
    for i in range(steps):
        losses.append(eng.step(tok).loss)
        if i == 0 and graph:
            eng.enable_graph(True)
    # loss of an unseen batch before its update: memorisation does not carry over, a leak would
    held = eng.step(np.random.default_rng(99).integers(0, W["V"], size=(2, W["seq"] + 1)).astype(np.int32)).loss
    print(f"{w} layers {layers} graph {graph}: ln V = {np.log(W['V']):.3f}, losses " +
          " ".join(f"{x:.4f}" for x in losses) + f", held-out batch {held:.4f}", flush=True)
    eng.close()
