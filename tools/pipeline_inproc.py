#!/usr/bin/env python
"""Seq1F1B vs batch-level 1F1B at pipeline depth P, executed: P Engine handles (rank r of
world P) on ONE B200, one host thread each, exchanging activations / gradients through the
in-process transport exactly as sp_comm_plan lists them (the multi-rank data plane of
engine.cpp; the reference's pipeline edges sim.cpp:20-23 / :31-33).

Per stage it reports what the device holds, measured:
  * activation_gb_device -- cudaMemGetInfo delta of creating that stage's engine minus its
                         weights / optimizer state: the activation arena (KV slabs, per-(m,s)
                         records) + the fp32 dK/dV accumulator + per-op workspaces, as allocated,
  * arena_gb_planned  -- the activation arena alone (what the device allocation holds),
  * peak_activation_gb -- the live high-water of the executed op order (StepReport),
  * bubble_ratio      -- idle / (last_end - first_start) of the stage's stream from per-op CUDA
                         events (sim.cpp:252-254 definition). With P stages time-sharing one GPU
                         the op durations are inflated by contention, so this is the dependency
                         structure's idle under sharing, not the P-GPU bubble (BASELINE.md §3
                         carries the modeled one, printed next to it).

python tools/pipeline_inproc.py [--model gpt-2.7b|llama-7b] [--P 4] [--layers-per-stage 2] [--seq 32768]
                                [--micro 8] [--k 4] [--sweep T:k:P,...]
Prints one JSON line per (schedule kind, point). --sweep runs the cfg-5 grid points given (k = 1 is
batch-level 1F1B, reference test_schedules.cpp:163-170) with M = 2P."""
import argparse
import faulthandler
import json
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2406_03488_b200 import _capi  # noqa: E402
from paper_2406_03488_b200 import engine as E  # noqa: E402

if "--variant" in sys.argv:  # a tuning build from tools/build_variant.py (investigations only)
    i = sys.argv.index("--variant")
    _capi.LIB_PATH = _capi.LIB_PATH.parent / "variants" / f"libseqpipe_b200_{sys.argv[i + 1]}.so"
    del sys.argv[i:i + 2]
from paper_2406_03488_b200 import planner as pl  # noqa: E402

MODELS = {"gpt-2.7b": dict(family=E.GPT, vocab=50257, hidden=2560, heads=32, head_dim=80, ffn=10240),
          "llama-7b": dict(family=E.LLAMA, vocab=32000, hidden=4096, heads=32, head_dim=128, ffn=11008),
          "tiny": dict(family=E.GPT, vocab=512, hidden=320, heads=4, head_dim=80, ffn=1280)}


def run(kind, P, lps, seq, micro, k, mode, model_name="gpt-2.7b"):
    layers = P * lps
    mk = MODELS[model_name]
    model = E.ModelConfig(dtype=E.BF16, layers=layers, max_seq=seq, seed=42, **mk)
    segs = k if kind.startswith("seq") else 1
    cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=micro, segments=segs, seq_len=seq, layers=layers,
                            hidden_dim=mk["hidden"], param_count=model.param_count())
    cfg.validate()
    part = pl.partition_for(cfg, mode if segs > 1 else "even")
    hub = E.LocalHub(P, watchdog_seconds=600.0)
    engines, dev_bytes = [], []
    torch.cuda.synchronize()
    for r in range(P):
        free0, _ = torch.cuda.mem_get_info(0)
        e = E.Engine(cfg, kind, part, model, rank=r, world_size=P, cuda_device=0)
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info(0)
        e.attach_local(hub)  # (its staging slots are transport memory, not the stage's)
        engines.append(e)
        dev_bytes.append(free0 - free1)
    tok = torch.randint(0, model.vocab, (micro, seq + 1), dtype=torch.int32).numpy()
    out = {}
    print(f"# {kind} P={P} engines built", file=sys.stderr, flush=True)
    for it in range(2):  # step 0 warms up (graph-free path, lazy workspaces), step 1 is reported
        reps, errs = [None] * P, [None] * P

        def go(r):
            try:
                reps[r] = engines[r].step(tok)
            except Exception as ex:  # noqa: BLE001
                errs[r] = ex

        th = [threading.Thread(target=go, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if any(errs):
            raise RuntimeError(errs)
        print(f"# {kind} step {it} done", file=sys.stderr, flush=True)
        out = reps
    stages = []
    for r, rep in enumerate(out):
        stages.append({
            "stage": r + 1,
            "activation_gb_device": round((dev_bytes[r] - rep.weight_bytes) / 1e9, 3),  # arena + dK/dV acc. + workspaces
            "engine_gb_device": round(dev_bytes[r] / 1e9, 3),
            "arena_gb_planned": round(rep.arena_bytes / 1e9, 3),
            "peak_activation_gb": round(rep.peak_activation_bytes / 1e9, 3),
            "bubble_ratio_shared_gpu": round(rep.bubble_ratio, 4),
            "step_ms": round(rep.step_ms, 1),
        })
    modeled = pl.simulate(pl.generate(cfg, kind, part), part, with_series=False)
    for e in engines:
        e.close()
    del hub
    torch.cuda.empty_cache()
    return {"model": model_name, "kind": kind, "P": P, "layers_per_stage": lps, "seq": seq, "micro_batches": micro,
            "segments": segs,
            "partition": list(part.lengths), "stages": stages,
            "modeled_bubble_ratio": float(modeled.aggregate_bubble_ratio),
            "loss": out[-1].loss}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=4)
    ap.add_argument("--layers-per-stage", type=int, default=2)
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--micro", type=int, default=8)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--partition", default="cwp")
    ap.add_argument("--kinds", default="seq1f1b,1f1b")
    ap.add_argument("--model", default="gpt-2.7b", choices=sorted(MODELS))
    ap.add_argument("--sweep", default="")
    ap.add_argument("--dump-after", type=float, default=600.0, help="dump every thread's stack after this many s")
    a = ap.parse_args()
    faulthandler.dump_traceback_later(a.dump_after, exit=False)
    if a.sweep:
        for pt in a.sweep.split(","):
            T, k, P = (int(v) for v in pt.split(":"))
            kind = "seq1f1b" if k > 1 else "1f1b"
            try:
                r = run(kind, P, a.layers_per_stage, T, 2 * P, k, a.partition, a.model)
            except Exception as ex:  # noqa: BLE001 -- e.g. a point whose P engines do not fit one GPU
                r = {"model": a.model, "kind": kind, "P": P, "seq": T, "segments": k, "error": str(ex)[:200]}
                torch.cuda.empty_cache()
            print(json.dumps(r), flush=True)
        return
    res = {}
    for kind in a.kinds.split(","):
        res[kind] = run(kind, a.P, a.layers_per_stage, a.seq, a.micro, a.k, a.partition, a.model)
        print(json.dumps(res[kind]), flush=True)
    if "seq1f1b" in res and "1f1b" in res:
        s, b = res["seq1f1b"]["stages"][0], res["1f1b"]["stages"][0]
        print(json.dumps({"stage1_device_ratio_seq1f1b_over_1f1b": s["activation_gb_device"] / b["activation_gb_device"],
                          "stage1_peak_ratio_seq1f1b_over_1f1b": s["peak_activation_gb"] / b["peak_activation_gb"]}))


if __name__ == "__main__":
    main()
