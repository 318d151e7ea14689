#!/usr/bin/env python
"""Seq1F1B training-step benchmark (B200, sm_100a engine).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): GPT-2.7B (h 2560, L 32, 32 heads x 80,
FFN 4h, vocab 50257, learned positions), seq 32K split into k = 4 computation-
balanced (cwp) sub-sequences, M = 8 micro-batches, Seq1F1B schedule, bf16 with
fp32 masters/grads and an AdamW step, random-init weights, synthetic tokens.
Pipeline depth = GPU count (one stage per rank, NCCL P2P between stages).

One JSON line on rank 0. `value` = tokens/s with tokens already in HBM;
`e2e` = the same through the public C-ABI with host tokens (H2D copy of the
step's tokens and D2H of the loss inside the timed region). Kernel roofline
from CUDA-event probes around every GEMM / attention launch of the timed
steps. `--impl reference` times the CPU restatement of the same step
(oracle/transformer.py, numpy fp32 on all host cores) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tokens/sec (8×B200, 32K seq) vs roofline; bubble ratio; peak activation GB/stage"
WORKLOAD = "GPT-2.7B seq 32K, 4 sub-sequences (cwp), Seq1F1B, pipeline depth = GPU count"


def peaks():
    """(burst, sustained) bf16 TFLOP/s and HBM GB/s: MEASURED_PEAKS.json when the driver wrote it,
    else the fallback figures of the B200 profiling recipe."""
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def traffic_of(kernel):
    """DRAM bytes per launch of the dominant kernel class from the committed ncu capture."""
    try:
        d = json.loads((ROOT / "profiles" / "r1_traffic.json").read_text())[kernel]
        return d["dram_bytes_per_launch"], d["launch"]
    except Exception:
        return None, None


def model_and_cfg(n_gpus: int, seq: int, micro: int, k: int, dtype_bf16=True):
    from paper_2406_03488_b200 import engine as E
    from paper_2406_03488_b200 import planner as pl
    model = E.ModelConfig(family=E.GPT, dtype=E.BF16 if dtype_bf16 else E.F32, vocab=50257, hidden=2560, layers=32,
                          heads=32, head_dim=80, ffn=4 * 2560, max_seq=seq, seed=42, lr=1e-4, weight_decay=0.0)
    cfg = pl.preset_scenario("gpt-2.7b")  # Table 1 preset, overridden as SURVEY §8d cfg-2
    pl.apply_scenario_override(cfg, "pipeline_size", str(n_gpus))
    pl.apply_scenario_override(cfg, "seq_len", str(seq))
    pl.apply_scenario_override(cfg, "segments", str(k))
    pl.apply_scenario_override(cfg, "micro_batches", str(micro))
    cfg.validate()
    return model, cfg


def flops_per_step(model, cfg, lengths):
    """Algorithmic FLOPs: per segment F = 2*N*n + 4*L*h*n*(prefix + n/2)
    (+ LM head 2*V*h*n), B = 2F; times M micro-batches."""
    h, L, F, V = model.hidden, model.layers, model.ffn, model.vocab
    n_nonemb = L * (4 * h * h + 2 * h * F)
    tot, pre = 0.0, 0
    for n in lengths:
        f = 2 * n_nonemb * n + 4 * L * h * n * (pre + n / 2) + 2 * V * h * n
        tot += 3 * f
        pre += n
    return tot * cfg.micro_batches


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(budget_s: float = 20.0):
    """Bounded CPU sample of the same step: numpy fp32 forward+backward of GPT-2.7B
    layers (h 2560, 32x80 heads, FFN 10240) on a 1024-token sub-sequence at prefix 0,
    repeated within the time budget, all host cores (BLAS threads). Returns FLOP/s."""
    from oracle.transformer import Model, GPT
    h, H, F, n = 2560, 32, 10240, 1024
    rng = np.random.default_rng(0)
    L = 1
    p = {"embed": rng.normal(0, .02, (512, h)).astype(np.float32), "pos": rng.normal(0, .02, (n, h)).astype(np.float32),
         "final_norm": np.ones((1, h), np.float32), "lm_head": rng.normal(0, .02, (512, h)).astype(np.float32),
         "layer0.norm1": np.ones((1, h), np.float32), "layer0.norm2": np.ones((1, h), np.float32),
         "layer0.wqkv": rng.normal(0, .02, (3 * h, h)).astype(np.float32),
         "layer0.wo": rng.normal(0, .02, (h, h)).astype(np.float32),
         "layer0.w1": rng.normal(0, .02, (F, h)).astype(np.float32),
         "layer0.w2": rng.normal(0, .02, (h, F)).astype(np.float32)}
    m = Model(GPT, 512, h, L, H, h // H, F)
    tok = rng.integers(0, 512, size=(1, n + 1)).astype(np.int32)
    layer_flops = 3 * (2 * (4 * h * h + 2 * h * F) * n + 4 * h * n * (n / 2)) + 3 * 2 * 512 * h * n
    done, t0 = 0, time.perf_counter()
    while True:
        m.step(p, tok, [n])
        done += 1
        el = time.perf_counter() - t0
        if el > budget_s or done >= 50:
            break
    return layer_flops * done / el, f"{done} x fwd+bwd of 1 GPT-2.7B layer (+head) on a 1024-token sub-sequence, " \
        f"numpy fp64 oracle, {el:.1f} s"


def run_reference(args, rank, world):
    """--impl reference: the CPU implementation of the path on the host cores."""
    if rank != 0:
        return 0
    from paper_2406_03488_b200 import planner as pl
    model, cfg = model_and_cfg(args.gpus, args.seq, args.micro, args.k)
    part = pl.cwp_partition(cfg)
    tokens = cfg.micro_batches * cfg.seq_len
    fl = flops_per_step(model, cfg, part.lengths)
    cores = os.cpu_count() or 1
    rates = []
    for i in range(args.warmup + args.steps):
        r, sample = cpu_sample(budget_s=max(2.0, args.ref_budget / max(1, args.steps + args.warmup)))
        if i >= args.warmup:
            rates.append(r)
    rate = statistics.median(rates)
    tps = rate / (fl / tokens)
    ms = fl / rate * 1e3
    planner_ns = None
    try:
        from oracle import ref
        planner_ns = ref.time_planner(cfg, "seq1f1b", "cwp", 20)
    except Exception:
        pass
    line = {"impl": "reference", "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD + " (CPU oracle, extrapolated by FLOPs)", "model": "gpt-2.7b",
                       "global_batch": cfg.micro_batches, "seq_len": cfg.seq_len, "parallelism": f"pp{args.gpus}"},
            "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample,
                             "reference_planner_ms": None if planner_ns is None else planner_ns / 1e6},
            "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--micro", type=int, default=0, help="micro-batches (default 8, 2P when P > 4)")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--kind", default="seq1f1b")
    ap.add_argument("--ref-budget", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--compare-1f1b", action="store_true", help="also run batch-level 1F1B (k=1)")
    args = ap.parse_args()
    if not args.micro:
        args.micro = 8 if args.gpus <= 4 else 2 * args.gpus

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE {world} != --gpus {args.gpus}"}))
        return 2
    dist = None
    if world > 1:
        import torch.distributed as dist  # plumbing only: id exchange, barriers, max-over-ranks
        dist.init_process_group("gloo")
    if args.impl == "reference":
        rc = run_reference(args, rank, world)
        if dist:
            dist.barrier()
        return rc

    from paper_2406_03488_b200 import engine as E
    from paper_2406_03488_b200 import planner as pl

    model, cfg = model_and_cfg(args.gpus, args.seq, args.micro, args.k)
    part = pl.cwp_partition(cfg) if args.k > 1 else pl.even_partition(cfg)
    model.flags = E.FLAG_TIMELINE
    eng = E.Engine(cfg, args.kind, part, model, rank=rank, world_size=world, cuda_device=local)
    if world > 1:
        ids = [E.nccl_unique_id() for _ in range(4)] if rank == 0 else [None] * 4
        dist.broadcast_object_list(ids, src=0)
        eng.comm_init(ids)

    T = cfg.seq_len
    rng = np.random.default_rng(1234)
    tokens = rng.integers(0, model.vocab, size=(cfg.micro_batches, T + 1), dtype=np.int64).astype(np.int32)
    import ctypes
    from paper_2406_03488_b200 import _capi
    lib = _capi.lib()
    tok_dev = ctypes.c_void_p()
    import torch  # device memory plumbing for the resident-token run
    tok_t = torch.from_numpy(tokens).to(f"cuda:{local}")
    tok_ptr = tok_t.data_ptr()

    def barrier():
        lib.sp_device_synchronize(local)
        if dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        eng.step(tok_ptr, on_device=True)

    # ---- timed: tokens resident in HBM, kernel probes on
    eng.set_flags(E.FLAG_TIMELINE | E.FLAG_KPROBE)
    barrier()
    reps = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            reps.append(eng.step(tok_ptr, on_device=True))
        barrier()
    step_ms = max_over_ranks(sum(r.step_ms for r in reps) / len(reps))
    # ---- timed e2e: host tokens through the public C-ABI, loss read back each step
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = eng.step(tokens, on_device=False)
        e2e_ms.append(r.step_ms)
    barrier()
    e2e_step = max_over_ranks(sum(e2e_ms) / len(e2e_ms))

    tok_per_step = cfg.micro_batches * T
    value = tok_per_step / (step_ms / 1e3)
    e2e = tok_per_step / (e2e_step / 1e3)
    last = reps[-1]
    fl = flops_per_step(model, cfg, part.lengths)
    burst, sustained, hbm, src = peaks()
    bubble = max_over_ranks(statistics.mean(r.bubble_ratio for r in reps))
    peak_act = max_over_ranks(last.peak_activation_bytes) / 1e9
    launches = int(sum(r.kernel_launches for r in reps))

    # dominant kernel class over the timed steps (probe events on the engine stream)
    cls_ms = [sum(r.class_ms[c] for r in reps) for c in range(3)]
    cls_fl = [sum(r.class_flops[c] for r in reps) for c in range(3)]
    cls_n = [sum(r.class_launches[c] for r in reps) for c in range(3)]
    dom = int(np.argmax(cls_ms))
    names = ["gemm_tcgen05", "attention_fwd", "attention_bwd"]
    achieved = cls_fl[dom] / (cls_ms[dom] / 1e3) / 1e12 if cls_ms[dom] > 0 else None

    # modeled reference numbers (compiled reference planner when present, else ours)
    modeled = {}
    try:
        sch = pl.generate(cfg, args.kind, part)
        rep_m = pl.simulate(sch, part, with_series=False)
        modeled = {"bubble_ratio": float(rep_m.aggregate_bubble_ratio),
                   "peak_tokens": float(rep_m.max_peak_memory)}
    except Exception as e:  # pragma: no cover
        modeled = {"error": str(e)}
    mem_1f1b = None
    try:
        cfg1 = model_and_cfg(args.gpus, args.seq, args.micro, 1)[1]
        p1 = pl.even_partition(cfg1)
        live, arena, dkv = E.plan_memory(cfg1, "1f1b", p1, model, stage=1)
        sch1 = pl.generate(cfg1, "1f1b", p1)
        r1 = pl.simulate(sch1, p1, with_series=False)
        mem_1f1b = {"peak_activation_gb_stage1_planned": live / 1e9,
                    "modeled_bubble_ratio": float(r1.aggregate_bubble_ratio)}
    except Exception as e:  # pragma: no cover
        mem_1f1b = {"error": str(e)}
    # Engine arena plan (host-side replay of each schedule's op order, KV-prefix slabs
    # included) for Seq1F1B vs batch-level 1F1B of the same model at several pipeline
    # depths: at depth 1 both schedules hold one micro-batch, the paper's memory claim is
    # about depth > 1 (stage 1 holds P micro-batches under 1F1B).
    memory_model = {}
    for P in sorted({args.gpus, 4, 8}):
        try:
            Mp = cfg.micro_batches if P == args.gpus else (8 if P <= 4 else 2 * P)
            cs = model_and_cfg(P, args.seq, Mp, args.k)[1]
            c1 = model_and_cfg(P, args.seq, Mp, 1)[1]
            ls, _, _ = E.plan_memory(cs, "seq1f1b", pl.cwp_partition(cs), model, stage=1)
            l1, _, _ = E.plan_memory(c1, "1f1b", pl.even_partition(c1), model, stage=1)
            rs = pl.simulate(pl.generate(cs, "seq1f1b", pl.cwp_partition(cs)), pl.cwp_partition(cs), with_series=False)
            rb = pl.simulate(pl.generate(c1, "1f1b", pl.even_partition(c1)), pl.even_partition(c1), with_series=False)
            memory_model[f"P{P}_M{Mp}"] = {
                "seq1f1b_peak_activation_gb_stage1": ls / 1e9, "1f1b_peak_activation_gb_stage1": l1 / 1e9,
                "ratio": ls / l1 if l1 else None,
                "seq1f1b_modeled_bubble": float(rs.aggregate_bubble_ratio),
                "1f1b_modeled_bubble": float(rb.aggregate_bubble_ratio)}
        except Exception as e:  # pragma: no cover
            memory_model[f"P{P}"] = {"error": str(e)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rate, sample = cpu_sample(budget_s=20.0)
        cpu = {"value": rate / (fl / tok_per_step), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
               "sample": sample}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, seed 1234; random-init weights)",
            "config": {"workload": WORKLOAD, "model": "gpt-2.7b", "global_batch": cfg.micro_batches,
                       "seq_len": T, "segments": cfg.segments, "partition": part.lengths,
                       "schedule": args.kind, "parallelism": f"pp{args.gpus}",
                       "l2": "inputs larger than L2 (weights+activations >> 126 MB)"},
            "tflops_per_gpu": fl / (step_ms / 1e3) / 1e12 / args.gpus,
            "model_flops_frac_of_peak": fl / (step_ms / 1e3) / 1e12 / args.gpus / sustained,
            "bubble_ratio": bubble, "modeled": modeled,
            "peak_activation_gb_per_stage": peak_act,
            "batch_level_1f1b": mem_1f1b,
            "memory_model": memory_model,
            # Kernels timed inside a seconds-long step run under the power cap: the
            # denominator is the sustained bf16 figure (burst reported beside it).
            "roofline": {"bound": "tensor", "kernel": names[dom], "achieved": achieved, "peak": sustained,
                         "peak_kind": f"bf16 sustained ({src})", "peak_burst": burst, "unit": "TFLOP/s",
                         "frac": (achieved / sustained) if achieved else None,
                         "frac_of_burst": (achieved / burst) if achieved else None,
                         "traffic": traffic_of(names[dom])[0], "traffic_launch": traffic_of(names[dom])[1],
                         "classes": {names[c]: {"ms": cls_ms[c], "tflops": (cls_fl[c] / cls_ms[c] / 1e9)
                                                if cls_ms[c] else None, "launches": cls_n[c]} for c in range(3)}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": int(tokens.nbytes),
                    "d2h_bytes_per_step": 8},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
