#!/usr/bin/env python
"""Seq1F1B training-step benchmark (B200, sm_100a engine).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg2|cfg3-stage|cfg4-stage]

Default workload (BASELINE.json configs[1]): GPT-2.7B (h 2560,
L 32, 32 heads x 80, FFN 4h, vocab 50257, learned positions), seq 32K split into
k = 4 computation-balanced (cwp) sub-sequences, M = 8 micro-batches, Seq1F1B,
bf16 with fp32 masters/grads and an AdamW step, random-init weights, synthetic
tokens. Pipeline depth = GPU count (one stage per rank, NCCL P2P between stages).
`--workload cfg3-stage|cfg4-stage` runs one pipeline stage of SURVEY cfg-3
(LLaMA-7B, 64K, k 8, 4 of 32 layers) / cfg-4 (GPT-13B, 128K, k 16, 5 of 40 layers)
on one GPU with the full config's partition (reported separately, not the headline).

One JSON line on rank 0:
  value     tokens/s with the step's tokens resident in HBM, device time of K steps
            (CUDA events on the engine stream), max over ranks; no kernel probes.
  e2e       the same K steps through the public C-ABI (sp_engine_step) with host
            tokens in pinned memory: host wall clock around each call, which includes
            the H2D copy of the tokens and the D2H read of the loss; max over ranks.
  roofline  per kernel class from a separate, untimed probe step (CUDA events around
            every GEMM / attention launch on the stream it is launched on).
  cpu_baseline  the reference's own CPU path on this config (oracle/_ref: the unmodified
            reference core's cwp_partition + generate + simulate + check_schedule, best of
            20, one thread), with the builder's numpy oracle sample labelled beside it.
`--impl reference` runs only oracle/_ref (planning) and the numpy oracle (a bounded,
FLOP-scaled execution sample of the same config) on the host cores; it never loads
libseqpipe_b200.so.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tokens/sec (8×B200, 32K seq) vs roofline; bubble ratio; peak activation GB/stage"
GPT, LLAMA = 0, 1

WORKLOADS = {
    "cfg2": dict(desc="GPT-2.7B seq 32K, 4 sub-sequences (cwp), Seq1F1B, pipeline depth = GPU count",
                 model="gpt-2.7b", family=GPT, preset="gpt-2.7b", h=2560, L=32, H=32, hd=80, F=4 * 2560, V=50257,
                 seq=32768, k=4, stage_layers=None),
    "cfg3-stage": dict(desc="one stage of cfg-3: LLaMA-7B (RMSNorm, RoPE, SwiGLU 11008, 32 x 128 heads) seq 64K, "
                            "8 sub-sequences, 4 of 32 layers (stage of an 8-stage pipeline) on one GPU",
                       model="llama-7b", family=LLAMA, preset="gpt-7b", h=4096, L=32, H=32, hd=128, F=11008,
                       V=32000, seq=65536, k=8, stage_layers=4, pipeline=8),
    "cfg4-stage": dict(desc="one stage of cfg-4: GPT-13B (40 x 128 heads, FFN 4h) seq 128K, 16 sub-sequences, "
                            "5 of 40 layers (stage of an 8-stage pipeline) on one GPU, no recomputation",
                       model="gpt-13b", family=GPT, preset="gpt-13b", h=5120, L=40, H=40, hd=128, F=4 * 5120,
                       V=50257, seq=131072, k=16, stage_layers=5, pipeline=8),
}


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
        d = json.loads((ROOT / "profiles" / "r2_traffic.json").read_text())[kernel]
        return d["dram_bytes_per_launch"], d["launch"]
    except Exception:
        return None, None


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def default_micro(w, n_gpus):
    if WORKLOADS[w]["stage_layers"]:
        return 2
    return 8 if n_gpus <= 4 else 2 * n_gpus


def scenario_overrides(w, n_gpus, micro, k, seq):
    """(preset, overrides) of the reference ScenarioConfig for this run."""
    W = WORKLOADS[w]
    P = W.get("pipeline", n_gpus)
    return W["preset"], [("pipeline_size", P), ("seq_len", seq), ("segments", k), ("micro_batches", micro)]


def flops_per_step(W, layers, micro, lengths, head=True):
    """Algorithmic FLOPs: per segment F = 2*N*n + 4*L*h*n*(prefix + n/2)
    (+ LM head 2*V*h*n), B = 2F; times M micro-batches."""
    h, F, V = W["h"], W["F"], W["V"]
    per_layer = 4 * h * h + (3 if W["family"] == LLAMA else 2) * h * F
    tot, pre = 0.0, 0
    for n in lengths:
        f = 2 * layers * per_layer * n + 4 * layers * h * n * (pre + n / 2) + (2 * V * h * n if head else 0)
        tot += 3 * f
        pre += n
    return tot * micro


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
        sm, mx, reasons, pw = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------------------------------
# CPU legs: the compiled reference planner (oracle/_ref) and the builder's numpy oracle.
# Test infrastructure: only these legs of bench.py touch oracle/.

def ref_scenario(w, n_gpus, micro, k, seq):
    """The ScenarioConfig built by the REFERENCE's own preset/override code (oracle/_ref)."""
    from oracle import ref
    preset, ov = scenario_overrides(w, n_gpus, micro, k, seq)
    cfg = ref.preset_scenario(preset)
    for key, v in ov:
        cfg = ref.apply_scenario_override(cfg, key, str(v))
    ref.validate(cfg)
    return cfg


def reference_planner(cfg, kind, mode, reps=20):
    """Best-of-reps ns of the reference's CPU path for one step of this config: cwp_partition +
    generate + simulate + check_schedule (partition.cpp:157-207, schedule.cpp:313-349,
    sim.cpp:121-317, validate.cpp:85-258), one thread (the reference has none)."""
    from oracle import ref
    return ref.time_planner(cfg, kind, mode, reps)


def oracle_sample(W, budget_s=None):
    """Bounded CPU execution sample with the builder's numpy fp64 oracle (oracle/transformer.py):
    forward + backward of ONE layer of the workload's width (h, heads, FFN, family) on a
    1024-token sequence in two segments (vocab 512 head), all host cores (BLAS threads).
    Returns (FLOP/s, sample FLOPs, seconds, description)."""
    from oracle.transformer import Model
    h, H, F, n = W["h"], W["H"], W["F"], 1024
    fup = 2 * F if W["family"] == LLAMA else F
    rng = np.random.default_rng(0)
    p = {"embed": rng.normal(0, .02, (512, h)), "final_norm": np.ones((1, h)),
         "lm_head": rng.normal(0, .02, (512, h)), "layer0.norm1": np.ones((1, h)), "layer0.norm2": np.ones((1, h)),
         "layer0.wqkv": rng.normal(0, .02, (3 * h, h)), "layer0.wo": rng.normal(0, .02, (h, h)),
         "layer0.w1": rng.normal(0, .02, (fup, h)), "layer0.w2": rng.normal(0, .02, (h, F))}
    if W["family"] == GPT:
        p["pos"] = rng.normal(0, .02, (n, h))
    m = Model(W["family"], 512, h, 1, H, W["hd"], F)
    tok = rng.integers(0, 512, size=(1, n + 1)).astype(np.int32)
    per_layer = 4 * h * h + (3 if W["family"] == LLAMA else 2) * h * F
    fl = 3 * (2 * per_layer * n + 4 * h * 512 * (0 + 256) + 4 * h * 512 * (512 + 256) + 2 * 512 * h * n)
    t0 = time.perf_counter()
    m.step(p, tok, [512, 512])
    el = time.perf_counter() - t0
    desc = (f"builder's numpy fp64 oracle (NOT the reference): fwd+bwd of 1 {W['model']} layer on 1024 tokens "
            f"(2 segments), {el:.2f} s, {os.cpu_count()} host threads; extrapolated to the step by FLOPs")
    return fl / el, fl, el, desc


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path on the host cores. Planning
    through the compiled, unmodified reference core (oracle/_ref); the reference has no tensor
    numerics, so each step adds a bounded execution sample of the same config with the numpy oracle
    port, FLOP-scaled to tokens. libseqpipe_b200.so is never loaded here."""
    if rank != 0:
        return 0
    from oracle import ref
    W = WORKLOADS[args.workload]
    cfg = ref_scenario(args.workload, args.gpus, args.micro, args.k, args.seq)
    part = ref.partition_for(cfg, args.partition)
    layers = W["stage_layers"] or W["L"]
    tokens = cfg.micro_batches * cfg.seq_len
    step_fl = flops_per_step(W, layers, cfg.micro_batches, part.lengths)
    times, eq_tokens, plan_ns = [], [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        pns = reference_planner(cfg, args.kind, args.partition, reps=1)
        rate, sfl, _, desc = oracle_sample(W)
        el = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(el)
            eq_tokens.append(tokens * sfl / step_fl)
            plan_ns.append(pns)
    ms = statistics.mean(times) * 1e3
    value = sum(eq_tokens) / sum(times)
    maps = Path(f"/proc/{os.getpid()}/maps").read_text() if Path(f"/proc/{os.getpid()}/maps").exists() else ""
    loaded = sorted({ln.split()[-1] for ln in maps.splitlines() if ln.endswith(".so") and str(ROOT) in ln})
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(args, cfg.micro_batches, cfg.seq_len, cfg.segments, part.lengths),
            "step_is_sample": True,
            "tokens_per_step_equiv": statistics.mean(eq_tokens),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                             "sample": f"per step: oracle/_ref planner (cwp+generate+simulate+check_schedule, "
                                       f"{statistics.mean(plan_ns) / 1e6:.3f} ms) + {desc}",
                             "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "repo_libraries_loaded": loaded,
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def stage1_budget(W, preset, args, E, pl):
    """Stage 1 of the workload's full pipeline (P = W["pipeline"], M = 2P): does it fit one B200?
    HBM of the stage = weights + grads + AdamW m/v (fp32) + bf16 compute copy (18 B/param; stage 1
    also holds the token / position embeddings) + the fp32 dK/dV accumulator + the activation arena
    (engine plan, offline-placed; sp_plan_memory) + per-op workspaces. If it does not fit, the plan
    that does: recompute the MLP up-projection output u in B instead of storing it (u is the largest
    per-token field of a record), priced in extra FLOPs."""
    import torch
    P = W["pipeline"]
    M = 2 * P
    h, F, L, V = W["h"], W["F"], W["L"], W["V"]
    c = pl.preset_scenario(preset)
    for key, v in (("pipeline_size", P), ("seq_len", args.seq), ("segments", args.k), ("micro_batches", M)):
        pl.apply_scenario_override(c, key, str(v))
    part = pl.partition_for(c, args.partition)

    def model(flags):
        m = E.ModelConfig(family=W["family"], dtype=E.BF16, vocab=V, hidden=h, layers=L, heads=W["H"],
                          head_dim=W["hd"], ffn=F, max_seq=args.seq)
        m.flags = flags
        return m
    live, arena, dkv = E.plan_memory(c, "seq1f1b", part, model(0), stage=1)
    live_nou, arena_nou, _ = E.plan_memory(c, "seq1f1b", part, model(E.FLAG_RECOMPUTE_MLP), stage=1)
    fup = 2 * F if W["family"] == LLAMA else F
    per_layer = 4 * h * h + (3 if W["family"] == LLAMA else 2) * h * F + 4 * h
    params = (L // P) * per_layer + V * h + (args.seq * h if W["family"] == GPT else 0)
    weights = 18 * params
    n = max(part.lengths)
    ws = 2 * n * (h + 2 * fup + 6 * h) + 4 * n * h + 8 * n * W["H"]
    cap = torch.cuda.mem_get_info(0)[1] if torch.cuda.is_available() else 180e9
    total = weights + dkv + arena + ws
    total_rc = weights + dkv + arena_nou + ws + 2 * n * fup  # + the recomputed-u workspace
    n_tok = sum(part.lengths)
    layer_fl = 2 * n_tok * per_layer  # forward GEMM FLOPs of a layer over the sequence (approx.)
    extra = 2 * n_tok * h * fup / (3 * layer_fl)
    gb = 1e9
    return {"pipeline": P, "micro_batches": M, "segments": args.k, "partition": args.partition,
            "weights_optimizer_gb": weights / gb, "dkv_accumulator_gb": dkv / gb, "arena_gb": arena / gb,
            "live_activation_peak_gb": live / gb, "workspaces_gb": ws / gb, "total_gb": total / gb,
            "device_capacity_gb": cap / gb, "fits": total <= cap,
            "if_oom_plan": None if total <= cap else {
                "recompute": "SP_FLAG_RECOMPUTE_MLP: the MLP up-projection output u is not kept in the (m,s) "
                             "record and is recomputed in B (one extra [n,h]x[h,Fup] GEMM per layer); engine "
                             "plan (sp_plan_memory) with the flag",
                "arena_gb": arena_nou / gb, "live_activation_peak_gb": live_nou / gb, "total_gb": total_rc / gb,
                "fits": total_rc <= cap, "extra_gemm_flops_frac": extra}}


def config_of(args, micro, seq, k, lengths):
    W = WORKLOADS[args.workload]
    return {"workload": W["desc"], "model": W["model"], "global_batch": micro, "seq_len": seq, "segments": k,
            "partition": list(lengths), "partition_mode": args.partition, "schedule": args.kind,
            "parallelism": f"pp{args.gpus}" if not W["stage_layers"] else f"stage of pp{W['pipeline']} on 1 GPU",
            "layers_on_gpu": W["stage_layers"] or W["L"],
            "recompute": "mlp-up (SP_FLAG_RECOMPUTE_MLP)" if getattr(args, "recompute_mlp", False) else "none",
            "l2": "inputs larger than L2 (weights + activations >> 126 MB per step)"}


# ---------------------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--seq", type=int, default=0)
    ap.add_argument("--micro", type=int, default=0, help="micro-batches (default 8, 2P when P > 4; 2 for stages)")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--kind", default="seq1f1b")
    ap.add_argument("--partition", default="cwp", choices=["cwp", "even"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", type=int, default=1, help="replay the step as a captured CUDA graph (P = 1)")
    ap.add_argument("--recompute-mlp", action="store_true", help="SP_FLAG_RECOMPUTE_MLP (recompute u in B)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1: NCCL P2P, or the peer-memory transport (CUDA IPC rings over NVLink)")
    args = ap.parse_args()
    W = WORKLOADS[args.workload]
    args.seq = args.seq or W["seq"]
    args.k = args.k or W["k"]
    args.micro = args.micro or default_micro(args.workload, args.gpus)
    if W["stage_layers"] and args.gpus != 1:
        print(json.dumps({"error": "stage workloads run on one GPU"}))
        return 2

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

    preset, ov = scenario_overrides(args.workload, args.gpus, args.micro, args.k, args.seq)
    full = pl.preset_scenario(preset)
    for key, v in ov:
        pl.apply_scenario_override(full, key, str(v))
    full.validate()
    part_full = pl.partition_for(full, args.partition) if args.k > 1 else pl.even_partition(full)
    layers = W["stage_layers"] or W["L"]
    model = E.ModelConfig(family=W["family"], dtype=E.BF16, vocab=W["V"], hidden=W["h"], layers=layers,
                          heads=W["H"], head_dim=W["hd"], ffn=W["F"], max_seq=args.seq, seed=42, lr=1e-4,
                          weight_decay=0.0)
    if W["stage_layers"]:  # one stage on one GPU: the engine runs P = 1 over the stage's layers
        cfg = pl.ScenarioConfig(pipeline_size=1, micro_batches=args.micro, segments=args.k, seq_len=args.seq,
                                layers=layers, hidden_dim=W["h"], param_count=model.param_count())
        part = pl.make_partition(part_full.lengths, cfg)
    else:
        cfg, part = full, part_full
    model.flags = E.FLAG_TIMELINE | (E.FLAG_RECOMPUTE_MLP if args.recompute_mlp else 0)
    import torch  # device / pinned memory plumbing only
    n_dev = torch.cuda.device_count()
    # One GPU per rank. Fewer GPUs than ranks (a functional check of the N > 1 path on a
    # smaller box, --transport ipc) puts several ranks on one device and says so in the line.
    local = local % n_dev if n_dev else local
    shared_gpu = world > 1 and n_dev < world
    eng = E.Engine(cfg, args.kind, part, model, rank=rank, world_size=world, cuda_device=local)
    if world > 1 and args.transport == "ipc":
        blobs = [None] * world
        dist.all_gather_object(blobs, eng.ipc_export())
        eng.ipc_connect(blobs)
    elif world > 1:
        n_ids = eng.comm_channels()
        ids = [E.nccl_unique_id() for _ in range(n_ids)] if rank == 0 else [None] * n_ids
        dist.broadcast_object_list(ids, src=0)
        eng.comm_init(ids)

    T = cfg.seq_len
    rng = np.random.default_rng(1234)
    tokens = rng.integers(0, model.vocab, size=(cfg.micro_batches, T + 1), dtype=np.int64).astype(np.int32)
    tok_t = torch.from_numpy(tokens).to(f"cuda:{local}")
    tok_ptr = tok_t.data_ptr()
    tok_pinned = torch.from_numpy(tokens).pin_memory()
    tok_host = tok_pinned.numpy()  # host view of the pinned buffer (sp_engine_step copies it H2D)
    from paper_2406_03488_b200 import _capi
    lib = _capi.lib()

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

    for i in range(args.warmup):
        eng.step(tok_ptr, on_device=True)
        if i == 0 and args.graph and world == 1:
            eng.enable_graph(True)  # capture the step once (after one eager step), replay from then on

    # ---- timed: tokens resident in HBM, no probes; device time of each step (CUDA events)
    barrier()
    reps = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            reps.append(eng.step(tok_ptr, on_device=True))
        barrier()
    step_ms = max_over_ranks(sum(r.step_ms for r in reps) / len(reps))
    # ---- timed e2e: host tokens (pinned) through the public C-ABI, loss read back; host wall clock
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = eng.step(tok_host, on_device=False)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    barrier()
    e2e_step = max_over_ranks(sum(e2e_ms) / len(e2e_ms))
    loss_last = r.loss
    if dist:  # the loss lives on the last stage's rank; the others report 0
        t = torch.tensor([loss_last], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        loss_last = float(t.item())
    # ---- untimed probe step: per-class kernel times for the roofline
    eng.set_flags(model.flags | E.FLAG_KPROBE)
    probe = eng.step(tok_ptr, on_device=True)
    eng.set_flags(model.flags)
    mem = eng.memory()

    tok_per_step = cfg.micro_batches * T
    value = tok_per_step / (step_ms / 1e3)
    e2e = tok_per_step / (e2e_step / 1e3)
    last = reps[-1]
    fl = flops_per_step(W, layers, cfg.micro_batches, part.lengths)
    burst, sustained, hbm, src = peaks()
    bubble = max_over_ranks(statistics.mean(r.bubble_ratio for r in reps))
    peak_act = max_over_ranks(last.peak_activation_bytes) / 1e9
    launches = int(sum(r.kernel_launches for r in reps))

    cls_ms = [probe.class_ms[c] for c in range(3)]
    cls_fl = [probe.class_flops[c] for c in range(3)]
    cls_n = [probe.class_launches[c] for c in range(3)]
    dom = int(np.argmax(cls_ms))
    names = ["gemm_tcgen05", "attention_fwd", "attention_bwd"]
    achieved = cls_fl[dom] / (cls_ms[dom] / 1e3) / 1e12 if cls_ms[dom] > 0 else None

    modeled, memory_model = {}, {}
    try:
        rep_m = pl.simulate(pl.generate(full, args.kind, part_full), part_full, with_series=False)
        modeled = {"bubble_ratio": float(rep_m.aggregate_bubble_ratio), "peak_tokens": float(rep_m.max_peak_memory),
                   "pipeline_size": full.pipeline_size}
    except Exception as e:  # pragma: no cover
        modeled = {"error": str(e)}
    # Engine arena plan (host replay of each schedule's op order, KV-prefix slabs included) for
    # Seq1F1B vs batch-level 1F1B of the same model at several pipeline depths, stage 1.
    full_model = E.ModelConfig(family=W["family"], dtype=E.BF16, vocab=W["V"], hidden=W["h"], layers=W["L"],
                               heads=W["H"], head_dim=W["hd"], ffn=W["F"], max_seq=args.seq)
    for P in sorted({full.pipeline_size, 4, 8}):
        try:
            Mp = full.micro_batches if P == full.pipeline_size else (8 if P <= 4 else 2 * P)
            cs, c1 = pl.preset_scenario(preset), pl.preset_scenario(preset)
            for c, kk in ((cs, args.k), (c1, 1)):
                for key, v in (("pipeline_size", P), ("seq_len", args.seq), ("segments", kk), ("micro_batches", Mp)):
                    pl.apply_scenario_override(c, key, str(v))
            ps, p1 = pl.partition_for(cs, args.partition), pl.even_partition(c1)
            ls, _, dkv = E.plan_memory(cs, "seq1f1b", ps, full_model, stage=1)
            l1, _, _ = E.plan_memory(c1, "1f1b", p1, full_model, stage=1)
            rs = pl.simulate(pl.generate(cs, "seq1f1b", ps), ps, with_series=False)
            rb = pl.simulate(pl.generate(c1, "1f1b", p1), p1, with_series=False)
            memory_model[f"P{P}_M{Mp}"] = {
                "seq1f1b_peak_activation_gb_stage1": ls / 1e9, "1f1b_peak_activation_gb_stage1": l1 / 1e9,
                "ratio": ls / l1 if l1 else None, "dkv_accumulator_gb": dkv / 1e9,
                "seq1f1b_modeled_bubble": float(rs.aggregate_bubble_ratio),
                "1f1b_modeled_bubble": float(rb.aggregate_bubble_ratio)}
        except Exception as e:  # pragma: no cover
            memory_model[f"P{P}"] = {"error": str(e)}

    stage1 = stage1_budget(W, preset, args, E, pl) if W["stage_layers"] else None

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            rcfg = ref_scenario(args.workload, args.gpus, args.micro, args.k, args.seq)
            ns = reference_planner(rcfg, args.kind, args.partition, reps=20)
            rate, sfl, el, desc = oracle_sample(W)
            cpu = {"value": tok_per_step / (ns / 1e9), "unit": "tokens/s", "cores": 1, "kind": "reference",
                   "sample": "oracle/_ref = the unmodified reference core: cwp_partition + generate + simulate + "
                             "check_schedule of this config (the reference's whole CPU path: it schedules and "
                             "models the step, it has no tensor numerics), best of 20, 1 thread; value = tokens "
                             "of the step / that time",
                   "planner_ms": ns / 1e6, "nproc": os.cpu_count(), "cpu_model": cpu_model(),
                   "builder_oracle": {"value": rate / (fl / tok_per_step), "unit": "tokens/s",
                                      "cores": os.cpu_count(), "kind": "port", "sample": desc}}
        except Exception as e:  # pragma: no cover
            cpu = {"error": f"reference CPU leg unavailable: {e}"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, seed 1234; random-init weights)",
            "config": config_of(args, cfg.micro_batches, T, cfg.segments, part.lengths),
            "loss": loss_last,
            "graph": bool(args.graph and world == 1),
            **({"transport": args.transport} if world > 1 else {}),
            **({"shared_gpu": f"{world} ranks on {n_dev} GPU(s): functional check, not a scaling number"}
               if shared_gpu else {}),
            "tflops_per_gpu": fl / (step_ms / 1e3) / 1e12 / args.gpus,
            "model_flops_frac_of_peak": fl / (step_ms / 1e3) / 1e12 / args.gpus / sustained,
            "bubble_ratio": bubble, "modeled": modeled,
            "peak_activation_gb_per_stage": peak_act,
            "device_memory_gb": {"engine_allocated": mem[0] / 1e9, "device_free": mem[1] / 1e9,
                                 "activation_arena": last.arena_bytes / 1e9},
            "memory_model": memory_model,
            **({"stage1_budget_full_pipeline": stage1} if stage1 else {}),
            "roofline": {"bound": "tensor", "kernel": names[dom], "achieved": achieved, "peak": sustained,
                         "peak_kind": f"bf16 sustained ({src})", "peak_burst": burst, "unit": "TFLOP/s",
                         "frac": (achieved / sustained) if achieved else None,
                         "frac_of_burst": (achieved / burst) if achieved else None,
                         "measured_in": "separate untimed probe step (events on each kernel's own stream)",
                         "traffic": traffic_of(names[dom])[0], "traffic_launch": traffic_of(names[dom])[1],
                         "classes": {names[c]: {"ms": cls_ms[c], "tflops": (cls_fl[c] / cls_ms[c] / 1e9)
                                                if cls_ms[c] else None, "launches": cls_n[c],
                                                "share_of_step": cls_ms[c] / probe.step_ms if probe.step_ms else None}
                                     for c in range(3)}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": int(tokens.nbytes),
                    "d2h_bytes_per_step": 8, "timing": "host wall clock around sp_engine_step, pinned host tokens"},
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
