"""End-to-end parity of the sm_100a Seq1F1B engine on one B200.

Every pipeline stage of the config runs in one process on cuda:0 (stage
hand-offs are device-local), executing the op tables of seqpipe::generate in a
dependency-respecting order. Checked against
  * the compiled reference planner (oracle/_ref): the executed op log is
    bit-identical to the reference generate() and passes check_schedule;
  * the CPU fp64 oracle (oracle/transformer.py): loss and every parameter
    gradient within relative L2 1e-5 (fp32 validation mode) / 2e-2 (bf16).
"""
import numpy as np
import pytest

from oracle import ref
from oracle.transformer import GPT, LLAMA, Model, rel_l2, tokens_for
from paper_2406_03488_b200 import engine as E
from paper_2406_03488_b200 import planner as pl

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5   # north star: relative L2 <= 1e-5 in the fp32 validation mode
TOL_BF16 = 2e-2  # north star: relative L2 <= 2e-2 in the bf16 production mode


def tiny_model(family=GPT, dtype=E.F32, vocab=512, layers=8, hidden=256, heads=4, ffn=1024, max_seq=2048):
    return E.ModelConfig(family=family, dtype=dtype, vocab=vocab, hidden=hidden, layers=layers, heads=heads,
                         head_dim=hidden // heads, ffn=ffn, max_seq=max_seq, seed=42)


def scenario(model, P=4, M=5, k=4, T=2048):
    cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=M, segments=k, seq_len=T, layers=model.layers,
                            hidden_dim=model.hidden, param_count=model.param_count())
    cfg.validate()
    return cfg


def run(model, cfg, kind="seq1f1b", mode="cwp", seed=1234):
    part = pl.partition_for(cfg, mode)
    eng = E.Engine(cfg, kind, part, model)
    tok = tokens_for(cfg.micro_batches, cfg.seq_len, model.vocab, seed=seed)
    rep = eng.step(tok)
    return eng, part, tok, rep


def oracle_of(model):
    return Model(model.family, model.vocab, model.hidden, model.layers, model.heads, model.head_dim, model.ffn,
                 eps=model.norm_eps, theta=model.rope_theta)


def compare(eng, model, part, tok, rep, tol):
    params = {n: eng.read_param(n) for n in eng.params()}
    loss, grads = oracle_of(model).step(params, tok, part.lengths)
    assert abs(rep.loss - loss) / abs(loss) < tol, (rep.loss, loss)
    worst = {}
    for name in params:
        g = eng.read_grad(name)
        worst[name] = rel_l2(g, grads[name])
    bad = {k: v for k, v in worst.items() if v > tol}
    assert not bad, bad
    return worst


def test_executed_op_log_is_reference_schedule(gpu):
    model = tiny_model(layers=4, hidden=128, heads=2, ffn=256, vocab=256, max_seq=512)
    cfg = scenario(model, P=4, M=6, k=4, T=512)
    eng, part, tok, rep = run(model, cfg)
    log = eng.op_log()
    want = ref.generate(cfg, "seq1f1b", part)
    assert log.device_orders == want.device_orders
    assert pl.check_schedule(log) == []
    assert ref.check_schedule(log) == []
    assert rep.ops_executed == sum(len(o) for o in want.device_orders)


def test_fp32_validation_tiny_gpt_cfgT(gpu):
    """cfg-T: tiny GPT (h256, L8, 4 stages, T=2K, k=4), fp32 validation mode."""
    model = tiny_model()
    cfg = scenario(model, P=4, M=5, k=4, T=2048)
    eng, part, tok, rep = run(model, cfg)
    assert part.lengths == ref.partition_for(cfg, "cwp").lengths
    compare(eng, model, part, tok, rep, TOL_F32)


def test_fp32_validation_llama(gpu):
    model = tiny_model(family=LLAMA, layers=4, hidden=256, heads=4, ffn=384, vocab=384)
    cfg = scenario(model, P=2, M=3, k=4, T=1024)
    eng, part, tok, rep = run(model, cfg)
    compare(eng, model, part, tok, rep, TOL_F32)


@pytest.mark.parametrize("kind,k", [("1f1b", 1), ("gpipe", 2), ("1f1b", 3)])
def test_fp32_batch_level_kinds(gpu, kind, k):
    model = tiny_model(layers=4, hidden=128, heads=2, ffn=512, vocab=256, max_seq=512)
    cfg = scenario(model, P=2, M=3, k=k, T=512)
    eng, part, tok, rep = run(model, cfg, kind=kind, mode="even")
    compare(eng, model, part, tok, rep, TOL_F32)


def test_bf16_production_tiny_gpt(gpu):
    model = tiny_model(dtype=E.BF16)
    cfg = scenario(model, P=4, M=5, k=4, T=2048)
    eng, part, tok, rep = run(model, cfg)
    compare(eng, model, part, tok, rep, TOL_BF16)


def test_bf16_production_llama_hd128(gpu):
    model = tiny_model(family=LLAMA, dtype=E.BF16, layers=2, hidden=256, heads=2, ffn=512, vocab=512)
    cfg = scenario(model, P=2, M=3, k=4, T=1024)
    eng, part, tok, rep = run(model, cfg)
    compare(eng, model, part, tok, rep, TOL_BF16)


def test_seq1f1b_equals_1f1b_numerics(gpu):
    """Splitting the sequence must not change the step (split == unsplit)."""
    model = tiny_model(layers=4, hidden=128, heads=2, ffn=512, vocab=256, max_seq=1024)
    cfg4 = scenario(model, P=2, M=3, k=4, T=1024)
    cfg1 = scenario(model, P=2, M=3, k=1, T=1024)
    e4, p4, t4, r4 = run(model, cfg4)
    e1, p1, t1, r1 = run(model, cfg1, kind="1f1b", mode="even")
    assert abs(r4.loss - r1.loss) / abs(r1.loss) < 1e-6
    for n in e4.params():
        assert rel_l2(e4.read_grad(n), e1.read_grad(n)) < 1e-5, n


def test_step_report_and_memory(gpu):
    model = tiny_model(dtype=E.BF16, layers=4, hidden=256, heads=4, ffn=1024, vocab=512)
    cfg = scenario(model, P=4, M=8, k=4, T=2048)
    eng, part, tok, rep = run(model, cfg)
    assert rep.step_ms > 0 and rep.busy_ms > 0 and 0 <= rep.bubble_ratio < 1
    assert rep.peak_activation_bytes > 0 and rep.arena_bytes >= rep.peak_activation_bytes
    cfg1 = scenario(model, P=4, M=8, k=1, T=2048)
    e1, p1, t1, r1 = run(model, cfg1, kind="1f1b", mode="even")
    # Seq1F1B keeps fewer tokens resident than batch-level 1F1B (SPEC criterion 4)
    assert rep.peak_activation_bytes < r1.peak_activation_bytes


def test_optimizer_step_changes_weights(gpu):
    model = tiny_model(dtype=E.BF16, layers=2, hidden=128, heads=2, ffn=256, vocab=256, max_seq=512)
    model.lr = 1e-3
    cfg = scenario(model, P=2, M=3, k=2, T=512)
    part = pl.partition_for(cfg, "cwp")
    eng = E.Engine(cfg, "seq1f1b", part, model)
    w0 = eng.read_param("layer0.wqkv")
    tok = tokens_for(3, 512, 256)
    l1 = eng.step(tok).loss
    w1 = eng.read_param("layer0.wqkv")
    assert not np.allclose(w0, w1)
    for _ in range(3):
        l2 = eng.step(tok).loss
    assert l2 < l1


def test_measured_report_and_executed_schedule_json(gpu):
    """(f3) wire formats on the engine: the executed op log as seqpipe.schedule.v1 (read back
    by the compiled reference, byte-identical to the planned schedule's document) and the
    measured step as seqpipe.simreport.v1 (ns times, sim.cpp metric definitions)."""
    import json

    model = tiny_model(layers=4, hidden=128, heads=2, ffn=256, vocab=256, max_seq=512)
    model.flags = E.FLAG_TIMELINE
    cfg = scenario(model, P=4, M=6, k=4, T=512)
    eng, part, tok, rep = run(model, cfg)
    log = eng.op_log()
    text = pl.schedule_to_json(log)
    assert text == pl.schedule_to_json(ref.generate(cfg, "seq1f1b", part))
    assert ref.schedule_json_roundtrip(text) == text
    doc = json.loads(eng.report_json())
    assert doc["schema"] == "seqpipe.simreport.v1" and doc["kind"] == "seq1f1b"
    assert doc["partition"] == part.lengths
    modeled = json.loads(ref.report_to_json(ref.generate(cfg, "seq1f1b", part), part))
    for dev, mod in zip(doc["devices"], modeled["devices"]):
        tasks = dev["tasks"]
        assert [(t["kind"], t["m"], t["s"]) for t in tasks] == [(t["kind"], t["m"], t["s"]) for t in mod["tasks"]]
        assert all(int(t["end"]) >= int(t["start"]) >= 0 for t in tasks)
        first, last, busy = int(dev["first_start"]), int(dev["last_end"]), int(dev["busy"])
        assert busy <= last - first + len(tasks)  # ns rounding per task
        num, _, den = dev["bubble_ratio"].partition("/")
        assert 0 <= int(num) / int(den or 1) <= 1
        assert dev["warmup_forward_tasks"] == mod["warmup_forward_tasks"]
        assert dev["peak_allocations"] == mod["peak_allocations"]
        assert int(dev["peak_memory"].split("/")[0]) > 0
    # the measured timeline through the reference renderers' rules (render.cpp:46-124)
    txt = eng.render_gantt("ascii", 100)
    rows = txt.splitlines()
    assert rows[0].startswith("kind=seq1f1b makespan=") and len(rows) == 1 + cfg.pipeline_size
    assert all(r.startswith(f"device {d + 1} |") and len(r) == len(f"device {d + 1} |") + 101
               for d, r in enumerate(rows[1:]))
    assert all(set(r.split("|")[1]) & {"F", "B"} for r in rows[1:])
    svg = eng.render_gantt("svg")
    assert svg.count('stroke="#ffffff"') == sum(len(o) for o in log.device_orders) and svg.endswith("</svg>\n")
    eng.close()


@pytest.mark.parametrize("kind,k,dtype,tol", [("zb1p", 1, E.F32, TOL_F32), ("seqzb1p", 4, E.F32, TOL_F32),
                                              ("seqzb1p", 4, E.BF16, TOL_BF16)])
def test_zero_bubble_input_weight_split(gpu, kind, k, dtype, tol):
    """(f2) SeqZB1P / ZB1P: the engine executes the reference's I / W op tables
    (schedule.cpp:217-309, W placed in idle gaps by simulate()) -- I = backward without
    the weight-gradient GEMMs, W = those GEMMs from the operands I saved -- and the step
    matches the CPU oracle; the executed log is the reference's and passes its checker."""
    model = tiny_model(dtype=dtype, layers=4, hidden=128, heads=2, ffn=256, vocab=256, max_seq=512)
    cfg = scenario(model, P=2, M=3, k=k, T=512)
    eng, part, tok, rep = run(model, cfg, kind=kind, mode="cwp" if k > 1 else "even")
    log = eng.op_log()
    assert log.device_orders == ref.generate(cfg, kind, part).device_orders
    assert ref.check_schedule(log) == []
    assert sum(1 for o in log.device_orders for t in o if t.kind == "W") == cfg.micro_batches * k * cfg.pipeline_size
    compare(eng, model, part, tok, rep, tol)
    eng.close()



def test_zero_bubble_deep_pipeline_no_record_reuse_race(gpu):
    """SeqZB1P at P=4 M=8 k=4 (even partition): W(m,s,v) runs after W(m,s,v-1) on this
    schedule, so stage v's layer-0 input must not alias stage v-1's (freed, reused) output
    record. fp32 step vs the oracle catches any stale read."""
    model = tiny_model(layers=4, hidden=128, heads=2, ffn=256, vocab=256, max_seq=512)
    cfg = scenario(model, P=4, M=8, k=4, T=512)
    eng, part, tok, rep = run(model, cfg, kind="seqzb1p", mode="even")
    log = eng.op_log()
    assert log.device_orders == ref.generate(cfg, "seqzb1p", part).device_orders
    compare(eng, model, part, tok, rep, TOL_F32)
    eng.close()


def test_adamw_update_matches_formula(gpu):
    """One AdamW step (elementwise.cu adamw kernels) == the closed form at step 1:
    m = (1-b1) g, v = (1-b2) g^2, p -= lr ((m/bc1) / (sqrt(v/bc2) + eps) + wd p)."""
    model = tiny_model(dtype=E.BF16, layers=2, hidden=128, heads=2, ffn=256, vocab=256, max_seq=512)
    model.lr, model.weight_decay = 1e-3, 0.1
    cfg = scenario(model, P=2, M=3, k=2, T=512)
    eng = E.Engine(cfg, "seq1f1b", pl.partition_for(cfg, "cwp"), model)
    names = ["layer0.wqkv", "layer1.w2", "lm_head"] if "lm_head" in eng.params() else ["layer0.wqkv", "layer1.w2"]
    before = {n: eng.read_param(n).astype(np.float64) for n in names}
    eng.step(tokens_for(3, 512, 256))
    b1, b2, eps = model.beta1, model.beta2, model.adam_eps
    for n in names:
        g = eng.read_grad(n).astype(np.float64)
        p0 = before[n]
        m, v = (1 - b1) * g, (1 - b2) * g * g
        want = p0 - model.lr * ((m / (1 - b1)) / (np.sqrt(v / (1 - b2)) + eps) + model.weight_decay * p0)
        got = eng.read_param(n).astype(np.float64)
        assert np.max(np.abs(got - want)) < 1e-6, (n, np.max(np.abs(got - want)))
    eng.close()


@pytest.mark.parametrize("kind,k,mode", [("seq1f1b-i", 2, "cwp"), ("1f1b-i", 1, "even")])
def test_interleaved_kinds_execute_reference_order(gpu, kind, k, mode):
    """(f1) Seq1F1B-I / 1F1B-I: n_v = 2 stage chunks per device (V = 2P stages), executed
    in-process in the reference's interleaved order (schedule.cpp:128-215); the executed log
    is the reference generate() and the step matches the fp64 oracle (fp32 mode)."""
    model = tiny_model(layers=4, hidden=128, heads=2, ffn=256, vocab=256, max_seq=512)
    cfg = pl.ScenarioConfig(pipeline_size=2, stages_per_device=2, micro_batches=4, segments=k, seq_len=512,
                            layers=model.layers, hidden_dim=model.hidden, param_count=model.param_count())
    cfg.validate()
    eng, part, tok, rep = run(model, cfg, kind=kind, mode=mode)
    log = eng.op_log()
    assert log.device_orders == ref.generate(cfg, kind, part).device_orders
    assert ref.check_schedule(log) == []
    compare(eng, model, part, tok, rep, TOL_F32)
    eng.close()


def test_bf16_gpt_2p7b_width_hd80(gpu):
    """The production kernel mix at GPT-2.7B width (h 2560, 32 heads x 80, FFN 4h): tcgen05
    attention at head dim 80 with the side-stream dQ kernel, the first-op dK/dV store, the
    two-warp norm backward, vectorised CE, side-stream weight gradients -- one layer, bf16,
    against the fp64 oracle."""
    model = tiny_model(dtype=E.BF16, vocab=512, layers=1, hidden=2560, heads=32, ffn=4 * 2560, max_seq=512)
    cfg = scenario(model, P=1, M=2, k=2, T=512)
    eng, part, tok, rep = run(model, cfg)
    compare(eng, model, part, tok, rep, TOL_BF16)
    eng.close()


def test_bf16_engine_step_at_benchmarked_cfg2_shape(gpu):
    """One GPT-2.7B-width layer (h 2560, 32 x 80 heads, FFN 4h, vocab 50257) run through the
    engine exactly at the benchmarked sequence shape: T = 32768 split by the cfg-2 cwp partition
    [10170, 8496, 7428, 6674] (the gpt-2.7b preset with bench.py's overrides), bf16 production
    kernels, M = 1. Loss and every parameter gradient vs the fp64 oracle (run on the GPU through
    its torch backend, attention chunked over heads): relative L2 <= 2e-2."""
    import torch
    from oracle.transformer import TorchOps
    bench_cfg = pl.preset_scenario("gpt-2.7b")
    for k_, v_ in (("pipeline_size", "1"), ("seq_len", "32768"), ("segments", "4"), ("micro_batches", "8")):
        pl.apply_scenario_override(bench_cfg, k_, v_)
    lengths = pl.cwp_partition(bench_cfg).lengths
    assert lengths == [10170, 8496, 7428, 6674]
    model = E.ModelConfig(family=GPT, dtype=E.BF16, vocab=50257, hidden=2560, layers=1, heads=32, head_dim=80,
                          ffn=4 * 2560, max_seq=32768, seed=42)
    cfg = pl.ScenarioConfig(pipeline_size=1, micro_batches=1, segments=4, seq_len=32768, layers=1, hidden_dim=2560,
                            param_count=model.param_count())
    part = pl.make_partition(lengths, cfg)
    eng = E.Engine(cfg, "seq1f1b", part, model)
    tok = tokens_for(1, 32768, model.vocab, seed=1234)
    rep = eng.step(tok)
    params = {n: eng.read_param(n) for n in eng.params()}
    oracle = Model(GPT, model.vocab, model.hidden, 1, 32, 80, model.ffn, ops=TorchOps("cuda"), head_chunk=2)
    loss, grads = oracle.step(params, tok, lengths)
    del oracle
    torch.cuda.empty_cache()
    assert abs(rep.loss - loss) / abs(loss) < TOL_BF16, (rep.loss, loss)
    worst = {n: rel_l2(eng.read_grad(n), grads[n]) for n in params}
    bad = {k: v for k, v in worst.items() if v > TOL_BF16}
    assert not bad, (bad, worst)
    eng.close()


def test_bf16_engine_step_at_benchmarked_cfg3_shape(gpu):
    """One LLaMA-7B-width layer (h 4096, 32 x 128 heads, SwiGLU 11008, RoPE, RMSNorm, vocab 32000)
    through the engine at the cfg-3 sequence shape bench.py runs (`--workload cfg3-stage`):
    T = 65536 split by the gpt-7b preset's cwp partition into k = 8 sub-sequences, bf16
    production kernels (head dim 128: split dK/dV + dQ attention backward), M = 1. Loss and
    every parameter gradient vs the fp64 oracle (torch backend on the GPU, attention chunked
    over heads): relative L2 <= 2e-2."""
    import torch
    from oracle.transformer import TorchOps
    bench_cfg = pl.preset_scenario("gpt-7b")
    for k_, v_ in (("pipeline_size", "8"), ("seq_len", "65536"), ("segments", "8"), ("micro_batches", "2")):
        pl.apply_scenario_override(bench_cfg, k_, v_)
    lengths = pl.cwp_partition(bench_cfg).lengths
    assert sum(lengths) == 65536 and len(lengths) == 8
    model = E.ModelConfig(family=LLAMA, dtype=E.BF16, vocab=32000, hidden=4096, layers=1, heads=32, head_dim=128,
                          ffn=11008, max_seq=65536, seed=42)
    cfg = pl.ScenarioConfig(pipeline_size=1, micro_batches=1, segments=8, seq_len=65536, layers=1, hidden_dim=4096,
                            param_count=model.param_count())
    part = pl.make_partition(lengths, cfg)
    eng = E.Engine(cfg, "seq1f1b", part, model)
    tok = tokens_for(1, 65536, model.vocab, seed=1234)
    rep = eng.step(tok)
    params = {n: eng.read_param(n) for n in eng.params()}
    grads_eng = {n: eng.read_grad(n) for n in params}
    eng.close()
    torch.cuda.empty_cache()
    oracle = Model(LLAMA, model.vocab, model.hidden, 1, 32, 128, model.ffn, eps=model.norm_eps,
                   theta=model.rope_theta, ops=TorchOps("cuda"), head_chunk=2)
    loss, grads = oracle.step(params, tok, lengths)
    del oracle
    torch.cuda.empty_cache()
    assert abs(rep.loss - loss) / abs(loss) < TOL_BF16, (rep.loss, loss)
    worst = {n: rel_l2(grads_eng[n], grads[n]) for n in params}
    bad = {k: v for k, v in worst.items() if v > TOL_BF16}
    assert not bad, (bad, worst)


@pytest.mark.parametrize("family,hd,ffn,vocab", [(LLAMA, 128, 11008, 32000), (GPT, 80, 4 * 2560, 50257)])
def test_fast_loss_drop_is_memorisation_not_a_causal_leak(gpu, family, hd, ffn, vocab):
    """At the bench widths the loss on one fixed batch of uniform random tokens falls fast
    (cfg-3 stage: 11.2 -> 0.4 in six AdamW steps, tools/loss_curve.py): Adam's first steps move
    every weight of the h = 4096 matrices coherently. A causal model can only memorise such a
    batch -- if a query could see its own target (a mask or KV-slab offset leak), the drop would
    carry over to unseen tokens. So: train on batch A, then the loss of a fresh batch B (read
    before that step's update) must stay at or above ln V."""
    import math
    h = 4096 if family == LLAMA else 2560
    H = h // hd
    model = E.ModelConfig(family=family, dtype=E.BF16, vocab=vocab, hidden=h, layers=2, heads=H, head_dim=hd,
                          ffn=ffn, max_seq=8192, seed=42, lr=1e-4, weight_decay=0.0)
    cfg = pl.ScenarioConfig(pipeline_size=1, micro_batches=2, segments=4, seq_len=8192, layers=2, hidden_dim=h,
                            param_count=model.param_count())
    eng = E.Engine(cfg, "seq1f1b", pl.cwp_partition(cfg), model)
    tok_a = tokens_for(2, 8192, vocab, seed=3)
    tok_b = tokens_for(2, 8192, vocab, seed=4)
    losses = [eng.step(tok_a).loss for _ in range(6)]
    held_out = eng.step(tok_b).loss
    eng.close()
    assert losses[-1] < losses[0] - 0.5, losses  # it does fit the batch ...
    assert held_out > math.log(vocab) - 0.1, (held_out, losses)  # ... without predicting unseen tokens


@pytest.mark.parametrize("family", [GPT, LLAMA])
def test_recompute_mlp_is_bit_identical_and_smaller(gpu, family):
    """SP_FLAG_RECOMPUTE_MLP drops the MLP up-projection output u from every (m,s) record and
    recomputes it in B with the same GEMM on the same operands: the loss is identical, every
    gradient matches the default engine to fp32 accumulation-order noise, the activation plan
    is smaller, and the zero-bubble kinds (which keep the MLP operands for W) refuse the flag."""
    hd = 128 if family == LLAMA else 80
    h = 4 * hd
    ffn = 3 * h if family == LLAMA else 4 * h
    cfg = pl.ScenarioConfig(pipeline_size=2, micro_batches=4, segments=4, seq_len=2048, layers=4, hidden_dim=h,
                            param_count=1)
    tok = tokens_for(4, 2048, 512, seed=21)
    out = []
    for flags in (0, E.FLAG_RECOMPUTE_MLP):
        model = E.ModelConfig(family=family, dtype=E.BF16, vocab=512, hidden=h, layers=4, heads=4, head_dim=hd,
                              ffn=ffn, max_seq=2048, seed=42)
        model.flags = flags
        cfg.param_count = model.param_count()
        part = pl.cwp_partition(cfg)
        eng = E.Engine(cfg, "seq1f1b", part, model)
        rep = eng.step(tok)
        out.append((rep.loss, rep.peak_activation_bytes, {n: eng.read_grad(n) for n in eng.params()}))
        eng.close()
    (l0, m0, g0), (l1, m1, g1) = out
    assert l0 == l1  # the forward does not change
    # the recomputed u is bit-identical, so the gradients differ only by the run-to-run order of
    # the fp32 atomics that accumulate the norm-gain / embedding gradients across CTAs
    worst = max(rel_l2(g1[n], g0[n]) for n in g0)
    assert worst < 1e-6, worst
    assert m1 < m0
    model.flags = E.FLAG_RECOMPUTE_MLP
    with pytest.raises(pl.InvalidArgument):
        E.Engine(cfg, "seqzb1p", pl.cwp_partition(cfg), model)
