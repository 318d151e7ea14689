"""The multi-rank engine data plane, executed: P Engine handles (rank r of world P), one
host thread each, on cuda:0, exchanging activations and gradients through the in-process
transport (transport.hpp LocalTransport) exactly as sp_comm_plan lists them -- the same
engine code path the NCCL transport drives between processes (one channel per pipeline
edge and direction, receives posted ahead into staging slots, sends on per-channel
streams). These are the pipeline edges of the reference dependency model
(/root/reference/proj/core/src/sim.cpp:20-23 activations, :31-33 gradients).

Checked: each rank's executed op log is the reference generate()'s device order; loss and
every parameter gradient match the fp64 oracle (fp32 mode, relative L2 <= 1e-5); a receive
that never pairs up fails with DeadlockError instead of hanging."""
import threading

import pytest

from oracle import ref
from oracle.transformer import GPT, Model, rel_l2, tokens_for
from paper_2406_03488_b200 import engine as E
from paper_2406_03488_b200 import planner as pl

pytestmark = pytest.mark.gpu
TOL_F32 = 1e-5


def _model(dtype=E.F32, layers=8):
    return E.ModelConfig(family=GPT, dtype=dtype, vocab=256, hidden=128, layers=layers, heads=2, head_dim=64,
                         ffn=256, max_seq=512, seed=42)


def _run_ranks(cfg, kind, part, model, tok, watchdog=60.0, only=None):
    P = cfg.pipeline_size
    hub = E.LocalHub(P, watchdog_seconds=watchdog)
    engines = [E.Engine(cfg, kind, part, model, rank=r, world_size=P, cuda_device=0) for r in range(P)]
    for e in engines:
        e.attach_local(hub)
    reps, errs = [None] * P, [None] * P

    def go(r):
        try:
            reps[r] = engines[r].step(tok)
        except Exception as ex:  # surfaced below
            errs[r] = ex

    ranks = range(P) if only is None else only
    th = [threading.Thread(target=go, args=(r,)) for r in ranks]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=watchdog + 120)
    assert not any(t.is_alive() for t in th), "a rank thread hung"
    return engines, reps, errs, hub


@pytest.mark.parametrize("kind,P,nv,k,mode", [
    ("seq1f1b", 2, 1, 4, "cwp"), ("seq1f1b", 4, 1, 4, "cwp"), ("1f1b", 4, 1, 1, "even"), ("gpipe", 2, 1, 2, "even"),
    ("seq1f1b-i", 2, 2, 2, "cwp"), ("1f1b-i", 2, 2, 1, "even"), ("seq1f1b-i", 4, 2, 2, "cwp"),
    ("seqzb1p", 4, 1, 4, "even"), ("zb1p", 2, 1, 1, "even")])
def test_multirank_step_matches_reference_order_and_oracle(gpu, kind, P, nv, k, mode):
    model = _model(layers=2 * P * nv)
    cfg = pl.ScenarioConfig(pipeline_size=P, stages_per_device=nv, micro_batches=2 * P, segments=k, seq_len=512,
                            layers=model.layers, hidden_dim=model.hidden, param_count=model.param_count())
    cfg.validate()
    part = pl.partition_for(cfg, mode)
    tok = tokens_for(cfg.micro_batches, cfg.seq_len, model.vocab, seed=5)
    engines, reps, errs, hub = _run_ranks(cfg, kind, part, model, tok)
    assert all(e is None for e in errs), errs
    want = ref.generate(cfg, kind, part).device_orders
    for r, eng in enumerate(engines):
        assert eng.op_log().device_orders[r] == want[r], f"rank {r} executed a different order"
    # the last stage lives on the last device (round-robin stage map, task.hpp:45-47)
    loss_rank = (cfg.total_stages() - 1) % P
    params, owner = {}, {}
    for eng in engines:
        for n in eng.params():
            params[n] = eng.read_param(n)
            owner[n] = eng
    loss, grads = Model(GPT, model.vocab, model.hidden, model.layers, model.heads, model.head_dim,
                        model.ffn).step(params, tok, part.lengths)
    assert abs(reps[loss_rank].loss - loss) / abs(loss) < TOL_F32, (reps[loss_rank].loss, loss)
    bad = {n: rel_l2(owner[n].read_grad(n), grads[n]) for n in params}
    assert max(bad.values()) < TOL_F32, {n: v for n, v in bad.items() if v >= TOL_F32}
    for e in engines:
        e.close()


def test_interleaved_table_the_reference_cannot_complete_is_refused(gpu):
    """seq1f1b-i at odd P: the reference generate() itself emits an order its own
    check_schedule flags as order_deadlock (validate.cpp); the engine refuses it up front
    instead of hanging in a receive."""
    model = _model(layers=12)
    cfg = pl.ScenarioConfig(pipeline_size=3, stages_per_device=2, micro_batches=6, segments=2, seq_len=512,
                            layers=12, hidden_dim=128, param_count=model.param_count())
    part = pl.cwp_partition(cfg)
    assert ref.check_schedule(ref.generate(cfg, "seq1f1b-i", part))  # the reference flags its own table
    with pytest.raises(pl.LogicError, match="order_deadlock"):
        E.Engine(cfg, "seq1f1b-i", part, model, rank=0, world_size=3, cuda_device=0)


def test_multirank_bf16_production_kernels(gpu):
    """The bf16 tcgen05 / tensor-core attention mix through the multi-rank data plane (P = 4)."""
    model = E.ModelConfig(family=GPT, dtype=E.BF16, vocab=512, hidden=320, layers=4, heads=4, head_dim=80, ffn=1280,
                          max_seq=1024, seed=42)
    cfg = pl.ScenarioConfig(pipeline_size=4, micro_batches=6, segments=4, seq_len=1024, layers=4, hidden_dim=320,
                            param_count=model.param_count())
    part = pl.cwp_partition(cfg)
    tok = tokens_for(cfg.micro_batches, cfg.seq_len, model.vocab, seed=8)
    engines, reps, errs, hub = _run_ranks(cfg, "seq1f1b", part, model, tok)
    assert all(e is None for e in errs), errs
    params, owner = {}, {}
    for eng in engines:
        for n in eng.params():
            params[n] = eng.read_param(n)
            owner[n] = eng
    loss, grads = Model(GPT, model.vocab, model.hidden, model.layers, model.heads, model.head_dim,
                        model.ffn).step(params, tok, part.lengths)
    assert abs(reps[3].loss - loss) / abs(loss) < 2e-2
    assert max(rel_l2(owner[n].read_grad(n), grads[n]) for n in params) < 2e-2
    for e in engines:
        e.close()


def test_unmatched_receive_is_a_deadlock_error_not_a_hang(gpu):
    """Only rank 1 steps: its first receive never pairs up. The transport's watchdog turns
    that into DeadlockError (the reference's failure mode for an order that cannot
    complete, sim.cpp:217-231) within the watchdog time."""
    model = _model(layers=2)
    cfg = pl.ScenarioConfig(pipeline_size=2, micro_batches=3, segments=2, seq_len=512, layers=2, hidden_dim=128,
                            param_count=model.param_count())
    part = pl.cwp_partition(cfg)
    tok = tokens_for(3, 512, model.vocab)
    engines, reps, errs, hub = _run_ranks(cfg, "seq1f1b", part, model, tok, watchdog=2.0, only=[1])
    assert isinstance(errs[1], pl.DeadlockError), errs
    for e in engines:
        e.close()
