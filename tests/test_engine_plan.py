"""Host-side engine planning (no GPU): the arena plan of every schedule kind,
including the zero-bubble I / W split, replayed from the reference op tables."""
import pytest

from paper_2406_03488_b200 import engine as E
from paper_2406_03488_b200 import planner as pl


def _model():
    return E.ModelConfig(family=E.GPT, dtype=E.F32, vocab=256, hidden=128, layers=4, heads=2, head_dim=64, ffn=256,
                         max_seq=512, seed=1)


def _cfg(model, P=2, M=4, k=4, T=512):
    cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=M, segments=k, seq_len=T, layers=model.layers,
                            hidden_dim=model.hidden, param_count=model.param_count())
    cfg.validate()
    return cfg


def test_zero_bubble_records_live_until_w():
    """ZB kinds free each (m, s) record at its W task (sim.cpp:279-293) and add the W
    record at I: the stage-1 peak is at least Seq1F1B's for the same partition."""
    model = _model()
    cfg = _cfg(model)
    part = pl.partition_for(cfg, "cwp")
    zb = E.plan_memory(cfg, "seqzb1p", part, model, stage=1)[0]
    sq = E.plan_memory(cfg, "seq1f1b", part, model, stage=1)[0]
    assert zb >= sq > 0


@pytest.mark.parametrize("kind", ["gpipe", "1f1b", "seq1f1b", "zb1p", "seqzb1p"])
def test_plan_every_kind(kind):
    model = _model()
    k = 1 if kind in ("zb1p", "1f1b", "gpipe") else 4
    cfg = _cfg(model, k=k)
    part = pl.partition_for(cfg, "even" if k == 1 else "cwp")
    for stage in (1, 2):
        live, arena, dkv = E.plan_memory(cfg, kind, part, model, stage=stage)
        assert 0 < live <= arena and dkv > 0


@pytest.mark.parametrize("kind", ["1f1b", "seq1f1b", "seqzb1p"])
@pytest.mark.parametrize("P,M,k,mode", [(2, 4, 4, "cwp"), (4, 8, 4, "cwp"), (4, 8, 4, "even"), (8, 16, 8, "cwp"),
                                        (3, 6, 2, "cwp"), (8, 16, 16, "even")])
def test_offline_arena_placement(kind, P, M, k, mode):
    """The arena offsets are placed offline over the known op order (stage.cpp place_offline;
    the planner throws if two records live at the same time would share bytes). The arena is
    never below the live high-water, equals it when every record has one size (even partitions
    and batch-level 1F1B without the zero-bubble W records), and stays within 20 % of it on
    the cwp partitions (records of k sizes)."""
    model = E.ModelConfig(family=E.GPT, dtype=E.BF16, vocab=512, hidden=256, layers=2 * P, heads=4, head_dim=64,
                          ffn=1024, max_seq=8192, seed=1)
    kk = 1 if kind == "1f1b" else k
    cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=M, segments=kk, seq_len=8192, layers=model.layers,
                            hidden_dim=model.hidden, param_count=model.param_count())
    part = pl.partition_for(cfg, mode if kk > 1 else "even")
    for stage in range(1, P + 1):
        live, arena, _ = E.plan_memory(cfg, kind, part, model, stage=stage)
        assert live <= arena <= 1.2 * live, (stage, live, arena)
        if (mode == "even" or kk == 1) and kind != "seqzb1p":
            assert arena == live, (stage, live, arena)


def test_recompute_mlp_plan_drops_u():
    """SP_FLAG_RECOMPUTE_MLP removes the MLP up-projection output (L_s x n x Fup elements) from
    every (m, s) record: at P = 1 with one micro-batch in flight the live peak drops by exactly
    that field's bytes over all of the micro-batch's segments."""
    model = E.ModelConfig(family=E.LLAMA, dtype=E.BF16, vocab=512, hidden=256, layers=2, heads=2, head_dim=128,
                          ffn=768, max_seq=4096, seed=1)
    cfg = pl.ScenarioConfig(pipeline_size=1, micro_batches=1, segments=4, seq_len=4096, layers=2, hidden_dim=256,
                            param_count=model.param_count())
    part = pl.partition_for(cfg, "cwp")
    live0 = E.plan_memory(cfg, "seq1f1b", part, model, stage=1)[0]
    model.flags = E.FLAG_RECOMPUTE_MLP
    live1 = E.plan_memory(cfg, "seq1f1b", part, model, stage=1)[0]
    u_bytes = 2 * 4096 * (2 * 768) * 2  # layers x tokens x Fup (SwiGLU: 2F) x bf16
    assert live0 - live1 == u_bytes
    with pytest.raises(pl.InvalidArgument):  # the zero-bubble kinds keep the MLP operands for W
        E.Engine(cfg, "seqzb1p", part, model)
