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
