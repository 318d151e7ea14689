"""The C-ABI boundary: the library loads, exports every entry point that
include/seqpipe_b200.h declares, the Python mirror binds exactly that set, and
errors surface as the reference's exception classes (no compute calls here)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2406_03488_b200 import _capi
from paper_2406_03488_b200 import planner as pl

HEADER = Path(__file__).resolve().parent.parent / "include" / "seqpipe_b200.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("sp_partition", "sp_schedule_ops", "sp_simulate", "sp_check_schedule", "sp_engine_create",
                 "sp_engine_step", "sp_device_partition", "sp_device_schedule_ops", "sp_gemm", "sp_attention_fwd",
                 "sp_attention_bwd", "sp_plan_memory", "sp_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_capi.LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_mirror_binds_exactly_the_header():
    assert sorted(_capi.EXPORTED) == declared()
    _capi.lib()
    assert _capi.MISSING == []


def test_version_and_errors():
    assert b"sm_100a" in _capi.lib().sp_version()
    with pytest.raises(pl.InvalidArgument):
        pl.preset_scenario("gpt-1t")
    with pytest.raises(pl.InvalidArgument):
        pl.ScenarioConfig(pipeline_size=0).validate()
    cfg = pl.ScenarioConfig(pipeline_size=2, micro_batches=4, segments=2, seq_len=32, stages_per_device=1)
    with pytest.raises(pl.UnsupportedScheduleError):
        pl.generate(cfg, "seq1f1b-i", pl.even_partition(cfg))
    with pytest.raises(pl.DomainError):
        pl.cwp_partition(pl.ScenarioConfig(segments=2, seq_len=10, layers=0, hidden_dim=0, param_count=0))
    with pytest.raises(pl.OutOfRange):
        pl.warmup_1f1b(4, 8, 5)


def test_plan_memory_is_host_only():
    from paper_2406_03488_b200 import engine as E
    m = E.ModelConfig(family=E.GPT, dtype=E.BF16, vocab=50257, hidden=2560, layers=32, heads=32, head_dim=80,
                      ffn=10240, max_seq=32768)
    cfg = pl.preset_scenario("gpt-2.7b")
    for k, v in (("pipeline_size", "4"), ("seq_len", "32768"), ("micro_batches", "8")):
        pl.apply_scenario_override(cfg, k, v)
    seq = E.plan_memory(cfg, "seq1f1b", pl.cwp_partition(cfg), m)
    cfg1 = pl.ScenarioConfig(**{**cfg.__dict__, "segments": 1})
    one = E.plan_memory(cfg1, "1f1b", pl.even_partition(cfg1), m)
    # Seq1F1B keeps roughly half the activation bytes of batch-level 1F1B on stage 1 (paper headline)
    assert 0.4 < seq[0] / one[0] < 0.6
