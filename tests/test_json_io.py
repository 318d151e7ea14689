"""seqpipe.schedule.v1 / seqpipe.simreport.v1 wire formats vs the compiled reference.

The engine's JSON IO (csrc/planner/json_io.cpp, own writer/parser) must emit the
reference's canonical bytes (core/src/json_io.cpp:59-159, nlohmann::json dump)
for every schedule kind, parse what the reference emits, and round-trip
dump(parse(text)) == text -- the reference test test_schedules.cpp:254-262
restated. CPU only.
"""
import itertools

import pytest

from oracle import ref
from paper_2406_03488_b200 import planner as pl

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

KINDS = ["gpipe", "1f1b", "1f1b-i", "seq1f1b", "seq1f1b-i", "zb1p", "seqzb1p"]


def _cfg(P, M, k, nv=1, seq=None, cost="flops"):
    text = (f"pipeline_size = {P}\nstages_per_device = {nv}\nmicro_batches = {M}\nsegments = {k}\n"
            f"seq_len = {seq or 16 * k}\nlayers = 8\nhidden_dim = 64\nparam_count = 1000000\n"
            f"cost_model = {cost}\ncomm_latency = 1/3\n")
    return pl.parse_scenario_text(text)


def _cases():
    for kind, (P, M, k) in itertools.product(KINDS, [(2, 4, 2), (4, 8, 4), (3, 5, 1)]):
        nv = 2 if kind.endswith("-i") else 1
        if kind == "seq1f1b-i" and k > P:
            continue
        yield kind, P, M, k, nv


@pytest.mark.parametrize("kind,P,M,k,nv", list(_cases()))
@pytest.mark.parametrize("indent", [2, 4, -1])
def test_schedule_json_bytes_match_reference(kind, P, M, k, nv, indent):
    cfg = _cfg(P, M, k, nv, cost="uniform" if kind in ("zb1p", "seqzb1p") else "flops")
    part = pl.partition_for(cfg, "cwp" if k > 1 else "even")
    sched = pl.generate(cfg, kind, part)
    ours = pl.schedule_to_json(sched, indent)
    assert ours == ref.schedule_to_json(sched, indent)
    back = pl.schedule_from_json(ours)
    assert back == sched
    assert pl.schedule_to_json(back, indent) == ours
    assert ref.schedule_json_roundtrip(ours, indent) == ours


@pytest.mark.parametrize("kind,P,M,k,nv", [c for c in _cases() if c[1] <= 4][:12])
@pytest.mark.parametrize("downsample", [0, 3])
def test_report_json_bytes_match_reference(kind, P, M, k, nv, downsample):
    cfg = _cfg(P, M, k, nv, cost="uniform" if kind in ("zb1p", "seqzb1p") else "flops")
    part = pl.partition_for(cfg, "cwp" if k > 1 else "even")
    sched = pl.generate(cfg, kind, part)
    assert pl.report_to_json(sched, part, 2, downsample) == ref.report_to_json(sched, part, 2, downsample)


def test_schedule_json_rejects_bad_documents():
    cfg = _cfg(2, 4, 2)
    sched = pl.generate(cfg, "seq1f1b", pl.partition_for(cfg, "cwp"))
    text = pl.schedule_to_json(sched)
    for bad in (text.replace("seqpipe.schedule.v1", "seqpipe.schedule.v2"), text[:-20], "[]", "{\"schema\": 1}",
                text.replace('"F"', '"Q"', 1)):
        with pytest.raises(pl.SeqpipeError if hasattr(pl, "SeqpipeError") else Exception):
            pl.schedule_from_json(bad)


def test_schedule_json_parser_bounds_nesting_and_escapes():
    """User-supplied schedule files (`seqpipe_b200 validate`): deep nesting is an error,
    not a stack overflow; \\u needs exactly four hex digits; surrogate pairs decode."""
    err = pl.SeqpipeError if hasattr(pl, "SeqpipeError") else Exception
    for bad in ("[" * 100000 + "]" * 100000, '{"schema": "\\u12G4"}', '{"schema": "\\ud800"}',
                '{"schema": "\\udc00x"}', '{"schema": "\\u12"}'):
        with pytest.raises(err):
            pl.schedule_from_json(bad)
    # Within the depth cap and with valid escapes the document parses far enough to fail on schema.
    for ok_syntax in ("[" * 200 + "]" * 200, '{"schema": "\\ud83d\\ude00"}'):
        with pytest.raises(err) as e:
            pl.schedule_from_json(ok_syntax)
        assert "json parse error" not in str(e.value)


def test_bench_config_schedule_and_report_bytes():
    """cfg-2 (GPT-2.7B preset, P 4, M 8, k 4, cwp): schedule and modeled report identical."""
    cfg = pl.preset_scenario("gpt-2.7b")
    for k, v in (("pipeline_size", "4"), ("seq_len", "32768"), ("segments", "4"), ("micro_batches", "8")):
        pl.apply_scenario_override(cfg, k, v)
    part = pl.cwp_partition(cfg)
    sched = pl.generate(cfg, "seq1f1b", part)
    assert pl.schedule_to_json(sched) == ref.schedule_to_json(sched)
    assert pl.report_to_json(sched, part, 2, 16) == ref.report_to_json(sched, part, 2, 16)
