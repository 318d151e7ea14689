"""Timeline renderers and the report comparison vs the compiled reference.

render_ascii_gantt / render_svg_gantt (core/src/render.cpp:46-124) and
compare(...).to_csv() (core/src/sim.cpp:319-367) are re-implemented in
csrc/planner/{render,sim}.cpp; for the same simulated report they must emit
the reference's bytes. CPU only (the engine's measured-timeline rendering is
covered in tests/test_gpu_engine.py).
"""
import itertools

import pytest

from oracle import ref
from paper_2406_03488_b200 import planner as pl

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

KINDS = ["gpipe", "1f1b", "1f1b-i", "seq1f1b", "seq1f1b-i", "zb1p", "seqzb1p"]


def _cfg(P, M, k, nv=1, seq=None, cost="flops", comm="1/3"):
    text = (f"pipeline_size = {P}\nstages_per_device = {nv}\nmicro_batches = {M}\nsegments = {k}\n"
            f"seq_len = {seq or 16 * k}\nlayers = 8\nhidden_dim = 64\nparam_count = 1000000\n"
            f"cost_model = {cost}\ncomm_latency = {comm}\n")
    return pl.parse_scenario_text(text)


def _run(kind, P, M, k, nv=1, **kw):
    cost = "uniform" if kind in ("zb1p", "seqzb1p") else "flops"
    cfg = _cfg(P, M, k, nv, cost=cost, **kw)
    part = pl.partition_for(cfg, "cwp" if k > 1 else "even")
    return pl.generate(cfg, kind, part), part


def _cases():
    for kind, (P, M, k) in itertools.product(KINDS, [(2, 4, 2), (4, 8, 4), (3, 5, 1), (4, 12, 8)]):
        nv = 2 if kind.endswith("-i") else 1
        if kind == "seq1f1b-i" and k > P:
            continue
        yield kind, P, M, k, nv


@pytest.mark.parametrize("kind,P,M,k,nv", list(_cases()))
@pytest.mark.parametrize("width", [1, 10, 37, 120, 400])
def test_ascii_gantt_bytes_match_reference(kind, P, M, k, nv, width):
    sched, part = _run(kind, P, M, k, nv)
    ours = pl.render_gantt(sched, part, "ascii", width)
    assert ours == ref.render_gantt(sched, part, "ascii", width)
    rows = ours.splitlines()[1:]
    assert len(rows) == P and all(len(r) == len(f"device {d + 1} |") + max(width, 10) + 1 for d, r in enumerate(rows))


@pytest.mark.parametrize("kind,P,M,k,nv", list(_cases()))
def test_svg_gantt_bytes_match_reference(kind, P, M, k, nv):
    sched, part = _run(kind, P, M, k, nv)
    ours = pl.render_gantt(sched, part, "svg")
    assert ours == ref.render_gantt(sched, part, "svg")
    assert ours.startswith("<?xml") and ours.endswith("</svg>\n")
    assert ours.count('stroke="#ffffff"') == sum(len(o) for o in sched.device_orders)


def test_render_zero_comm_and_rejects_unknown_format():
    sched, part = _run("seq1f1b", 4, 8, 4, comm="0")
    assert pl.render_gantt(sched, part, "ascii", 80) == ref.render_gantt(sched, part, "ascii", 80)
    with pytest.raises(KeyError):
        pl.render_gantt(sched, part, "png")


@pytest.mark.parametrize("P,M", [(2, 4), (4, 8), (8, 16)])
def test_compare_csv_matches_reference(P, M):
    # the ablation the paper reports: batch-level vs sequence-level, with and without ZB
    runs = [_run("1f1b", P, M, 1, seq=256), _run("seq1f1b", P, M, 4, seq=256), _run("gpipe", P, M, 1, seq=256),
            _run("seqzb1p", P, M, 4, seq=256), _run("seq1f1b", P, M, 8, seq=256)]
    try:
        want = ref.compare_csv(runs)
    except RuntimeError as e:  # the reference's exact-rational ratio overflowed int64 (std::overflow_error)
        assert "overflow" in str(e)
        with pytest.raises(pl.RationalOverflow):
            pl.compare_csv(runs)
        runs = runs[:2]
        want = ref.compare_csv(runs)
    ours = pl.compare_csv(runs)
    assert ours == want
    lines = ours.splitlines()
    assert lines[0].startswith("kind,pipeline_size") and len(lines) == len(runs) + 1
    assert lines[1].endswith("1.000000,1.000000,1.000000,1.000000") or ",," in lines[1]


def test_compare_mixed_workloads_and_errors():
    a = _run("1f1b", 2, 4, 1, seq=64)
    b = _run("seq1f1b", 2, 4, 4, seq=64)
    c = _run("seq1f1b", 2, 6, 4, seq=64)
    with pytest.raises(pl.InvalidArgument):
        pl.compare_csv([a])
    with pytest.raises(pl.InvalidArgument):
        pl.compare_csv([a, c])
    assert pl.compare_csv([a, b, c], allow_mixed=True) == ref.compare_csv([a, b, c], allow_mixed=True)
    assert pl.compare_csv([a, b]) == ref.compare_csv([a, b])
