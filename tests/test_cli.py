"""bin/seqpipe_b200, the command-line front end.

The planning subcommands keep the reference CLI's surface and bytes
(tools/src/seqpipe_main.cpp:122-289): every output here is recomputed through
the compiled reference library (oracle/_ref) and compared byte for byte; exit
codes follow seqpipe_main.cpp:29-32 (1 runtime, 2 usage, 3 validation). The
B200 `execute` subcommand is covered by tests/test_gpu_cli.py. CPU only.
"""
import json
import subprocess
from fractions import Fraction
from pathlib import Path

import pytest

from oracle import ref
from paper_2406_03488_b200 import planner as pl

CLI = Path(__file__).resolve().parent.parent / "paper_2406_03488_b200" / "bin" / "seqpipe_b200"
pytestmark = [pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built"),
              pytest.mark.skipif(not CLI.exists(), reason="CLI not built")]

CFG2 = ["--preset", "gpt-2.7b", "--set", "pipeline_size=4", "seq_len=32768", "segments=4", "micro_batches=8"]


def run(*args, ok=True):
    r = subprocess.run([str(CLI), *args], capture_output=True, text=True, timeout=120)
    if ok:
        assert r.returncode == 0, (args, r.returncode, r.stderr)
    return r


def cfg_of(preset, **over):
    c = ref.preset_scenario(preset)
    for k, v in over.items():
        c = ref.apply_scenario_override(c, k, str(v))
    return c


def dec6(x: Fraction) -> str:
    """format_decimal(x, 6): fixed point, round half away from zero (rational.hpp)."""
    q = abs(x) * 10 ** 6
    n = q.numerator // q.denominator
    if (q - n) * 2 >= 1:
        n += 1
    s = f"{n // 10 ** 6}.{n % 10 ** 6:06d}"
    return ("-" + s) if x < 0 and n else s


@pytest.mark.parametrize("kind,mode", [("seq1f1b", "cwp"), ("1f1b", "even"), ("seqzb1p", "cwp"), ("seq1f1b-i", "even")])
def test_simulate_report_schedule_and_gantt_match_reference(tmp_path, kind, mode):
    over = dict(pipeline_size=4, seq_len=32768, segments=4, micro_batches=8)
    if kind == "seq1f1b-i":
        over["stages_per_device"] = 2
    if kind == "seqzb1p":
        over["cost_model"] = "uniform"
    sets = [f"{k}={v}" for k, v in over.items()]
    r = run("simulate", "--preset", "gpt-2.7b", "--set", *sets, "--kind", kind, "--partition", mode,
            "--emit-schedule", str(tmp_path / "s.json"), "--gantt", "ascii", "--gantt-out", str(tmp_path / "g.txt"),
            "--gantt-width", "90", "--validate", "--memory-downsample", "4")
    cfg = cfg_of("gpt-2.7b", **over)
    part = ref.partition_for(cfg, mode)
    sch = ref.generate(cfg, kind, part)
    assert r.stdout == ref.report_to_json(sch, part, 2, 4)
    assert (tmp_path / "s.json").read_text() == ref.schedule_to_json(sch)
    assert (tmp_path / "g.txt").read_text() == ref.render_gantt(sch, part, "ascii", 90)
    svg = run("simulate", "--preset", "gpt-2.7b", "--set", *sets, "--kind", kind, "--partition", mode,
              "--out", str(tmp_path / "r.json"), "--gantt", "svg").stdout
    assert svg == ref.render_gantt(sch, part, "svg")
    stamped = run("simulate", "--preset", "gpt-2.7b", "--set", *sets, "--kind", kind, "--partition", mode,
                  "--stamp").stdout
    assert json.loads(stamped)["generated_at"].endswith("Z")


def test_partition_table_and_json_match_reference():
    cfg = cfg_of("gpt-2.7b", pipeline_size=4, seq_len=32768, segments=4, micro_batches=8)
    part = ref.partition_for(cfg, "cwp")
    costs, imb = ref.balance_report(part, cfg)
    doc = json.loads(run("partition", *CFG2, "--json").stdout)
    assert doc["lengths"] == part.lengths == [10170, 8496, 7428, 6674]  # SURVEY §8 a7 golden
    assert doc["segment_costs"] == [str(c) for c in costs] and Fraction(doc["imbalance"]) == imb
    table = run("partition", *CFG2).stdout.splitlines()
    assert table[0] == "segment  tokens  forward_cost"
    assert table[1:5] == [f"{i + 1}  {n}  {c}" for i, (n, c) in enumerate(zip(part.lengths, costs))]
    assert table[5] == f"imbalance = {imb.numerator}/{imb.denominator} ({dec6(imb)})"
    even = json.loads(run("partition", *CFG2, "--mode", "even", "-k", "8", "--json").stdout)
    assert even["lengths"] == [4096] * 8


def test_sweep_rows_match_reference_simulations():
    out = run("sweep", "--preset", "gpt-2.7b", "--set", "seq_len=8192", "--kinds", "1f1b,seq1f1b,seq1f1b-i",
              "--pipeline-sizes", "2,4", "--segment-counts", "1,4,8", "--micro-batches", "8",
              "--partition", "cwp").stdout.splitlines()
    assert out[0] == ("kind,pipeline_size,stages_per_device,micro_batches,segments,seq_len,partition,status,"
                      "makespan,bubble_ratio,peak_memory,throughput")
    rows = [r.split(",") for r in out[1:]]
    assert len(rows) == 3 * 2 * 3
    n_ok = 0
    for kind, P, nv, M, k, T, mode, status, *vals in rows:
        if status.startswith("skip:"):
            assert vals == ["", "", "", ""]
            continue
        cfg = cfg_of("gpt-2.7b", seq_len=T, pipeline_size=P, micro_batches=M, segments=k, stages_per_device=nv)
        part = ref.partition_for(cfg, mode)
        _t, _d, summ, _n = ref.simulate_raw(ref.generate(cfg, kind, part), part)
        want = [dec6(ref._frac(getattr(summ, f))) for f in
                ("makespan", "aggregate_bubble_ratio", "max_peak_memory", "modeled_throughput")]
        assert vals == want, (kind, P, k)
        n_ok += 1
    assert n_ok >= 12
    # infeasible points are reported, not fatal (reference :221-229)
    skip = run("sweep", "--preset", "gpt-2.7b", "--kinds", "seq1f1b-i", "--pipeline-sizes", "2",
               "--segment-counts", "4", "--stages-per-device", "2").stdout.splitlines()
    assert skip[1].split(",")[7].startswith("skip:")


def test_validate_ok_and_violation_exit_code(tmp_path):
    cfg = cfg_of("gpt-2.7b", pipeline_size=4, seq_len=4096, segments=4, micro_batches=8)
    part = ref.partition_for(cfg, "cwp")
    sch = ref.generate(cfg, "seq1f1b", part)
    good = tmp_path / "good.json"
    good.write_text(ref.schedule_to_json(sch))
    assert run("validate", str(good)).stdout == "ok\n"
    orders = [list(o) for o in sch.device_orders]
    orders[0][0], orders[0][1] = orders[0][1], orders[0][0]
    bad_sch = pl.Schedule(sch.config, sch.kind, orders)
    bad = tmp_path / "bad.json"
    bad.write_text(ref.schedule_to_json(bad_sch))
    r = run("validate", str(bad), ok=False)
    assert r.returncode == 3 and r.stderr and ref.check_schedule(bad_sch)


@pytest.mark.parametrize("args,code", [
    ((), 2), (("frobnicate",), 2), (("simulate", "--preset", "gpt-2.7b"), 2),
    (("simulate", "--preset", "gpt-2.7b", "--kind", "nope"), 2),
    (("simulate", "--preset", "gpt-2.7b", "--kind", "seq1f1b", "--partition", "magic"), 2),
    (("simulate", "--preset", "gpt-2.7b", "--config", "x.txt", "--kind", "1f1b"), 2),
    (("simulate", "--preset", "gpt-2.7b", "--kind", "1f1b", "--set", "nonsense"), 1),
    (("simulate", "--preset", "gpt-2.7b", "--kind", "1f1b", "--set", "no_such_key=3"), 1),
    (("partition", "--preset", "gpt-2.7b", "-k", "x"), 2),
    (("validate",), 2), (("validate", "/nonexistent.json"), 1),
])
def test_exit_codes(args, code):
    assert run(*args, ok=False).returncode == code


def test_kind_is_case_insensitive_like_reference():
    a = run("simulate", *CFG2, "--kind", "SEQ1F1B", "--partition", "cwp").stdout
    b = run("simulate", *CFG2, "--kind", "seq1f1b", "--partition", "cwp").stdout
    assert a == b and '"kind": "seq1f1b"' in a
