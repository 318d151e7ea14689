"""Live differential test of the engine's planner against the compiled
reference planner (oracle/_ref): partitions, op tables of all seven kinds,
simulate() report fields, validator verdicts, warm-up formulas, POQ, config
parsing and the error behaviour (same exception class) over sweep grids."""
import itertools
from fractions import Fraction

import pytest

from oracle import ref
from paper_2406_03488_b200 import planner as pl

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _outcome(fn):
    try:
        return ("ok", fn())
    except Exception as e:  # noqa: BLE001
        return ("err", type(e).__name__)


def _same_error(ours, theirs):
    # both raise, and they map to the same reference exception family
    return ours[0] == theirs[0] == "err" and ours[1] == theirs[1]


def test_partition_grid():
    n = 0
    for T, k, L, d, params in itertools.product([1, 2, 3, 7, 64, 100, 257, 2048, 32768], [1, 2, 3, 4, 5, 8, 16],
                                                [0, 1, 8, 32], [0, 1, 256, 2560], [0, 1000, 12 * 8 * 256 * 256]):
        cfg = pl.ScenarioConfig(pipeline_size=1, micro_batches=1, segments=k, seq_len=T, layers=L, hidden_dim=d,
                                param_count=params)
        for mode in ("even", "cwp"):
            a = _outcome(lambda: pl.partition_for(cfg, mode))
            b = _outcome(lambda: ref.partition_for(cfg, mode))
            assert a == b or _same_error(a, b), (T, k, L, d, params, mode, a, b)
            n += 1
    assert n > 5000


def test_oracle_partition_small():
    for T, k in [(8, 2), (17, 3), (40, 4), (100, 2)]:
        cfg = pl.ScenarioConfig(segments=k, seq_len=T, layers=2, hidden_dim=4, param_count=100)
        assert pl.oracle_partition(cfg).lengths == ref.partition_for(cfg, "oracle").lengths
    cfg = pl.ScenarioConfig(segments=5, seq_len=100)
    with pytest.raises(pl.InvalidArgument):
        pl.oracle_partition(cfg)


@pytest.mark.parametrize("kind", pl.SCHEDULE_KINDS)
def test_schedule_simulate_validate_grid(kind):
    checked = 0
    for P, M, k, nv in itertools.product([1, 2, 3, 4, 8], [1, 2, 3, 4, 5, 8, 9, 16], [1, 2, 3, 4, 8], [1, 2]):
        for cost in ("uniform", "flops"):
            cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=M, segments=k, stages_per_device=nv,
                                    seq_len=16 * k, layers=2, hidden_dim=8, param_count=1000, cost_model=cost,
                                    comm_latency=Fraction(1, 3) if P % 2 else 0)
            part = pl.partition_for(cfg, "cwp")
            a = _outcome(lambda: pl.generate(cfg, kind, part))
            b = _outcome(lambda: ref.generate(cfg, kind, part))
            assert (a[0] == b[0]) and (a[1] == b[1] if a[0] == "err" else a[1].device_orders == b[1].device_orders), \
                (P, M, k, nv, cost, a if a[0] == "err" else "", b if b[0] == "err" else "")
            if a[0] == "err":
                continue
            s = a[1]
            ra = _outcome(lambda: pl.simulate(s, part, with_series=False))
            rb = _outcome(lambda: ref.simulate_raw(s, part))
            if ra[0] == "err" or rb[0] == "err":  # e.g. reference seq1f1b-i orders that deadlock
                assert _same_error(ra, rb), (P, M, k, nv, ra, rb)
                assert [v.code for v in pl.check_schedule(s)] == [v.code for v in ref.check_schedule(s)]
                continue
            rep = ra[1]
            timings, devs, summ, nops = rb[1]
            assert rep.makespan == pl._frac(summ.makespan)
            assert rep.aggregate_bubble_ratio == pl._frac(summ.aggregate_bubble_ratio)
            assert rep.aggregate_bubble_ratio_in_makespan == pl._frac(summ.aggregate_bubble_ratio_in_makespan)
            assert rep.max_peak_memory == pl._frac(summ.max_peak_memory)
            assert rep.modeled_throughput == pl._frac(summ.modeled_throughput)
            flat = [t for dev in rep.task_times for t in dev]
            assert [(pl._frac(timings[i].start), pl._frac(timings[i].end)) for i in range(nops)] == \
                [(t[1], t[2]) for t in flat]
            for d, dr in enumerate(rep.devices):
                assert dr.peak_allocations == devs[d].peak_allocations
                assert dr.warmup_forward_tasks == devs[d].warmup_forward_tasks
                assert dr.idle == pl._frac(devs[d].idle)
            assert pl.check_schedule(s) == ref.check_schedule(s) == []
            checked += 1
    assert checked > 50


def test_validator_catches_every_mutation_like_reference():
    """Mutation fault injection (acceptance criterion 5): swap each same-device
    (prerequisite, dependent) pair; both validators must flag every mutant with
    identical violation codes and devices."""
    cfg = pl.ScenarioConfig(pipeline_size=3, micro_batches=4, segments=3, seq_len=48, cost_model="uniform")
    part = pl.partition_for(cfg, "even")
    s = pl.generate(cfg, "seq1f1b", part)
    mutants = 0
    for d, order in enumerate(s.device_orders):
        pos = {t: i for i, t in enumerate(order)}
        for i, t in enumerate(order):
            for dep in pl.dependencies(t, cfg):
                if dep.device != t.device or dep not in pos:
                    continue
                j = pos[dep]
                new = [list(o) for o in s.device_orders]
                new[d][i], new[d][j] = new[d][j], new[d][i]
                m = pl.Schedule(cfg, "seq1f1b", new)
                va = pl.check_schedule(m)
                vb = ref.check_schedule(m)
                assert va, (d, i, j)
                assert [(v.code, v.device) for v in va] == [(v.code, v.device) for v in vb]
                mutants += 1
    assert mutants > 20


def test_warmup_formulas_and_checker():
    for formula, a_vals in ((0, [2, 4, 8, 16, 32]), (1, [2, 4, 8, 16, 32]), (2, [1, 2, 3]), (3, [1, 2, 3])):
        for P, a, k in itertools.product([1, 2, 4, 8], a_vals, [1, 2, 4]):
            for d in range(0, P + 2):
                ours = _outcome(lambda: pl._warm(formula, P, a, k, d))
                theirs = _outcome(lambda: ref.warmup(formula, P, a, k, d))
                assert ours == theirs or _same_error(ours, theirs)
    for kind in ("1f1b", "seq1f1b", "1f1b-i", "seq1f1b-i"):
        for P, mult, k, nv in itertools.product([2, 4, 8], [2, 4], [1, 2, 4], [1, 2]):
            if ("-i" in kind) != (nv == 2):
                continue
            cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=mult * P, segments=k, stages_per_device=nv,
                                    seq_len=16 * k, cost_model="uniform")
            try:
                s = pl.generate(cfg, kind, pl.even_partition(cfg))
            except pl.UnsupportedScheduleError:
                continue
            assert pl.check_warmup_formulas(s) == ref.check_warmup_formulas(s) == []


def test_poq_matches_reference_model():
    state = 99
    ops, contents = [], []

    def nxt():
        nonlocal state
        state = (state * 6364136223846793005 + 1442695040888963407) % (1 << 64)
        return state >> 33
    for _ in range(500):
        if not contents or (nxt() % 2 == 0 and len(ops) < 400):
            m, s = nxt() % 20 + 1, nxt() % 20 + 1
            if (m, s) in contents:
                continue
            ops.append((0, m, s))
            contents.append((m, s))
        else:
            ops.append((1, 0, 0))
            exp = min(contents, key=lambda e: (e[0], -e[1]))
            contents.remove(exp)
    pops = ref.poq_run(ops)
    model = []
    cont = []
    for op in ops:
        if op[0] == 0:
            cont.append(op[1:])
        else:
            e = min(cont, key=lambda e: (e[0], -e[1]))
            cont.remove(e)
            model.append(e)
    assert pops == model


def test_config_parsing_and_presets_match_reference():
    for name in pl.preset_names():
        assert pl.preset_scenario(name) == ref.preset_scenario(name)
        assert pl.scenario_to_text(pl.preset_scenario(name)) == ref.scenario_to_text(ref.preset_scenario(name))
    text = open("/root/reference/proj/configs/sample.cfg").read() if __import__("os").path.exists(
        "/root/reference/proj/configs/sample.cfg") else "pipeline_size = 4\nsegments = 4\nseq_len = 64\n"
    assert pl.parse_scenario_text(text) == ref.parse_scenario_text(text)
    for bad in ("foo = 1", "pipeline_size = x", "pipeline_size", "bw_split_ratio = 1", "comm_latency = 1/0",
                "cost_model = fast", "seq_len = 1.5", "time_per_flop = 1."):
        a = _outcome(lambda: pl.parse_scenario_text(bad))
        b = _outcome(lambda: ref.parse_scenario_text(bad))
        assert _same_error(a, b), (bad, a, b)
    for key, val in (("backward_ratio", "5/2"), ("comm_latency", "0.25"), ("bw_split_ratio", "1, 3/2"),
                     ("segments", "16"), ("cost_model", "uniform")):
        c = pl.ScenarioConfig()
        pl.apply_scenario_override(c, key, val)
        assert c == ref.apply_scenario_override(pl.ScenarioConfig(), key, val)
