"""Known-answer tests of the reference's own suites, restated against the
engine's planner (the reference doctest suites cannot build here: doctest.h is
absent). Sources: /root/reference/proj/tests/test_schedules.cpp,
test_partition.cpp, test_core.cpp, test_sim.cpp, test_validate.cpp,
acceptance_main.cpp (cited per test)."""
from fractions import Fraction

import pytest

from paper_2406_03488_b200 import planner as pl


def sweep(P, M, k, nv=1, factor=8):
    cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=M, segments=k, stages_per_device=nv, seq_len=factor * k,
                            cost_model="uniform")
    cfg.validate()
    return cfg


def make(cfg, kind):
    return pl.generate(cfg, kind, pl.even_partition(cfg))


def brief(order, n):
    return " ".join(t.brief() for t in order[:n])


def test_warmup_formulas():  # test_schedules.cpp:48-73
    assert pl.warmup_1f1b(8, 32, 1) == 7
    assert pl.warmup_1f1b(4, 8, 4) == 0
    assert pl.warmup_1f1b(8, 4, 3) == 4
    assert pl.warmup_seq1f1b(4, 8, 2, 4) == 1
    assert pl.warmup_seq1f1b(8, 32, 4, 1) == 10
    for d in range(1, 5):
        assert pl.warmup_seq1f1b(4, 8, 1, d) == pl.warmup_1f1b(4, 8, d)
    assert pl.warmup_1f1b_interleaved(4, 2, 1) == 10
    assert pl.warmup_1f1b_interleaved(4, 2, 4) == 4
    assert pl.warmup_1f1b_interleaved(5, 1, 5) == 0
    assert pl.warmup_seq1f1b_interleaved(4, 2, 2, 1) == 11
    assert pl.warmup_seq1f1b_interleaved(4, 2, 4, 4) == 7
    assert [pl.warmup_seq1f1b_interleaved(4, 2, 2, d) for d in range(1, 5)] == [11, 9, 7, 5]


def test_seq1f1b_last_device_kat():  # test_schedules.cpp:125-128
    assert brief(make(sweep(4, 8, 2), "seq1f1b").device_orders[3], 5) == "F1.1 F1.2 B1.2 F2.1 B1.1"


def test_1f1b_last_device_kat():  # test_schedules.cpp:130-133
    assert brief(make(sweep(4, 8, 1), "1f1b").device_orders[3], 4) == "F1.1 B1.1 F2.1 B2.1"


def test_single_micro_batch():  # test_schedules.cpp:135-142
    for order in make(sweep(3, 1, 1), "1f1b").device_orders:
        assert [t.kind for t in order] == ["F", "B"]


def test_gpipe_all_forwards_first():  # test_schedules.cpp:144-155
    s = make(sweep(4, 6, 2), "gpipe")
    for order in s.device_orders:
        kinds = [t.kind for t in order]
        assert kinds == ["F"] * 12 + ["B"] * 12


def test_k1_equals_batch_level():  # test_schedules.cpp:163-170
    a = make(sweep(4, 8, 1), "seq1f1b")
    b = make(sweep(4, 8, 1), "1f1b")
    assert a.device_orders == b.device_orders


def test_m_le_p_degrades_to_gpipe():  # SURVEY Appendix A (P4 M4 k4)
    s = make(sweep(4, 4, 4), "seq1f1b")
    for order in s.device_orders:
        assert [t.kind for t in order[:16]] == ["F"] * 16
        assert brief(order[16:], 5) == "B1.4 B1.3 B1.2 B1.1 B2.4"


def test_feasibility_errors():  # test_schedules.cpp:187-202
    with pytest.raises(pl.UnsupportedScheduleError):
        make(sweep(4, 8, 2, nv=1), "1f1b-i")
    with pytest.raises(pl.UnsupportedScheduleError):
        make(sweep(4, 8, 2, nv=2), "seq1f1b")
    with pytest.raises(pl.UnsupportedScheduleError):
        make(sweep(2, 8, 4, nv=2), "seq1f1b-i")  # k > P


def test_cwp_kat_62_38():  # test_partition.cpp:40-47, test_cli.cpp:162-172
    cfg = pl.ScenarioConfig(segments=2, seq_len=100, layers=1, hidden_dim=1, param_count=0)
    assert pl.cwp_partition(cfg).lengths == [62, 38]


def test_even_remainder_first():  # test_partition.cpp:32-38
    cfg = pl.ScenarioConfig(segments=3, seq_len=10)
    assert pl.even_partition(cfg).lengths == [4, 3, 3]


def test_linear_cost_gives_even():  # test_partition.cpp:57-64
    cfg = pl.ScenarioConfig(segments=4, seq_len=100, layers=0, hidden_dim=0, param_count=10)
    assert pl.cwp_partition(cfg).lengths == [25, 25, 25, 25]


def test_cwp_lengths_non_increasing_and_balanced():  # test_partition.cpp:120-143
    for T, k in [(2048, 4), (32768, 4), (65536, 8), (131072, 16), (999, 7)]:
        cfg = pl.ScenarioConfig(segments=k, seq_len=T, layers=8, hidden_dim=256, param_count=12 * 8 * 256 * 256)
        c = pl.cwp_partition(cfg)
        e = pl.even_partition(cfg)
        assert all(a >= b for a, b in zip(c.lengths, c.lengths[1:]))
        assert c.imbalance <= e.imbalance


def test_cost_kats():  # test_core.cpp:110-141
    cfg = pl.ScenarioConfig(segments=3, seq_len=100, layers=1, hidden_dim=1, param_count=0)
    p = pl.make_partition([62, 38, 0 + 0] if False else [50, 25, 25], cfg)
    assert pl.segment_flops(cfg, 0, 50) == 2 * 50 * 50
    assert pl.forward_cost(cfg, p, 1) == Fraction(2 * 50 * 50)
    assert pl.forward_cost(cfg, p, 2) == Fraction(2 * 25 * 75)
    cfg2 = pl.ScenarioConfig(pipeline_size=2, stages_per_device=2, segments=1, seq_len=10, layers=1, hidden_dim=1,
                             param_count=0)
    p2 = pl.make_partition([10], cfg2)
    assert pl.forward_cost(cfg2, p2, 1) == Fraction(200, 4)


def test_uniform_cost_quarter_and_eighth():  # test_core.cpp:161-174
    cfg = pl.ScenarioConfig(segments=4, seq_len=64, cost_model="uniform")
    p = pl.even_partition(cfg)
    assert pl.forward_cost(cfg, p, 2) == Fraction(1, 4)
    cfg2 = pl.ScenarioConfig(segments=4, stages_per_device=2, seq_len=64, cost_model="uniform")
    assert pl.forward_cost(cfg2, pl.even_partition(cfg2), 1) == Fraction(1, 8)


def test_makespan_closed_form():  # test_sim.cpp:65-76: (M+P-1)(tf+tb) for 1F1B uniform
    for P, M in [(2, 4), (4, 8), (8, 16)]:
        cfg = sweep(P, M, 1)
        rep = pl.simulate(make(cfg, "1f1b"), pl.even_partition(cfg))
        assert rep.makespan == (M + P - 1) * 3


def test_seq1f1b_first_device_idle():  # test_sim.cpp:104-116: idle(dev1) = 3(P-1)/k
    for P, k in [(4, 2), (4, 4), (8, 4)]:
        cfg = sweep(P, 2 * P, k)
        rep = pl.simulate(make(cfg, "seq1f1b"), pl.even_partition(cfg))
        assert rep.devices[0].idle == Fraction(3 * (P - 1), k)


def test_peak_allocations_warmup_plus_one():  # test_sim.cpp:157-169 / SURVEY App. A: 7/6/5/4
    cfg = sweep(4, 8, 4)
    rep = pl.simulate(make(cfg, "seq1f1b"), pl.even_partition(cfg))
    assert [d.peak_allocations for d in rep.devices] == [7, 6, 5, 4]


def test_memory_seq1f1b_below_1f1b():  # acceptance criterion 4 (acceptance_main.cpp:150-185)
    for P in (2, 4, 8):
        for k in (2, 4):
            cs = sweep(P, 2 * P, k)
            c1 = sweep(P, 2 * P, 1, factor=8 * k)
            rs = pl.simulate(make(cs, "seq1f1b"), pl.even_partition(cs), with_series=False)
            r1 = pl.simulate(make(c1, "1f1b"), pl.even_partition(c1), with_series=False)
            assert rs.devices[0].peak_memory < r1.devices[0].peak_memory
            assert rs.max_peak_memory < r1.max_peak_memory


def test_deadlock_and_missing_dependency():  # test_sim.cpp:230-245
    cfg = sweep(2, 2, 1)
    s = make(cfg, "1f1b")
    bad = pl.Schedule(cfg, "1f1b", [list(reversed(s.device_orders[0])), s.device_orders[1]])
    with pytest.raises(pl.DeadlockError):
        pl.simulate(bad, pl.even_partition(cfg))
    missing = pl.Schedule(cfg, "1f1b", [s.device_orders[0][1:], s.device_orders[1]])  # drop F(1,1) at stage 1
    with pytest.raises(pl.MissingDependencyError):
        pl.simulate(missing, pl.even_partition(cfg))


def test_validator_codes():  # test_validate.cpp:67-119
    cfg = sweep(2, 4, 2)
    s = make(cfg, "seq1f1b")
    o = [list(x) for x in s.device_orders]
    o[0] = o[0][:-1]
    codes = {v.code for v in pl.check_schedule(pl.Schedule(cfg, "seq1f1b", o))}
    assert "completeness" in codes and "accumulation_count" in codes
    o = [list(x) for x in s.device_orders]
    o[0], o[1] = o[1], o[0]
    assert "misplaced_task" in {v.code for v in pl.check_schedule(pl.Schedule(cfg, "seq1f1b", o))}


def test_throughput():  # test_sim.cpp:247-251
    cfg = sweep(2, 4, 1)
    rep = pl.simulate(make(cfg, "1f1b"), pl.even_partition(cfg))
    assert rep.modeled_throughput == Fraction(4 * cfg.seq_len) / rep.makespan


def test_scenario_text_round_trip():  # test_core.cpp:46-71
    cfg = pl.preset_scenario("gpt-7b")
    cfg.comm_latency = Fraction(1, 3)
    cfg.cost_model = "uniform"
    assert pl.parse_scenario_text(pl.scenario_to_text(cfg)) == cfg
