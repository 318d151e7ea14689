"""TEST INFRASTRUCTURE ONLY: ctypes access to the compiled reference planner.

oracle/_ref/libseqpipe_ref.so is the UNMODIFIED reference seqpipe core
(/root/reference/proj/core/src/*.cpp) plus oracle/ref_shim.cpp, built by
oracle/build_ref.sh. It is the parity anchor for the planning half
(partition, op tables, simulate, validate). Only tests/, __graft_entry__.smoke()
and bench.py's reference/cpu_baseline legs may use it.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

from paper_2406_03488_b200 import planner as pl
from paper_2406_03488_b200._capi import DeviceReport, Rational, Scenario, SimSummary, Task, TaskTiming

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libseqpipe_ref.so"
P = C.POINTER
_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_preset_scenario": (C.c_int, [C.c_char_p, P(Scenario)]),
    "ref_parse_scenario_text": (C.c_int, [C.c_char_p, P(Scenario)]),
    "ref_apply_override": (C.c_int, [P(Scenario), C.c_char_p, C.c_char_p]),
    "ref_scenario_validate": (C.c_int, [P(Scenario)]),
    "ref_scenario_to_text": (C.c_int, [P(Scenario), C.c_char_p, P(C.c_size_t)]),
    "ref_partition": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Rational)]),
    "ref_make_partition": (C.c_int, [P(Scenario), P(C.c_int64), C.c_int32, P(Rational)]),
    "ref_balance_report": (C.c_int, [P(Scenario), P(C.c_int64), C.c_int32, P(Rational), P(Rational)]),
    "ref_segment_flops": (C.c_int, [P(Scenario), C.c_int64, C.c_int64, P(C.c_int64), P(C.c_uint64)]),
    "ref_task_cost": (C.c_int, [P(Scenario), P(C.c_int64), P(Task), P(Rational)]),
    "ref_warmup": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_int32)]),
    "ref_schedule_ops": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Task), P(C.c_int64)]),
    "ref_dependencies": (C.c_int, [P(Task), P(Scenario), P(Task), P(C.c_int32)]),
    "ref_simulate": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Task), P(C.c_int64), P(TaskTiming),
                               P(DeviceReport), P(SimSummary)]),
    "ref_check_schedule": (C.c_int, [P(Scenario), C.c_int32, P(Task), P(C.c_int64), C.c_char_p,
                                     P(C.c_size_t), P(C.c_int32)]),
    "ref_check_warmup_formulas": (C.c_int, [P(Scenario), C.c_int32, P(Task), P(C.c_int64), C.c_char_p,
                                            P(C.c_size_t), P(C.c_int32)]),
    "ref_poq_run": (C.c_int, [P(C.c_int32), C.c_int32, P(C.c_int32), P(C.c_int32)]),
    "ref_time_planner": (C.c_int, [P(Scenario), C.c_int32, C.c_int32, C.c_int32, P(C.c_double)]),
    "ref_schedule_to_json": (C.c_int, [P(Scenario), C.c_int32, P(Task), P(C.c_int64), C.c_int32, C.c_char_p,
                                       P(C.c_size_t)]),
    "ref_schedule_json_roundtrip": (C.c_int, [C.c_char_p, C.c_int32, C.c_char_p, P(C.c_size_t)]),
    "ref_report_to_json": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Task), P(C.c_int64), C.c_int32,
                                     C.c_int64, C.c_char_p, P(C.c_size_t)]),
    "ref_render_gantt": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Task), P(C.c_int64), C.c_int32,
                                   C.c_int32, C.c_char_p, P(C.c_size_t)]),
    "ref_compare_csv": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.c_char_p, P(C.c_size_t)]),
}
_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not REF_LIB.exists():
            subprocess.run(["bash", str(HERE / "build_ref.sh")], check=True)
        if not REF_LIB.exists():
            raise RuntimeError("reference oracle library not built (needs /root/reference)")
        _lib = C.CDLL(str(REF_LIB))
        for n, (r, a) in _SIGS.items():
            f = getattr(_lib, n)
            f.restype = r
            f.argtypes = a
    return _lib


def _chk(code):
    pl._check(code, lib(), "ref_last_error")


def _frac(r):
    return pl._frac(r)


def preset_scenario(name: str) -> pl.ScenarioConfig:
    s = Scenario()
    _chk(lib().ref_preset_scenario(name.encode(), C.byref(s)))
    return pl.ScenarioConfig.from_c(s)


def parse_scenario_text(text: str) -> pl.ScenarioConfig:
    s = Scenario()
    _chk(lib().ref_parse_scenario_text(text.encode(), C.byref(s)))
    return pl.ScenarioConfig.from_c(s)


def apply_scenario_override(cfg, key, value):
    s = cfg.to_c()
    _chk(lib().ref_apply_override(C.byref(s), key.encode(), str(value).encode()))
    return pl.ScenarioConfig.from_c(s)


def validate(cfg):
    s = cfg.to_c()
    _chk(lib().ref_scenario_validate(C.byref(s)))


def scenario_to_text(cfg) -> str:
    s = cfg.to_c()
    n = C.c_size_t(0)
    _chk(lib().ref_scenario_to_text(C.byref(s), None, C.byref(n)))
    b = C.create_string_buffer(n.value)
    _chk(lib().ref_scenario_to_text(C.byref(s), b, C.byref(n)))
    return b.value.decode()


def partition_for(cfg, mode: str) -> pl.SequencePartition:
    s = cfg.to_c()
    out = (C.c_int64 * max(1, cfg.segments))()
    imb = Rational()
    _chk(lib().ref_partition(C.byref(s), pl.PARTITION_MODES.index(mode), out, C.byref(imb)))
    ls = list(out[: cfg.segments])
    return pl.SequencePartition(ls, sum(ls), _frac(imb))


def make_partition(lengths, cfg):
    s = cfg.to_c()
    imb = Rational()
    arr = (C.c_int64 * max(1, len(lengths)))(*lengths)
    _chk(lib().ref_make_partition(C.byref(s), arr, len(lengths), C.byref(imb)))
    return pl.SequencePartition(list(lengths), sum(lengths), _frac(imb))


def balance_report(p, cfg):
    s = cfg.to_c()
    k = len(p.lengths)
    costs = (Rational * k)()
    imb = Rational()
    _chk(lib().ref_balance_report(C.byref(s), (C.c_int64 * k)(*p.lengths), k, costs, C.byref(imb)))
    return [_frac(x) for x in costs], _frac(imb)


def segment_flops(cfg, before, n) -> int:
    s = cfg.to_c()
    hi, lo = C.c_int64(), C.c_uint64()
    _chk(lib().ref_segment_flops(C.byref(s), before, n, C.byref(hi), C.byref(lo)))
    return (hi.value << 64) + lo.value


def task_cost(cfg, p, t: pl.Task):
    s = cfg.to_c()
    out = Rational()
    tc = pl._task_c(t)
    _chk(lib().ref_task_cost(C.byref(s), (C.c_int64 * len(p.lengths))(*p.lengths), C.byref(tc), C.byref(out)))
    return _frac(out)


def warmup(formula, P_, a, k, d):
    out = C.c_int32()
    _chk(lib().ref_warmup(formula, P_, a, k, d, C.byref(out)))
    return out.value


def generate(cfg, kind, p) -> pl.Schedule:
    s = cfg.to_c()
    kid = pl.kind_id(kind)
    lens = (C.c_int64 * len(p.lengths))(*p.lengths)
    counts = (C.c_int64 * max(1, cfg.pipeline_size))()
    _chk(lib().ref_schedule_ops(C.byref(s), kid, lens, None, counts))
    ops = (Task * max(1, sum(counts[: cfg.pipeline_size])))()
    _chk(lib().ref_schedule_ops(C.byref(s), kid, lens, ops, counts))
    return pl.Schedule(cfg, pl.SCHEDULE_KINDS[kid], pl._unflatten(cfg.pipeline_size, ops, counts))


def dependencies(task, cfg):
    s = cfg.to_c()
    out = (Task * 3)()
    n = C.c_int32()
    t = pl._task_c(task)
    _chk(lib().ref_dependencies(C.byref(t), C.byref(s), out, C.byref(n)))
    return [pl._task_py(out[i]) for i in range(n.value)]


def simulate_raw(schedule, p):
    """(timings list, device reports, summary) as raw ctypes values for field-wise diffing."""
    cfg = schedule.config
    s = cfg.to_c()
    ops, counts = schedule.flat()
    n = sum(counts[: cfg.pipeline_size])
    timings = (TaskTiming * max(1, n))()
    devs = (DeviceReport * cfg.pipeline_size)()
    summ = SimSummary()
    _chk(lib().ref_simulate(C.byref(s), pl.kind_id(schedule.kind), (C.c_int64 * len(p.lengths))(*p.lengths), ops,
                            counts, timings, devs, C.byref(summ)))
    return timings, devs, summ, n


def check_schedule(schedule):
    return pl._violations("ref_check_schedule", schedule, lib(), "ref_last_error")


def check_warmup_formulas(schedule):
    return pl._violations("ref_check_warmup_formulas", schedule, lib(), "ref_last_error")


def poq_run(ops):
    flat = [x for op in ops for x in op]
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    pops = (C.c_int32 * (2 * max(1, len(ops))))()
    npops = C.c_int32()
    _chk(lib().ref_poq_run(arr, len(ops), pops, C.byref(npops)))
    return [(pops[2 * i], pops[2 * i + 1]) for i in range(npops.value)]


def time_planner(cfg, kind="seq1f1b", mode="cwp", reps=20) -> float:
    """Best-of-reps wall time (ns) of cwp_partition + generate + simulate + check_schedule."""
    s = cfg.to_c()
    out = C.c_double()
    _chk(lib().ref_time_planner(C.byref(s), pl.kind_id(kind), pl.PARTITION_MODES.index(mode), reps, C.byref(out)))
    return out.value


def _text(fn, *args) -> str:
    n = C.c_size_t(0)
    _chk(fn(*args, None, C.byref(n)))
    b = C.create_string_buffer(n.value)
    _chk(fn(*args, b, C.byref(n)))
    return b.value.decode()


def schedule_to_json(schedule, indent: int = 2) -> str:
    """Reference json_io.cpp:59-74 bytes of a schedule."""
    s = schedule.config.to_c()
    ops, counts = schedule.flat()
    return _text(lib().ref_schedule_to_json, C.byref(s), pl.kind_id(schedule.kind), ops, counts, indent)


def schedule_json_roundtrip(text: str, indent: int = 2) -> str:
    """Reference dump(parse(text)) (json_io.cpp:59-97)."""
    return _text(lib().ref_schedule_json_roundtrip, text.encode(), indent)


def report_to_json(schedule, p, indent: int = 2, memory_downsample: int = 0) -> str:
    """Reference json_io.cpp:99-159 bytes of simulate(schedule, p)."""
    s = schedule.config.to_c()
    ops, counts = schedule.flat()
    return _text(lib().ref_report_to_json, C.byref(s), pl.kind_id(schedule.kind),
                 (C.c_int64 * len(p.lengths))(*p.lengths), ops, counts, indent, memory_downsample)


def render_gantt(schedule, p, fmt: str = "ascii", width: int = 120) -> str:
    """Reference render.cpp:46-124 bytes of simulate(schedule, p)."""
    s = schedule.config.to_c()
    ops, counts = schedule.flat()
    return _text(lib().ref_render_gantt, C.byref(s), pl.kind_id(schedule.kind),
                 (C.c_int64 * len(p.lengths))(*p.lengths), ops, counts, pl.RENDER_FORMATS[fmt], width)


def compare_csv(runs, allow_mixed: bool = False) -> str:
    """Reference sim.cpp:319-367: compare(simulate(...) for each run).to_csv()."""
    n, cfgs, kinds, lens, opss, cnts, _keep = pl._compare_args(runs)
    return _text(lib().ref_compare_csv, n, cfgs, kinds, lens, opss, cnts, int(allow_mixed))
