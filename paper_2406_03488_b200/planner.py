"""Python host mirror of the reference seqpipe planning API.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/core/include/seqpipe/*.hpp); every call goes through the
C-ABI of libseqpipe_b200.so (include/seqpipe_b200.h). Reference exception types
map onto Python classes of the same name:
  std::invalid_argument -> InvalidArgument(ValueError)
  UnsupportedScheduleError -> UnsupportedScheduleError(InvalidArgument)
  std::out_of_range -> OutOfRange(IndexError)
  std::domain_error -> DomainError(ArithmeticError)
  std::overflow_error -> RationalOverflow(OverflowError)
  DeadlockError / MissingDependencyError -> RuntimeError subclasses
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields
from fractions import Fraction
from typing import NamedTuple, Sequence

from . import _capi
from ._capi import Rational as _R, Scenario as _S, Task as _T


class InvalidArgument(ValueError):
    pass


class UnsupportedScheduleError(InvalidArgument):
    pass


class OutOfRange(IndexError):
    pass


class DomainError(ArithmeticError):
    pass


class RationalOverflow(OverflowError):
    pass


class DeadlockError(RuntimeError):
    pass


class MissingDependencyError(RuntimeError):
    pass


class LogicError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_EXC = {1: InvalidArgument, 2: UnsupportedScheduleError, 3: OutOfRange, 4: DomainError,
        5: RationalOverflow, 6: DeadlockError, 7: MissingDependencyError, 8: LogicError,
        9: RuntimeError, 10: CudaError, 11: CudaError, 12: RuntimeError}


def _check(code: int, handle=None, err_fn: str = "sp_last_error"):
    if code != 0:
        h = handle or _capi.lib()
        raise _EXC.get(code, RuntimeError)(getattr(h, err_fn)().decode())


SCHEDULE_KINDS = ("gpipe", "1f1b", "1f1b-i", "seq1f1b", "seq1f1b-i", "zb1p", "seqzb1p")
PARTITION_MODES = ("even", "cwp", "oracle")
TASK_KINDS = ("F", "B", "I", "W")


def kind_id(kind) -> int:
    if isinstance(kind, int):
        return kind
    k = str(kind).lower()
    if k not in SCHEDULE_KINDS:
        raise InvalidArgument(f"unknown schedule kind '{kind}'")
    return SCHEDULE_KINDS.index(k)


def is_sequence_level(kind) -> bool:
    return SCHEDULE_KINDS[kind_id(kind)] in ("seq1f1b", "seq1f1b-i", "seqzb1p")


def is_interleaved(kind) -> bool:
    return SCHEDULE_KINDS[kind_id(kind)] in ("1f1b-i", "seq1f1b-i")


def is_zero_bubble(kind) -> bool:
    return SCHEDULE_KINDS[kind_id(kind)] in ("zb1p", "seqzb1p")


def _frac(r: _R) -> Fraction:
    return Fraction(r.num, r.den)


def _rat(x) -> _R:
    f = Fraction(x)
    return _R(f.numerator, f.denominator)


_RAT_FIELDS = ("backward_ratio", "bw_input_ratio", "bw_weight_ratio", "comm_latency",
               "activation_cost_per_token", "time_per_flop", "uniform_forward")


@dataclass
class ScenarioConfig:
    """ScenarioConfig (scenario.hpp:25-50). Rational fields are Fractions."""
    pipeline_size: int = 1
    stages_per_device: int = 1
    micro_batches: int = 1
    segments: int = 1
    seq_len: int = 1
    layers: int = 1
    hidden_dim: int = 1
    param_count: int = 0
    backward_ratio: Fraction = Fraction(2)
    bw_input_ratio: Fraction = Fraction(1)
    bw_weight_ratio: Fraction = Fraction(1)
    comm_latency: Fraction = Fraction(0)
    activation_cost_per_token: Fraction = Fraction(1)
    time_per_flop: Fraction = Fraction(1)
    cost_model: str = "flops"
    uniform_forward: Fraction = Fraction(1)

    def total_stages(self) -> int:
        return self.pipeline_size * self.stages_per_device

    def to_c(self) -> _S:
        s = _S()
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name in _RAT_FIELDS:
                setattr(s, f.name, _rat(v))
            elif f.name == "cost_model":
                if v not in ("flops", "uniform"):
                    raise InvalidArgument(f"unknown cost_model '{v}'")
                s.cost_model = 1 if v == "uniform" else 0
            else:
                setattr(s, f.name, int(v))
        return s

    @classmethod
    def from_c(cls, s: _S) -> "ScenarioConfig":
        kw = {}
        for f in fields(cls):
            v = getattr(s, f.name)
            if f.name in _RAT_FIELDS:
                kw[f.name] = _frac(v)
            elif f.name == "cost_model":
                kw[f.name] = "uniform" if v == 1 else "flops"
            else:
                kw[f.name] = int(v)
        return cls(**kw)

    def validate(self) -> None:
        c = self.to_c()
        _check(_capi.lib().sp_scenario_validate(C.byref(c)))


def preset_scenario(name: str) -> ScenarioConfig:
    s = _S()
    _check(_capi.lib().sp_preset_scenario(name.encode(), C.byref(s)))
    return ScenarioConfig.from_c(s)


def preset_names():
    return ["gpt-2.7b", "gpt-7b", "gpt-13b", "gpt-30b"]


def parse_scenario_text(text: str) -> ScenarioConfig:
    s = _S()
    _check(_capi.lib().sp_parse_scenario_text(text.encode(), C.byref(s)))
    return ScenarioConfig.from_c(s)


def load_scenario_file(path: str) -> ScenarioConfig:
    with open(path) as f:
        return parse_scenario_text(f.read())


def apply_scenario_override(cfg: ScenarioConfig, key: str, value: str) -> ScenarioConfig:
    """Applies key=value in place (and returns cfg for chaining)."""
    s = cfg.to_c()
    _check(_capi.lib().sp_apply_override(C.byref(s), key.encode(), str(value).encode()))
    new = ScenarioConfig.from_c(s)
    for f in fields(cfg):
        setattr(cfg, f.name, getattr(new, f.name))
    return cfg


def scenario_to_text(cfg: ScenarioConfig) -> str:
    s = cfg.to_c()
    n = C.c_size_t(0)
    _check(_capi.lib().sp_scenario_to_text(C.byref(s), None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(_capi.lib().sp_scenario_to_text(C.byref(s), buf, C.byref(n)))
    return buf.value.decode()


# ------------------------------------------------------------------ partitions / cost

@dataclass
class SequencePartition:
    lengths: list
    total: int
    imbalance: Fraction = Fraction(0)

    def segment_count(self) -> int:
        return len(self.lengths)

    def prefix(self, i: int) -> int:
        return sum(self.lengths[:i])


def _lengths(p) -> C.Array:
    ls = p.lengths if isinstance(p, SequencePartition) else list(p)
    return (C.c_int64 * len(ls))(*ls)


def make_partition(lengths: Sequence[int], cfg: ScenarioConfig) -> SequencePartition:
    c = cfg.to_c()
    imb = _R()
    arr = (C.c_int64 * max(1, len(lengths)))(*lengths)
    _check(_capi.lib().sp_make_partition(C.byref(c), arr, len(lengths), C.byref(imb)))
    return SequencePartition(list(lengths), sum(lengths), _frac(imb))


def partition_for(cfg: ScenarioConfig, mode: str) -> SequencePartition:
    if mode not in PARTITION_MODES:
        raise InvalidArgument(f"unknown partition mode '{mode}'")
    c = cfg.to_c()
    out = (C.c_int64 * max(1, cfg.segments))()
    imb = _R()
    _check(_capi.lib().sp_partition(C.byref(c), PARTITION_MODES.index(mode), out, C.byref(imb)))
    ls = list(out[: cfg.segments])
    return SequencePartition(ls, sum(ls), _frac(imb))


def even_partition(cfg_or_n, k: int | None = None, cfg: ScenarioConfig | None = None) -> SequencePartition:
    if isinstance(cfg_or_n, ScenarioConfig):
        return partition_for(cfg_or_n, "even")
    n = int(cfg_or_n)
    c = cfg.to_c()
    out = (C.c_int64 * max(1, k))()
    imb = _R()
    _check(_capi.lib().sp_even_partition(n, k, C.byref(c), out, C.byref(imb)))
    ls = list(out[:k])
    return SequencePartition(ls, sum(ls), _frac(imb))


def cwp_partition(cfg: ScenarioConfig) -> SequencePartition:
    return partition_for(cfg, "cwp")


def oracle_partition(cfg: ScenarioConfig) -> SequencePartition:
    return partition_for(cfg, "oracle")


def balance_report(p: SequencePartition, cfg: ScenarioConfig):
    c = cfg.to_c()
    k = len(p.lengths)
    costs = (_R * k)()
    imb = _R()
    _check(_capi.lib().sp_balance_report(C.byref(c), _lengths(p), k, costs, C.byref(imb)))
    return [_frac(x) for x in costs], _frac(imb)


def segment_flops(cfg: ScenarioConfig, prefix_before: int, length: int) -> int:
    c = cfg.to_c()
    hi, lo = C.c_int64(), C.c_uint64()
    _check(_capi.lib().sp_segment_flops(C.byref(c), prefix_before, length, C.byref(hi), C.byref(lo)))
    return (hi.value << 64) + lo.value


def forward_cost(cfg: ScenarioConfig, p: SequencePartition, i: int) -> Fraction:
    c = cfg.to_c()
    out = _R()
    _check(_capi.lib().sp_forward_cost(C.byref(c), _lengths(p), len(p.lengths), i, C.byref(out)))
    return _frac(out)


class Task(NamedTuple):
    kind: str
    micro_batch: int
    segment: int
    stage: int
    device: int

    def brief(self) -> str:
        return f"{self.kind}{self.micro_batch}.{self.segment}"


def make_task(kind: str, m: int, s: int, stage: int, pipeline_size: int) -> Task:
    return Task(kind, m, s, stage, (stage - 1) % pipeline_size + 1)


def _task_c(t: Task) -> _T:
    return _T(TASK_KINDS.index(t.kind), t.micro_batch, t.segment, t.stage, t.device)


def _task_py(t: _T) -> Task:
    return Task(TASK_KINDS[t.kind], t.micro_batch, t.segment, t.stage, t.device)


def task_cost(cfg: ScenarioConfig, p: SequencePartition, t: Task) -> Fraction:
    c = cfg.to_c()
    out = _R()
    tc = _task_c(t)
    _check(_capi.lib().sp_task_cost(C.byref(c), _lengths(p), len(p.lengths), C.byref(tc), C.byref(out)))
    return _frac(out)


# ------------------------------------------------------------------ schedules

def _warm(formula, P, a, k, d):
    out = C.c_int32()
    _check(_capi.lib().sp_warmup(formula, P, a, k, d, C.byref(out)))
    return out.value


def warmup_1f1b(P, M, d):
    return _warm(0, P, M, 1, d)


def warmup_seq1f1b(P, M, k, d):
    return _warm(1, P, M, k, d)


def warmup_1f1b_interleaved(P, nv, d):
    return _warm(2, P, nv, 1, d)


def warmup_seq1f1b_interleaved(P, nv, k, d):
    return _warm(3, P, nv, k, d)


@dataclass
class Schedule:
    config: ScenarioConfig
    kind: str
    device_orders: list = field(default_factory=list)

    def flat(self):
        """(ops array, counts array) in the C layout."""
        n = sum(len(o) for o in self.device_orders)
        ops = (_T * max(1, n))()
        counts = (C.c_int64 * max(1, len(self.device_orders)))()
        i = 0
        for d, order in enumerate(self.device_orders):
            counts[d] = len(order)
            for t in order:
                ops[i] = _task_c(t)
                i += 1
        return ops, counts

    def __eq__(self, other):
        return (isinstance(other, Schedule) and self.config == other.config
                and self.kind == other.kind and self.device_orders == other.device_orders)


def _unflatten(P: int, ops, counts):
    orders, off = [], 0
    for d in range(P):
        n = counts[d]
        orders.append([_task_py(ops[off + i]) for i in range(n)])
        off += n
    return orders


def generate(cfg: ScenarioConfig, kind, partition: SequencePartition) -> Schedule:
    c = cfg.to_c()
    kid = kind_id(kind)
    lens = _lengths(partition)
    counts = (C.c_int64 * max(1, cfg.pipeline_size))()
    _check(_capi.lib().sp_schedule_ops(C.byref(c), kid, lens, None, counts))
    total = sum(counts[: cfg.pipeline_size])
    ops = (_T * max(1, total))()
    _check(_capi.lib().sp_schedule_ops(C.byref(c), kid, lens, ops, counts))
    return Schedule(cfg, SCHEDULE_KINDS[kid], _unflatten(cfg.pipeline_size, ops, counts))


def device_schedule(cfg: ScenarioConfig, kind, cuda_device: int = 0) -> Schedule:
    """Op tables generated by the GPU-resident launcher kernel (gpipe / 1f1b / seq1f1b)."""
    c = cfg.to_c()
    kid = kind_id(kind)
    counts = (C.c_int64 * max(1, cfg.pipeline_size))()
    n = 2 * cfg.micro_batches * cfg.segments * cfg.pipeline_size
    ops = (_T * max(1, n))()
    _check(_capi.lib().sp_device_schedule_ops(C.byref(c), kid, cuda_device, ops, counts))
    return Schedule(cfg, SCHEDULE_KINDS[kid], _unflatten(cfg.pipeline_size, ops, counts))


def device_partition(cfg: ScenarioConfig, mode: str = "cwp", cuda_device: int = 0) -> list:
    c = cfg.to_c()
    out = (C.c_int64 * max(1, cfg.segments))()
    _check(_capi.lib().sp_device_partition(C.byref(c), PARTITION_MODES.index(mode), cuda_device, out))
    return list(out[: cfg.segments])


def dependencies(task: Task, cfg: ScenarioConfig):
    c = cfg.to_c()
    out = (_T * 3)()
    n = C.c_int32()
    t = _task_c(task)
    _check(_capi.lib().sp_dependencies(C.byref(t), C.byref(c), out, C.byref(n)))
    return [_task_py(out[i]) for i in range(n.value)]


# ------------------------------------------------------------------ simulate / validate

@dataclass
class DeviceReport:
    device: int
    first_start: Fraction
    last_end: Fraction
    busy: Fraction
    idle: Fraction
    bubble_ratio: Fraction
    idle_in_makespan: Fraction
    bubble_ratio_in_makespan: Fraction
    peak_memory: Fraction
    peak_allocations: int
    warmup_forward_tasks: int
    memory_series: list


@dataclass
class SimReport:
    kind: str
    config: ScenarioConfig
    partition_lengths: list
    task_times: list
    makespan: Fraction
    devices: list
    aggregate_bubble_ratio: Fraction
    aggregate_bubble_ratio_in_makespan: Fraction
    max_peak_memory: Fraction
    modeled_throughput: Fraction


def simulate(schedule: Schedule, partition: SequencePartition, with_series: bool = True) -> SimReport:
    cfg = schedule.config
    c = cfg.to_c()
    kid = kind_id(schedule.kind)
    ops, counts = schedule.flat()
    n = sum(counts[: cfg.pipeline_size])
    timings = (_capi.TaskTiming * max(1, n))()
    devs = (_capi.DeviceReport * max(1, cfg.pipeline_size))()
    summ = _capi.SimSummary()
    lens = _lengths(partition)
    _check(_capi.lib().sp_simulate(C.byref(c), kid, lens, ops, counts, timings, devs, C.byref(summ)))
    tt, off = [], 0
    for d in range(cfg.pipeline_size):
        tt.append([(_task_py(timings[off + i].task), _frac(timings[off + i].start), _frac(timings[off + i].end))
                   for i in range(counts[d])])
        off += counts[d]
    devices = []
    for d in range(cfg.pipeline_size):
        r = devs[d]
        series = []
        if with_series:
            ln = C.c_int64(r.memory_series_len)
            buf = (_R * max(2, 2 * ln.value))()
            _check(_capi.lib().sp_simulate_memory_series(C.byref(c), kid, lens, ops, counts, d + 1, buf, C.byref(ln)))
            series = [(_frac(buf[2 * i]), _frac(buf[2 * i + 1])) for i in range(ln.value)]
        devices.append(DeviceReport(r.device, _frac(r.first_start), _frac(r.last_end), _frac(r.busy), _frac(r.idle),
                                    _frac(r.bubble_ratio), _frac(r.idle_in_makespan),
                                    _frac(r.bubble_ratio_in_makespan), _frac(r.peak_memory), r.peak_allocations,
                                    r.warmup_forward_tasks, series))
    return SimReport(SCHEDULE_KINDS[kid], cfg, list(partition.lengths), tt, _frac(summ.makespan), devices,
                     _frac(summ.aggregate_bubble_ratio), _frac(summ.aggregate_bubble_ratio_in_makespan),
                     _frac(summ.max_peak_memory), _frac(summ.modeled_throughput))


class Violation(NamedTuple):
    code: str
    device: int
    detail: str


def _violations(fn_name: str, schedule: Schedule, handle=None, err_fn="sp_last_error"):
    h = handle or _capi.lib()
    fn = getattr(h, fn_name)
    c = schedule.config.to_c()
    ops, counts = schedule.flat()
    n = C.c_size_t(0)
    nv = C.c_int32(0)
    _check(fn(C.byref(c), kind_id(schedule.kind), ops, counts, None, C.byref(n), C.byref(nv)), h, err_fn)
    buf = C.create_string_buffer(n.value)
    _check(fn(C.byref(c), kind_id(schedule.kind), ops, counts, buf, C.byref(n), C.byref(nv)), h, err_fn)
    out = []
    for line in buf.value.decode().splitlines():
        code, dev, detail = line.split("\t", 2)
        out.append(Violation(code, int(dev), detail))
    return out


def check_schedule(schedule: Schedule):
    return _violations("sp_check_schedule", schedule)


def check_warmup_formulas(schedule: Schedule):
    return _violations("sp_check_warmup_formulas", schedule)


def violations_to_string(vs) -> str:
    return "".join(f"{v.code}{f' [device {v.device}]' if v.device > 0 else ''}: {v.detail}\n" for v in vs)


# ---------------------------------------------------------------- JSON wire formats
# seqpipe.schedule.v1 / seqpipe.simreport.v1 (reference core/include/seqpipe/json_io.hpp:19-26).

def _text_out(fn, *args) -> str:
    n = C.c_size_t(0)
    _check(fn(*args, None, C.byref(n)))
    b = C.create_string_buffer(n.value)
    _check(fn(*args, b, C.byref(n)))
    return b.value.decode()


def schedule_to_json(schedule: Schedule, indent: int = 2) -> str:
    c = schedule.config.to_c()
    ops, counts = schedule.flat()
    return _text_out(_capi.lib().sp_schedule_to_json, C.byref(c), kind_id(schedule.kind), ops, counts, indent)


def schedule_from_json(text: str, max_devices: int = 4096) -> Schedule:
    c = _capi.Scenario()
    kind = C.c_int32(0)
    counts = (C.c_int64 * max_devices)()
    raw = text.encode()
    _check(_capi.lib().sp_schedule_from_json(raw, C.byref(c), C.byref(kind), None, counts, max_devices))
    cfg = ScenarioConfig.from_c(c)
    total = sum(counts[: cfg.pipeline_size])
    ops = (_T * max(1, total))()
    _check(_capi.lib().sp_schedule_from_json(raw, C.byref(c), C.byref(kind), ops, counts, max_devices))
    return Schedule(cfg, SCHEDULE_KINDS[kind.value], _unflatten(cfg.pipeline_size, ops, counts))


def report_to_json(schedule: Schedule, partition: SequencePartition, indent: int = 2,
                   memory_downsample: int = 0) -> str:
    """simulate(schedule, partition) serialised as seqpipe.simreport.v1."""
    c = schedule.config.to_c()
    ops, counts = schedule.flat()
    return _text_out(_capi.lib().sp_report_to_json, C.byref(c), kind_id(schedule.kind), _lengths(partition), ops,
                     counts, indent, memory_downsample)


RENDER_FORMATS = {"ascii": 0, "svg": 1}


def render_gantt(schedule: Schedule, partition: SequencePartition, fmt: str = "ascii", width: int = 120) -> str:
    """Timeline of simulate(schedule, partition): render_ascii_gantt (width cells per device row) or
    render_svg_gantt (reference render.hpp:15-21, render.cpp:46-124)."""
    c = schedule.config.to_c()
    ops, counts = schedule.flat()
    return _text_out(_capi.lib().sp_render_gantt, C.byref(c), kind_id(schedule.kind), _lengths(partition), ops, counts,
                     RENDER_FORMATS[fmt], width)


def _compare_args(runs):
    n = len(runs)
    cfgs = (_capi.Scenario * max(1, n))()
    kinds = (C.c_int32 * max(1, n))()
    keep, lens, opss, cnts = [], (C.c_void_p * max(1, n))(), (C.c_void_p * max(1, n))(), (C.c_void_p * max(1, n))()
    for i, (sch, part) in enumerate(runs):
        cfgs[i] = sch.config.to_c()
        kinds[i] = kind_id(sch.kind)
        ops, counts = sch.flat()
        ls = _lengths(part)
        keep += [ops, counts, ls]
        lens[i], opss[i], cnts[i] = C.addressof(ls), C.addressof(ops), C.addressof(counts)
    return n, cfgs, kinds, lens, opss, cnts, keep


def compare_csv(runs, allow_mixed: bool = False) -> str:
    """compare() of the simulations of [(schedule, partition), ...] as ComparisonTable::to_csv
    (reference sim.hpp:82-99, sim.cpp:319-367). Raises InvalidArgument for < 2 runs or mixed
    workloads without allow_mixed."""
    n, cfgs, kinds, lens, opss, cnts, _keep = _compare_args(runs)
    return _text_out(_capi.lib().sp_compare_csv, n, cfgs, kinds, lens, opss, cnts, int(allow_mixed))
