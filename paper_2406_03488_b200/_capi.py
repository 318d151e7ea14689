"""ctypes declarations of the C-ABI in include/seqpipe_b200.h.

The product library is paper_2406_03488_b200/lib/libseqpipe_b200.so, built in
tree by build.py. Loading fails loudly when it is missing: there is no Python
or CPU fallback for anything this package exposes.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libseqpipe_b200.so"

SP_OK = 0
ERR_NAMES = {
    1: "invalid_argument", 2: "unsupported", 3: "out_of_range", 4: "domain_error",
    5: "overflow_error", 6: "deadlock", 7: "missing_dependency", 8: "logic_error",
    9: "runtime_error", 10: "cuda", 11: "nccl", 12: "buffer_too_small",
}


class Rational(C.Structure):
    _fields_ = [("num", C.c_int64), ("den", C.c_int64)]


class Scenario(C.Structure):
    _fields_ = [
        ("pipeline_size", C.c_int32), ("stages_per_device", C.c_int32),
        ("micro_batches", C.c_int32), ("segments", C.c_int32),
        ("seq_len", C.c_int64), ("layers", C.c_int32), ("cost_model", C.c_int32),
        ("hidden_dim", C.c_int64), ("param_count", C.c_int64),
        ("backward_ratio", Rational), ("bw_input_ratio", Rational), ("bw_weight_ratio", Rational),
        ("comm_latency", Rational), ("activation_cost_per_token", Rational),
        ("time_per_flop", Rational), ("uniform_forward", Rational),
    ]


class Task(C.Structure):
    _fields_ = [("kind", C.c_int32), ("micro_batch", C.c_int32), ("segment", C.c_int32),
                ("stage", C.c_int32), ("device", C.c_int32)]


class TaskTiming(C.Structure):
    _fields_ = [("task", Task), ("start", Rational), ("end", Rational)]


class DeviceReport(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("warmup_forward_tasks", C.c_int32), ("peak_allocations", C.c_int64),
        ("first_start", Rational), ("last_end", Rational), ("busy", Rational), ("idle", Rational),
        ("bubble_ratio", Rational), ("idle_in_makespan", Rational),
        ("bubble_ratio_in_makespan", Rational), ("peak_memory", Rational),
        ("memory_series_len", C.c_int64),
    ]


class SimSummary(C.Structure):
    _fields_ = [("makespan", Rational), ("aggregate_bubble_ratio", Rational),
                ("aggregate_bubble_ratio_in_makespan", Rational), ("max_peak_memory", Rational),
                ("modeled_throughput", Rational)]


class Model(C.Structure):
    _fields_ = [
        ("family", C.c_int32), ("dtype", C.c_int32), ("vocab", C.c_int32), ("hidden", C.c_int32),
        ("layers", C.c_int32), ("heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
        ("max_seq", C.c_int64), ("seed", C.c_uint64), ("init_std", C.c_float), ("norm_eps", C.c_float),
        ("rope_theta", C.c_float), ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
        ("adam_eps", C.c_float), ("weight_decay", C.c_float), ("flags", C.c_int32), ("reserved", C.c_int32),
    ]


class StepReport(C.Structure):
    _fields_ = [
        ("step_ms", C.c_double), ("busy_ms", C.c_double), ("first_start_ms", C.c_double),
        ("last_end_ms", C.c_double), ("bubble_ratio", C.c_double), ("loss", C.c_double),
        ("peak_activation_bytes", C.c_double), ("arena_bytes", C.c_double), ("weight_bytes", C.c_double),
        ("ops_executed", C.c_int64), ("kernel_launches", C.c_int64), ("dominant_kernel_ms", C.c_double),
        ("dominant_kernel_launches", C.c_int64), ("dominant_kernel_flops", C.c_double),
        ("dominant_kernel_class", C.c_int32), ("reserved0", C.c_int32),
        ("class_ms", C.c_double * 3), ("class_flops", C.c_double * 3), ("class_launches", C.c_int64 * 3),
    ]


class CommOp(C.Structure):
    _fields_ = [("op_index", C.c_int32), ("when", C.c_int32), ("dir", C.c_int32), ("peer", C.c_int32),
                ("channel", C.c_int32), ("kind", C.c_int32), ("micro_batch", C.c_int32), ("segment", C.c_int32),
                ("stage", C.c_int32), ("reserved", C.c_int32), ("elems", C.c_int64)]


P = C.POINTER
_SIGS = {
    "sp_comm_plan": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), C.c_int32, C.c_int64, P(CommOp), P(C.c_int64)]),
    "sp_last_error": (C.c_char_p, []),
    "sp_version": (C.c_char_p, []),
    "sp_scenario_default": (None, [P(Scenario)]),
    "sp_scenario_validate": (C.c_int, [P(Scenario)]),
    "sp_preset_scenario": (C.c_int, [C.c_char_p, P(Scenario)]),
    "sp_apply_override": (C.c_int, [P(Scenario), C.c_char_p, C.c_char_p]),
    "sp_parse_scenario_text": (C.c_int, [C.c_char_p, P(Scenario)]),
    "sp_scenario_to_text": (C.c_int, [P(Scenario), C.c_char_p, P(C.c_size_t)]),
    "sp_segment_flops": (C.c_int, [P(Scenario), C.c_int64, C.c_int64, P(C.c_int64), P(C.c_uint64)]),
    "sp_forward_cost": (C.c_int, [P(Scenario), P(C.c_int64), C.c_int32, C.c_int32, P(Rational)]),
    "sp_task_cost": (C.c_int, [P(Scenario), P(C.c_int64), C.c_int32, P(Task), P(Rational)]),
    "sp_partition": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Rational)]),
    "sp_even_partition": (C.c_int, [C.c_int64, C.c_int32, P(Scenario), P(C.c_int64), P(Rational)]),
    "sp_make_partition": (C.c_int, [P(Scenario), P(C.c_int64), C.c_int32, P(Rational)]),
    "sp_balance_report": (C.c_int, [P(Scenario), P(C.c_int64), C.c_int32, P(Rational), P(Rational)]),
    "sp_warmup": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_int32)]),
    "sp_schedule_ops": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Task), P(C.c_int64)]),
    "sp_dependencies": (C.c_int, [P(Task), P(Scenario), P(Task), P(C.c_int32)]),
    "sp_simulate": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Task), P(C.c_int64),
                              P(TaskTiming), P(DeviceReport), P(SimSummary)]),
    "sp_simulate_memory_series": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Task), P(C.c_int64),
                                            C.c_int32, P(Rational), P(C.c_int64)]),
    "sp_check_schedule": (C.c_int, [P(Scenario), C.c_int32, P(Task), P(C.c_int64), C.c_char_p,
                                    P(C.c_size_t), P(C.c_int32)]),
    "sp_check_warmup_formulas": (C.c_int, [P(Scenario), C.c_int32, P(Task), P(C.c_int64), C.c_char_p,
                                           P(C.c_size_t), P(C.c_int32)]),
    "sp_device_partition": (C.c_int, [P(Scenario), C.c_int32, C.c_int32, P(C.c_int64)]),
    "sp_device_schedule_ops": (C.c_int, [P(Scenario), C.c_int32, C.c_int32, P(Task), P(C.c_int64)]),
    "sp_engine_create": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Model), C.c_int32, C.c_int32,
                                   C.c_int32, P(C.c_void_p)]),
    "sp_engine_destroy": (C.c_int, [C.c_void_p]),
    "sp_plan_memory": (C.c_int, [P(Scenario), C.c_int32, P(C.c_int64), P(Model), C.c_int32, P(C.c_double),
                                 P(C.c_double), P(C.c_double)]),
    "sp_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_size_t]),
    "sp_engine_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, P(C.c_size_t)]),
    "sp_engine_ipc_connect": (C.c_int, [C.c_void_p, P(C.c_void_p), P(C.c_size_t), C.c_int32]),
    "sp_engine_comm_init": (C.c_int, [C.c_void_p, P(C.c_char_p), C.c_int32]),
    "sp_engine_comm_channels": (C.c_int, [C.c_void_p, P(C.c_int32)]),
    "sp_local_hub_create": (C.c_int, [C.c_int32, C.c_double, P(C.c_void_p)]),
    "sp_local_hub_destroy": (C.c_int, [C.c_void_p]),
    "sp_engine_attach_local": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sp_engine_enable_graph": (C.c_int, [C.c_void_p, C.c_int32]),
    "sp_engine_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, P(StepReport)]),
    "sp_engine_set_flags": (C.c_int, [C.c_void_p, C.c_int32]),
    "sp_engine_op_log": (C.c_int, [C.c_void_p, P(Task), P(C.c_int64)]),
    "sp_engine_timeline": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_int64)]),
    "sp_engine_param_count": (C.c_int, [C.c_void_p, P(C.c_int64)]),
    "sp_engine_param_info": (C.c_int, [C.c_void_p, C.c_int64, C.c_char_p, C.c_size_t, P(C.c_int64),
                                       P(C.c_int32), P(C.c_int32)]),
    "sp_engine_read_param": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_float), C.c_int64]),
    "sp_engine_read_grad": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_float), C.c_int64]),
    "sp_engine_write_param": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_float), C.c_int64]),
    "sp_engine_memory": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_double)]),
    "sp_engine_report_json": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_char_p, P(C.c_size_t)]),
    "sp_gemm": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                          C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]),
    "sp_attention_fwd": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_void_p]),
    "sp_attention_bwd": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                   C.c_int32, C.c_int32, C.c_void_p]),
    "sp_schedule_to_json": (C.c_int, [P(Scenario), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_char_p,
                                      P(C.c_size_t)]),
    "sp_schedule_from_json": (C.c_int, [C.c_char_p, P(Scenario), P(C.c_int32), C.c_void_p, C.c_void_p, C.c_int32]),
    "sp_report_to_json": (C.c_int, [P(Scenario), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64,
                                    C.c_char_p, P(C.c_size_t)]),
    "sp_render_gantt": (C.c_int, [P(Scenario), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                  C.c_char_p, P(C.c_size_t)]),
    "sp_compare_csv": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                 C.c_char_p, P(C.c_size_t)]),
    "sp_engine_render_gantt": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, P(C.c_size_t)]),
    "sp_norm_fwd": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_int64, C.c_int32, C.c_float, C.c_void_p]),
    "sp_norm_bwd": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "sp_act_fwd": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "sp_act_bwd": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                             C.c_void_p]),
    "sp_device_synchronize": (C.c_int, [C.c_int32]),
    "sp_cuda_device_count": (C.c_int, [P(C.c_int32)]),
}
EXPORTED = tuple(_SIGS)

_lib = None
MISSING: list = []


class SeqpipeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERR_NAMES.get(code, code)}] {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))


def lib():
    """Load libseqpipe_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2406_03488_b200.build` "
                               "(no CPU/Python fallback exists)")
        for var in ("SP_LIB_VARIANT", "SP_ATTN_DBG", "SP_ATTN_TRACE"):
            if os.environ.get(var):  # profiling-only knobs of earlier tuning builds: refuse, never honour
                raise RuntimeError(f"{var} is set: the product library has no debug / variant switches "
                                   "(profiling builds live under tools/); unset it")
        _lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(_lib, name, None)
            if fn is None:
                MISSING.append(name)
                continue
            fn.restype = res
            fn.argtypes = args
    return _lib


def check(code: int, lib_handle=None, err_fn: str = "sp_last_error"):
    if code != SP_OK:
        h = lib_handle or lib()
        raise SeqpipeError(code, getattr(h, err_fn)().decode())
