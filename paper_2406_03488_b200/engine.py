"""Python handle over the sm_100a Seq1F1B execution engine (sp_engine_* C-ABI).

`Engine(cfg, kind, partition, model)` runs every pipeline stage of `cfg` on one
GPU when world_size == 1 (single-GPU validation layout) or one device's stages
when launched one process per GPU (world_size == pipeline_size, NCCL P2P).
There is no Python/CPU execution path: every call goes to libseqpipe_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from . import planner as pl

GPT, LLAMA = 0, 1
F32, BF16 = 0, 1
FLAG_NO_TCGEN05, FLAG_NO_TC_ATTN, FLAG_TIMELINE, FLAG_KPROBE, FLAG_RECOMPUTE_MLP = 1, 2, 4, 8, 16


@dataclass
class ModelConfig:
    family: int = GPT
    dtype: int = BF16
    vocab: int = 50257
    hidden: int = 256
    layers: int = 8
    heads: int = 4
    head_dim: int = 64
    ffn: int = 1024
    max_seq: int = 2048
    seed: int = 42
    init_std: float = 0.02
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0
    lr: float = 0.0
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    weight_decay: float = 0.0
    flags: int = 0

    def to_c(self) -> _capi.Model:
        m = _capi.Model()
        for k, v in self.__dict__.items():
            setattr(m, k, v)
        return m

    def param_count(self) -> int:
        """Exact trainable parameter count of the instantiated model (untied head)."""
        h, L, F, V = self.hidden, self.layers, self.ffn, self.vocab
        fup = 2 * F if self.family == LLAMA else F
        per_layer = 2 * h + 3 * h * h + h * h + fup * h + h * F
        emb = V * h + (self.max_seq * h if self.family == GPT else 0)
        return emb + L * per_layer + h + V * h


def _check(code):
    pl._check(code)


class Engine:
    def __init__(self, cfg: pl.ScenarioConfig, kind, partition: pl.SequencePartition, model: ModelConfig,
                 rank: int = 0, world_size: int = 1, cuda_device: int = 0):
        self.cfg, self.kind, self.partition, self.model = cfg, pl.SCHEDULE_KINDS[pl.kind_id(kind)], partition, model
        self.rank, self.world_size = rank, world_size
        self._h = C.c_void_p()
        c = cfg.to_c()
        lens = (C.c_int64 * len(partition.lengths))(*partition.lengths)
        mc = model.to_c()
        _check(_capi.lib().sp_engine_create(C.byref(c), pl.kind_id(kind), lens, C.byref(mc), rank, world_size,
                                            cuda_device, C.byref(self._h)))

    def close(self):
        if self._h:
            _capi.lib().sp_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_flags(self, flags: int):
        self.model.flags = flags
        _check(_capi.lib().sp_engine_set_flags(self._h, flags))

    def comm_channels(self) -> int:
        """Number of P2P channels (pipeline edges x 2 directions): NCCL ids comm_init needs."""
        n = C.c_int32()
        _check(_capi.lib().sp_engine_comm_channels(self._h, C.byref(n)))
        return n.value

    def comm_init(self, ids: list):
        """NCCL data plane: one unique id per channel (rank 0 creates them, every rank passes all)."""
        arr = (C.c_char_p * len(ids))(*ids)
        _check(_capi.lib().sp_engine_comm_init(self._h, arr, len(ids)))

    def ipc_export(self) -> bytes:
        """Peer-memory data plane (one process per GPU, CUDA IPC), phase 1: this rank's blob."""
        n = C.c_size_t(0)
        _check(_capi.lib().sp_engine_ipc_export(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(_capi.lib().sp_engine_ipc_export(self._h, buf, C.byref(n)))
        return buf.raw[: n.value]

    def ipc_connect(self, blobs: list):
        """Phase 2: every rank's blob, in rank order (exchanged over any side channel)."""
        keep = [C.create_string_buffer(b, len(b)) for b in blobs]
        ptrs = (C.c_void_p * len(blobs))(*[C.cast(k, C.c_void_p) for k in keep])
        lens = (C.c_size_t * len(blobs))(*[len(b) for b in blobs])
        _check(_capi.lib().sp_engine_ipc_connect(self._h, ptrs, lens, len(blobs)))

    def attach_local(self, hub: "LocalHub"):
        """In-process data plane: several engines of one process (one host thread each)."""
        self._hub = hub  # keep the hub alive as long as the engine
        _check(_capi.lib().sp_engine_attach_local(self._h, hub._h))

    def enable_graph(self, on: bool = True):
        """Capture the step body into a CUDA graph on the next step and replay it (world size 1)."""
        _check(_capi.lib().sp_engine_enable_graph(self._h, 1 if on else 0))

    def memory(self):
        """(bytes allocated on the engine's device, bytes free) after a synchronize."""
        a, f = C.c_double(), C.c_double()
        _check(_capi.lib().sp_engine_memory(self._h, C.byref(a), C.byref(f)))
        return a.value, f.value

    def step(self, tokens, on_device: bool = False) -> _capi.StepReport:
        """One training step (all micro-batches, optimizer included). tokens: int32 [M, T+1]
        host array, or a device pointer (int) when on_device."""
        rep = _capi.StepReport()
        if on_device:
            ptr = C.c_void_p(int(tokens))
        else:
            tok = np.ascontiguousarray(tokens, dtype=np.int32)
            assert tok.shape == (self.cfg.micro_batches, self.cfg.seq_len + 1), tok.shape
            ptr = tok.ctypes.data_as(C.c_void_p)
        _check(_capi.lib().sp_engine_step(self._h, ptr, 1 if on_device else 0, C.byref(rep)))
        return rep

    def report_json(self, indent: int = 2, memory_downsample: int = 0) -> str:
        """The last step as seqpipe.simreport.v1 with measured ns times (needs FLAG_TIMELINE)."""
        n = C.c_size_t(0)
        _check(_capi.lib().sp_engine_report_json(self._h, indent, memory_downsample, None, C.byref(n)))
        b = C.create_string_buffer(n.value)
        _check(_capi.lib().sp_engine_report_json(self._h, indent, memory_downsample, b, C.byref(n)))
        return b.value.decode()

    def render_gantt(self, fmt: str = "ascii", width: int = 120) -> str:
        """The last MEASURED step (ns times) drawn by the reference renderers' rules (needs FLAG_TIMELINE)."""
        n = C.c_size_t(0)
        f = pl.RENDER_FORMATS[fmt]
        _check(_capi.lib().sp_engine_render_gantt(self._h, f, width, None, C.byref(n)))
        b = C.create_string_buffer(n.value)
        _check(_capi.lib().sp_engine_render_gantt(self._h, f, width, b, C.byref(n)))
        return b.value.decode()

    def op_log(self) -> pl.Schedule:
        P = self.cfg.pipeline_size
        counts = (C.c_int64 * P)()
        _check(_capi.lib().sp_engine_op_log(self._h, None, counts))
        ops = (_capi.Task * max(1, sum(counts)))()
        _check(_capi.lib().sp_engine_op_log(self._h, ops, counts))
        return pl.Schedule(self.cfg, self.kind, pl._unflatten(P, ops, counts))

    def timeline(self):
        n = C.c_int64(0)
        _check(_capi.lib().sp_engine_timeline(self._h, None, None, C.byref(n)))
        a = (C.c_double * max(1, n.value))()
        b = (C.c_double * max(1, n.value))()
        _check(_capi.lib().sp_engine_timeline(self._h, a, b, C.byref(n)))
        return np.array(a[: n.value]), np.array(b[: n.value])

    def params(self) -> dict:
        """name -> (rows, cols) of every parameter held by this engine."""
        n = C.c_int64()
        _check(_capi.lib().sp_engine_param_count(self._h, C.byref(n)))
        out = {}
        for i in range(n.value):
            name = C.create_string_buffer(128)
            numel, r, c = C.c_int64(), C.c_int32(), C.c_int32()
            _check(_capi.lib().sp_engine_param_info(self._h, i, name, 128, C.byref(numel), C.byref(r), C.byref(c)))
            out[name.value.decode()] = (r.value, c.value)
        return out

    def _rows(self, name, rows):
        return self.model.vocab if name == "lm_head" else rows

    def read_param(self, name: str) -> np.ndarray:
        r, c = self.params()[name]
        r = self._rows(name, r)
        out = np.empty((r, c), dtype=np.float32)
        _check(_capi.lib().sp_engine_read_param(self._h, name.encode(), out.ctypes.data_as(C.POINTER(C.c_float)),
                                                out.size))
        return out

    def read_grad(self, name: str) -> np.ndarray:
        r, c = self.params()[name]
        r = self._rows(name, r)
        out = np.empty((r, c), dtype=np.float32)
        _check(_capi.lib().sp_engine_read_grad(self._h, name.encode(), out.ctypes.data_as(C.POINTER(C.c_float)),
                                               out.size))
        return out

    def write_param(self, name: str, value: np.ndarray):
        v = np.ascontiguousarray(value, dtype=np.float32)
        _check(_capi.lib().sp_engine_write_param(self._h, name.encode(), v.ctypes.data_as(C.POINTER(C.c_float)),
                                                 v.size))


class LocalHub:
    """In-process P2P hub shared by the `world_size` engines of one process (sp_local_hub_*)."""

    def __init__(self, world_size: int, watchdog_seconds: float = 120.0):
        self._h = C.c_void_p()
        _check(_capi.lib().sp_local_hub_create(world_size, watchdog_seconds, C.byref(self._h)))

    def __del__(self):
        try:
            if self._h:
                _capi.lib().sp_local_hub_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def plan_memory(cfg: pl.ScenarioConfig, kind, partition: pl.SequencePartition, model: ModelConfig, stage: int = 1):
    """(live peak bytes, arena bytes, dKV accumulator bytes) of one stage, computed on the host."""
    c = cfg.to_c()
    lens = (C.c_int64 * len(partition.lengths))(*partition.lengths)
    mc = model.to_c()
    a, b, d = C.c_double(), C.c_double(), C.c_double()
    _check(_capi.lib().sp_plan_memory(C.byref(c), pl.kind_id(kind), lens, C.byref(mc), stage, C.byref(a), C.byref(b),
                                      C.byref(d)))
    return a.value, b.value, d.value


def comm_plan(cfg: pl.ScenarioConfig, kind, partition: pl.SequencePartition, device: int, hidden: int):
    """P2P transfers the multi-process engine issues on `device` (1-based), in issue order:
    list of dicts (op_index, when 'pre'/'post', dir 'send'/'recv', peer rank, channel, task, elems)."""
    c = cfg.to_c()
    lens = (C.c_int64 * len(partition.lengths))(*partition.lengths)
    n = C.c_int64(0)
    _check(_capi.lib().sp_comm_plan(C.byref(c), pl.kind_id(kind), lens, device, hidden, None, C.byref(n)))
    buf = (_capi.CommOp * max(1, n.value))()
    _check(_capi.lib().sp_comm_plan(C.byref(c), pl.kind_id(kind), lens, device, hidden, buf, C.byref(n)))
    out = []
    for o in buf[: n.value]:
        out.append({"op_index": o.op_index, "when": "pre" if o.when == 0 else "post",
                    "dir": "send" if o.dir == 0 else "recv", "peer": o.peer, "channel": o.channel,
                    "task": (pl.TASK_KINDS[o.kind], o.micro_batch, o.segment, o.stage), "elems": o.elems})
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_capi.lib().sp_nccl_unique_id(buf, 128))
    return buf.raw
