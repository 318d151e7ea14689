"""B200-native Seq1F1B training engine.

Layers:
  include/seqpipe/*.hpp, include/seqpipe_b200.h   C++ API + C-ABI (the drop-in boundary)
  csrc/planner       host C++ planner (partition, op tables, simulate, validate)
  csrc/cuda          sm_100a kernels (tcgen05 GEMM, prefix flash attention, norms, CE, launcher)
  csrc/engine        per-stage executor: arena, KV-prefix cache, streams, NCCL P2P
  planner.py / engine.py   Python mirror of the reference API over the C-ABI (ctypes)
"""
from . import planner  # noqa: F401

__all__ = ["planner"]
