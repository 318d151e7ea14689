#!/usr/bin/env python
"""Our tcgen05 GEMM vs cuBLAS (torch.matmul) at the GPT-2.7B per-segment shapes, same operands,
CUDA-event timed after warm-up (bf16 out; reference point only, cuBLAS is not on the product path)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent))
from kernel_bench import gemm_case  # noqa: E402

n, h, F = 10170, 2560, 10240
for role, (M, N, K) in {"qkv_fwd": (n, 3 * h, h), "mlp_up_fwd": (n, F, h), "mlp_down_fwd": (n, h, F),
                        "o_fwd": (n, h, h)}.items():
    ms, tf = gemm_case(M, N, K, 1, 1, 0, 0)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        c = a @ b.t()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        c = a @ b.t()
    e1.record()
    torch.cuda.synchronize()
    cms = e0.elapsed_time(e1) / 10
    print(f"{role:14s} M{M} N{N} K{K}: ours {ms:.3f} ms {tf:.0f} TF | cuBLAS {cms:.3f} ms {2 * M * N * K / cms / 1e9:.0f} TF")
