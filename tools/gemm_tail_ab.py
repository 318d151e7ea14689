#!/usr/bin/env python
"""tcgen05 GEMM at the cfg-2 shapes whose 256x256 tile count leaves a partial last wave on
74 CTA pairs, in the roles the engine runs them (fwd: A, B K-major, bf16 out; dgrad: B
MN-major; wgrad: A, B MN-major, fp32 +=). CUDA events, L2 flushed before each call, median
of 15 (SP_GEMM_REPS). SP_GEMM_ONLY=name runs one case (ncu captures). tools/gemm_tail_ab.py [tag]"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2406_03488_b200 import _capi  # noqa: E402

args = sys.argv[1:]
if args[:1] == ["--variant"]:  # a tuning build from tools/build_variant.py
    _capi.LIB_PATH = _capi.LIB_PATH.parent / "variants" / f"libseqpipe_b200_{args[1]}.so"
    args = args[2:] or [args[1]]
tag = args[0] if args else "default"
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
n, h, F = 10170, 2560, 10240
# name, M, N, K, a_kmajor, b_kmajor, c_f32, accumulate
CASES = [("o_fwd", n, h, h, 1, 1, 0, 0), ("mlp_down_fwd", n, h, F, 1, 1, 0, 0),
         ("qkv_dgrad", n, h, 3 * h, 1, 0, 0, 0), ("mlp_up_dgrad", n, h, F, 1, 0, 0, 0),
         ("o_wgrad", h, h, n, 0, 0, 1, 1), ("qkv_wgrad", 3 * h, h, n, 0, 0, 1, 1),
         ("mlp_down_wgrad", h, F, n, 0, 0, 1, 1), ("mlp_up_wgrad", F, h, n, 0, 0, 1, 1)]
ONLY = os.environ.get("SP_GEMM_ONLY")
REPS = int(os.environ.get("SP_GEMM_REPS", "15"))
for name, M, N, K, ak, bk, cf, acc in CASES:
    if ONLY and name != ONLY:
        continue
    A = torch.randn((M, K) if ak else (K, M), device="cuda").to(torch.bfloat16)
    B = torch.randn((N, K) if bk else (K, N), device="cuda").to(torch.bfloat16)
    Cm = torch.zeros(M, N, device="cuda", dtype=torch.float32 if cf else torch.bfloat16)

    def fn():
        _capi.check(_capi.lib().sp_gemm(1, 2, P(A), ak, P(B), bk, P(Cm), cf, acc, M, N, K, s))
    for _ in range(3):
        fn()
    ts = []
    for _ in range(REPS):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    tiles = ((M + 255) // 256) * ((N + 255) // 256)
    print(json.dumps({"tag": tag, "gemm": name, "M": M, "N": N, "K": K, "tiles": tiles, "waves": round(tiles / 74, 2),
                      "ms": round(ms, 4), "tflops": round(2 * M * N * K / ms / 1e9, 1)}), flush=True)
