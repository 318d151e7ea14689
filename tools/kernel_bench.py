#!/usr/bin/env python
"""Kernel microbenchmarks on the B200 through the C-ABI (CUDA events, warm L2
flushed between reps by a 256 MB write). Prints one JSON line per case:
tcgen05 GEMM at the GPT-2.7B / 7B / 13B per-segment shapes in all three roles
(forward, dgrad, wgrad) and prefix attention fwd/bwd."""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2406_03488_b200 import _capi  # noqa: E402

BF16 = 1


def timed(fn, reps=10, warm=3):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def gemm_case(M, N, K, a_k, b_k, c_f32, acc, impl=2):
    A = torch.randn((M, K) if a_k else (K, M), device="cuda").to(torch.bfloat16)
    B = torch.randn((N, K) if b_k else (K, N), device="cuda").to(torch.bfloat16)
    Cm = torch.zeros(M, N, device="cuda", dtype=torch.float32 if c_f32 else torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream

    def fn():
        _capi.check(_capi.lib().sp_gemm(BF16, impl, C.c_void_p(A.data_ptr()), a_k, C.c_void_p(B.data_ptr()), b_k,
                                        C.c_void_p(Cm.data_ptr()), c_f32, acc, M, N, K, C.c_void_p(s)))
    ms = timed(fn)
    return ms, 2.0 * M * N * K / (ms / 1e3) / 1e12


def attn_case(n, q_off, H, hd, bwd):
    h = H * hd
    L = q_off + n
    q = torch.randn(n, h, device="cuda").to(torch.bfloat16)
    kv = torch.randn(L, 2 * h, device="cuda").to(torch.bfloat16)
    o = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda")
    dout = torch.randn(n, h, device="cuda").to(torch.bfloat16)
    dq = torch.empty_like(q)
    dkv = torch.zeros(L, 2 * h, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    lib = _capi.lib()
    _capi.check(lib.sp_attention_fwd(BF16, 0, C.c_void_p(q.data_ptr()), C.c_void_p(kv.data_ptr()),
                                     C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()), n, q_off, L, H, hd,
                                     C.c_void_p(s)))

    def fwd():
        _capi.check(lib.sp_attention_fwd(BF16, 0, C.c_void_p(q.data_ptr()), C.c_void_p(kv.data_ptr()),
                                         C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()), n, q_off, L, H, hd,
                                         C.c_void_p(s)))

    def bwdf():
        _capi.check(lib.sp_attention_bwd(BF16, 0, C.c_void_p(q.data_ptr()), C.c_void_p(kv.data_ptr()),
                                         C.c_void_p(o.data_ptr()), C.c_void_p(dout.data_ptr()),
                                         C.c_void_p(lse.data_ptr()), C.c_void_p(dq.data_ptr()),
                                         C.c_void_p(dkv.data_ptr()), n, q_off, L, H, hd, C.c_void_p(s)))
    ms = timed(bwdf if bwd else fwd, reps=5, warm=2)
    fl = 4.0 * h * (n * q_off + 0.5 * n * n) * (2 if bwd else 1)
    return ms, fl / (ms / 1e3) / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--attn", action="store_true")
    ap.add_argument("--attn-only", action="store_true")
    args = ap.parse_args()
    args.attn |= args.attn_only
    shapes = [("2.7b", 10170, 2560, 10240), ("7b", 11428, 4096, 11008), ("13b", 14094, 5120, 20480)]
    if args.quick:
        shapes = shapes[:1]
    if args.attn_only:
        shapes = []
    for name, n, h, F in shapes:
        for role, (M, N, K, ak, bk, cf, acc) in {
            "qkv_fwd": (n, 3 * h, h, 1, 1, 0, 0),
            "mlp_up_fwd": (n, F, h, 1, 1, 0, 0),
            "mlp_down_fwd": (n, h, F, 1, 1, 0, 0),
            "mlp_up_dgrad": (n, h, F, 1, 0, 0, 0),
            "mlp_up_wgrad": (F, h, n, 0, 0, 1, 1),
            "qkv_wgrad": (3 * h, h, n, 0, 0, 1, 1),
            "o_wgrad": (h, h, n, 0, 0, 1, 1),
            "mlp_down_wgrad": (h, F, n, 0, 0, 1, 1),
        }.items():
            ms, tf = gemm_case(M, N, K, ak, bk, cf, acc)
            print(json.dumps({"kernel": "gemm_tcgen05", "model": name, "role": role, "M": M, "N": N, "K": K,
                              "ms": ms, "tflops": tf}), flush=True)
    if args.attn:
        for n, q_off, H, hd in [(10170, 0, 32, 80), (6674, 26094, 32, 80), (8192, 8192, 32, 128)]:
            for bwd in (False, True):
                ms, tf = attn_case(n, q_off, H, hd, bwd)
                print(json.dumps({"kernel": "attention_" + ("bwd" if bwd else "fwd"), "n": n, "q_off": q_off, "H": H,
                                  "hd": hd, "ms": ms, "tflops": tf}), flush=True)


if __name__ == "__main__":
    main()
