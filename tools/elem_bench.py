#!/usr/bin/env python
"""HBM roofline of the bf16 elementwise kernels at the bench shapes, through the C-ABI:
norm fwd / bwd (+ residual gradient) and the MLP activation fwd / bwd. CUDA events around
single launches, median of 15, L2 flushed before each by READING a 256 MB buffer (a write
flush leaves ~126 MB of dirty lines whose write-back lands inside the next kernel: the
round-2 numbers taken that way are ~30 % low for these ~100 MB kernels; SP_FLUSH=write
reproduces them). Algorithmic bytes = tensors read + written once; fraction against
MEASURED_PEAKS.json hbm_gbs. tools/elem_bench.py [n] [h] [F]"""
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2406_03488_b200 import _capi  # noqa: E402

n, h, F = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10170, 2560, 10240)))
try:
    HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
except Exception:  # noqa: BLE001
    HBM = 7700.0
lib = _capi.lib()
P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
import os  # noqa: E402
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB
FLUSH_WRITE = os.environ.get("SP_FLUSH", "read") == "write"


def timed(fn, reps=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if FLUSH_WRITE:
            flush.fill_(1.0)
        else:
            flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] * 1e-3


bf = dict(device="cuda", dtype=torch.bfloat16)
x = torch.randn(n, h, **bf)
dy = torch.randn(n, h, **bf)
dres = torch.randn(n, h, **bf)
y = torch.empty(n, h, **bf)
dx = torch.empty(n, h, **bf)
g = torch.rand(h, device="cuda") + 0.5
mean = torch.empty(n, device="cuda")
rstd = torch.empty(n, device="cuda")
dg = torch.zeros(h, device="cuda")
u = torch.randn(n, F, **bf)
a_out = torch.empty(n, F, **bf)
du = torch.empty(n, F, **bf)
E = n * h * 2
cases = [
    ("norm_fwd (LayerNorm)", lambda: _capi.check(lib.sp_norm_fwd(1, 0, P(x), P(g), P(y), P(mean), P(rstd), n, h,
                                                                  C.c_float(1e-5), s)), 2 * E + 8 * n),
    ("norm_fwd (RMSNorm)", lambda: _capi.check(lib.sp_norm_fwd(1, 1, P(x), P(g), P(y), P(mean), P(rstd), n, h,
                                                                C.c_float(1e-5), s)), 2 * E + 4 * n),
    ("norm_bwd (LayerNorm, + dres)", lambda: _capi.check(lib.sp_norm_bwd(1, 0, P(dy), P(x), P(g), P(mean), P(rstd),
                                                                          P(dres), P(dx), P(dg), n, h, s)),
     4 * E + 8 * n),
    ("norm_bwd (LayerNorm)", lambda: _capi.check(lib.sp_norm_bwd(1, 0, P(dy), P(x), P(g), P(mean), P(rstd), None,
                                                                  P(dx), P(dg), n, h, s)), 3 * E + 8 * n),
    ("act_fwd (GeLU)", lambda: _capi.check(lib.sp_act_fwd(1, 0, P(u), P(a_out), n, F, s)), 2 * n * F * 2),
    ("act_bwd (GeLU)", lambda: _capi.check(lib.sp_act_bwd(1, 0, P(u), P(a_out), P(du), n, F, s)), 3 * n * F * 2),
]
for name, fn, byts in cases:
    t = timed(fn)
    print(json.dumps({"kernel": name, "flush": "write" if FLUSH_WRITE else "read", "n": n, "h": h, "F": F,
                      "us": round(t * 1e6, 1),
                      "algorithmic_MB": round(byts / 1e6, 1), "GBps": round(byts / t / 1e9),
                      "frac_of_hbm": round(byts / t / 1e9 / HBM, 3)}), flush=True)
