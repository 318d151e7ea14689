#!/usr/bin/env python
"""Time sp_norm_fwd / sp_norm_bwd (bf16, LayerNorm) at [n, h]: norm_once.py [n h]. The ncu capture target."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2406_03488_b200 import _capi  # noqa: E402

n, h = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (8192, 2560)))
x = torch.randn(n, h, device="cuda").to(torch.bfloat16)
dy = torch.randn(n, h, device="cuda").to(torch.bfloat16)
g = torch.ones(h, device="cuda")
y = torch.empty_like(x)
dx = torch.empty_like(x)
mean = torch.empty(n, device="cuda")
rstd = torch.empty(n, device="cuda")
dg = torch.zeros(h, device="cuda")
lib = _capi.lib()
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for _ in range(3):
    ev[0].record()
    _capi.check(lib.sp_norm_fwd(1, 0, P(x), P(g), P(y), P(mean), P(rstd), n, h, C.c_float(1e-5), s))
    ev[1].record()
    _capi.check(lib.sp_norm_bwd(1, 0, P(dy), P(x), P(g), P(mean), P(rstd), None, P(dx), P(dg), n, h, s))
    ev[2].record()
torch.cuda.synchronize()
mb = n * h * 2 / 1e6
print(f"norm fwd {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us ({2 * mb / ev[0].elapsed_time(ev[1]) / 1e3:.2f} TB/s)  "
      f"bwd {ev[1].elapsed_time(ev[2]) * 1e3:.1f} us ({3 * mb / ev[1].elapsed_time(ev[2]) / 1e3:.2f} TB/s)")
