#!/usr/bin/env python
"""One forward + one backward of the tcgen05 prefix attention at the cfg-2 last-segment
shape (n 6674 over a 32768-key prefix, 32 heads x 80) — the ncu capture target.
Prints CUDA-event times of a second (warm) fwd and bwd."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2406_03488_b200 import _capi  # noqa: E402

args = sys.argv[1:]
if args[:1] == ["--variant"]:  # a tuning build from tools/build_variant.py
    _capi.LIB_PATH = _capi.LIB_PATH.parent / "variants" / f"libseqpipe_b200_{args[1]}.so"
    args = args[2:]
n, q_off, H, hd = (int(x) for x in (args[:4] if len(args) > 3 else (6674, 26094, 32, 80)))
h, L = H * hd, q_off + n
q = torch.randn(n, h, device="cuda").to(torch.bfloat16)
kv = torch.randn(L, 2 * h, device="cuda").to(torch.bfloat16)
o = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(H, n, device="cuda")
dout = torch.randn(n, h, device="cuda").to(torch.bfloat16)
dq = torch.empty_like(q)
dkv = torch.zeros(L, 2 * h, device="cuda")
lib = _capi.lib()
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
s = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for _ in range(2):
    ev[0].record()
    _capi.check(lib.sp_attention_fwd(1, 0, P(q), P(kv), P(o), P(lse), n, q_off, L, H, hd, C.c_void_p(s)))
    ev[1].record()
    _capi.check(lib.sp_attention_bwd(1, 0, P(q), P(kv), P(o), P(dout), P(lse), P(dq), P(dkv), n, q_off, L, H, hd,
                                     C.c_void_p(s)))
    ev[2].record()
torch.cuda.synchronize()
print(f"fwd {ev[0].elapsed_time(ev[1]):.3f} ms  bwd {ev[1].elapsed_time(ev[2]):.3f} ms")
