#!/usr/bin/env python
"""SM clock / power / throttle reasons while the attention kernels run back to back:
attn_clock.py [fwd|bwd] [n q_off H hd]. Prints ms per call, algorithmic TFLOP/s
(fwd 4*H*hd*(n*q_off + n^2/2), bwd twice that) and the median SM clock."""
import ctypes as C
import sys
import threading
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import pynvml  # noqa: E402
import torch  # noqa: E402
from paper_2406_03488_b200 import _capi  # noqa: E402

args = sys.argv[1:]
variant = None
if args[:1] == ["--variant"]:  # a tuning build from tools/build_variant.py
    variant = args[1]
    _capi.LIB_PATH = _capi.LIB_PATH.parent / "variants" / f"libseqpipe_b200_{variant}.so"
    args = args[2:]
which = args[0] if args else "bwd"
n, q_off, H, hd = (int(x) for x in (args[1:5] if len(args) > 4 else (6674, 26094, 32, 80)))
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


def fwd():
    _capi.check(lib.sp_attention_fwd(1, 0, P(q), P(kv), P(o), P(lse), n, q_off, L, H, hd, C.c_void_p(s)))


BWD_IMPL = 0


def bwd():
    _capi.check(lib.sp_attention_bwd(1, BWD_IMPL, P(q), P(kv), P(o), P(dout), P(lse), P(dq), P(dkv), n, q_off, L, H, hd,
                                     C.c_void_p(s)))


fwd()
bwd()
torch.cuda.synchronize()
pynvml.nvmlInit()
dev = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def sample():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(dev, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(dev) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(dev)))
        time.sleep(0.02)


f = fwd if which == "fwd" else bwd
reps = 300 if which == "fwd" else 100
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
th = threading.Thread(target=sample)
th.start()
e0.record()
for _ in range(reps):
    f()
e1.record()
torch.cuda.synchronize()
stop.set()
th.join()
clk = sorted(x[0] for x in samples)
pw = sorted(x[1] for x in samples)
reasons = 0
for x in samples:
    reasons |= x[2]
ms = e0.elapsed_time(e1) / reps
fl = 4 * H * hd * (n * q_off + n * n / 2) * (1 if which == "fwd" else 2)
print(f"{variant or 'product'} {which}: {ms:.3f} ms/call  {fl / ms / 1e9:.0f} TF algorithmic  sm_mhz median {clk[len(clk) // 2]} "
      f"(min {clk[0]} max {clk[-1]})  power median {pw[len(pw) // 2]:.0f} W  reasons 0x{reasons:x}")
