#!/usr/bin/env python
"""Forward (and backward) of a tuning build of the attention kernels against an fp64 torch
reference, before a variant is adopted: tools/attn_variant_check.py VARIANT.
Shapes: small / ragged ones (masking, partial tiles, odd tile counts) and the cfg-2 long
prefix (heads chunked). Prints max relative-L2 errors; exit 1 above the bf16 tolerance."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2406_03488_b200 import _capi  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "product":
    _capi.LIB_PATH = _capi.LIB_PATH.parent / "variants" / f"libseqpipe_b200_{sys.argv[1]}.so"
lib = _capi.lib()
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def rel(a, b):
    return float((a.double() - b).norm() / b.norm())


def ref(q, kv, dout, n, q_off, H, hd):
    h = H * hd
    L = q_off + n
    outs = []
    for h0 in range(0, H, 4):
        hs = slice(h0 * hd, min(H, h0 + 4) * hd)
        qq = q[:, hs].double().view(n, -1, hd).transpose(0, 1).requires_grad_()
        kk = kv[:, hs].double().view(L, -1, hd).transpose(0, 1).requires_grad_()
        vv = kv[:, h:][:, hs].double().view(L, -1, hd).transpose(0, 1).requires_grad_()
        s = qq @ kk.transpose(1, 2) / hd ** 0.5
        mask = torch.arange(L, device=q.device)[None, :] > (q_off + torch.arange(n, device=q.device))[:, None]
        s = s.masked_fill(mask, float("-inf"))
        lse = torch.logsumexp(s, -1)
        o = torch.softmax(s, -1) @ vv
        go = dout[:, hs].double().view(n, -1, hd).transpose(0, 1)
        dq, dk, dv = torch.autograd.grad(o, (qq, kk, vv), go)
        outs.append((o.transpose(0, 1).reshape(n, -1), lse, dq.transpose(0, 1).reshape(n, -1),
                     dk.transpose(0, 1).reshape(L, -1), dv.transpose(0, 1).reshape(L, -1)))
    return [torch.cat([x[i] for x in outs], dim=0 if i == 1 else 1) for i in range(5)]


worst = 0.0
for n, q_off, H, hd in [(77, 0, 2, 64), (130, 200, 4, 64), (96, 160, 3, 80), (700, 1111, 2, 80), (1000, 0, 2, 80),
                        (385, 0, 3, 80), (6674, 26094, 4, 80), (10170, 0, 2, 80)]:
    h, L = H * hd, q_off + n
    g = torch.Generator(device="cuda").manual_seed(n + q_off)
    q = torch.randn(n, h, device="cuda", generator=g).to(torch.bfloat16)
    kv = torch.randn(L, 2 * h, device="cuda", generator=g).to(torch.bfloat16)
    dout = torch.randn(n, h, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda")
    _capi.check(lib.sp_attention_fwd(1, 2, P(q), P(kv), P(o), P(lse), n, q_off, L, H, hd, None))
    dq = torch.empty_like(q)
    dkv = torch.zeros(L, 2 * h, device="cuda")
    _capi.check(lib.sp_attention_bwd(1, 2, P(q), P(kv), P(o), P(dout), P(lse), P(dq), P(dkv), n, q_off, L, H, hd,
                                     None))
    torch.cuda.synchronize()
    o_r, lse_r, dq_r, dk_r, dv_r = ref(q, kv, dout, n, q_off, H, hd)
    errs = {"o": rel(o.float(), o_r), "lse": rel(lse, lse_r), "dq": rel(dq.float(), dq_r),
            "dk": rel(dkv[:, :h], dk_r), "dv": rel(dkv[:, h:], dv_r)}
    worst = max(worst, errs["o"], errs["dq"], errs["dk"], errs["dv"])
    print(f"n {n} q_off {q_off} H {H} hd {hd}: " + " ".join(f"{k} {v:.2e}" for k, v in errs.items()), flush=True)
print(f"worst {worst:.2e}")
sys.exit(0 if worst < 2e-2 else 1)
