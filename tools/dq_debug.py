import ctypes as C, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2406_03488_b200 import _capi
def P(t): return C.c_void_p(t.data_ptr())
for (n, q_off, H, hd) in [(130, 200, 4, 64), (130, 200, 4, 80), (77, 0, 2, 64), (96, 160, 3, 80), (700, 1111, 2, 80), (64, 0, 1, 64), (33, 0, 1, 64), (130, 0, 1, 64)]:
    h = H * hd; L = q_off + n
    g = torch.Generator(device="cuda").manual_seed(n + q_off)
    q = torch.randn(n, h, device="cuda", generator=g).bfloat16()
    kv = torch.randn(L, 2 * h, device="cuda", generator=g).bfloat16()
    dout = torch.randn(n, h, device="cuda", generator=g).bfloat16()
    o = torch.empty(n, h, device="cuda", dtype=torch.bfloat16); lse = torch.empty(H, n, device="cuda")
    lib = _capi.lib()
    _capi.check(lib.sp_attention_fwd(1, 2, P(q), P(kv), P(o), P(lse), n, q_off, L, H, hd, None))
    res = []
    for impl in (2, 3):
        dq = torch.empty(n, h, device="cuda", dtype=torch.bfloat16); dkv = torch.zeros(L, 2 * h, device="cuda")
        _capi.check(lib.sp_attention_bwd(1, impl, P(q), P(kv), P(o), P(dout), P(lse), P(dq), P(dkv), n, q_off, L, H, hd, None))
        torch.cuda.synchronize(); res.append((dq.float(), dkv))
    d = (res[0][0] - res[1][0]).view(n, H, hd)
    rowerr = d.norm(dim=2) / res[1][0].view(n, H, hd).norm(dim=2).clamp_min(1e-9)
    bad = (rowerr > 0.02).nonzero()
    print((n, q_off, H, hd), "dq rel", float((res[0][0]-res[1][0]).norm()/res[1][0].norm()), "dkv rel", float((res[0][1]-res[1][1]).norm()/res[1][1].norm()),
          "bad (row,head):", bad[:12].tolist(), "nbad", len(bad))
