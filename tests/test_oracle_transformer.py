"""Pins the CPU fp64 transformer oracle (oracle/transformer.py) — the parity
anchor of the execution half, which the reference cannot pin (it has no tensor
code): (1) against torch.autograd in float64 on identical weights/tokens, and
(2) split == unsplit: the Seq1F1B segment loop (KV prefix forward, reverse
dK/dV accumulation) equals the whole-sequence pass."""
import numpy as np
import pytest

from oracle.transformer import GPT, LLAMA, Model, rel_l2, tokens_for

torch = pytest.importorskip("torch")


def params(family, V, h, L, F, T, seed=0):
    rng = np.random.default_rng(seed)
    p = {"embed": rng.normal(0, .02, (V, h)), "final_norm": 1 + rng.normal(0, .1, (1, h)),
         "lm_head": rng.normal(0, .02, (V, h))}
    if family == GPT:
        p["pos"] = rng.normal(0, .02, (T, h))
    fup = 2 * F if family == LLAMA else F
    for l in range(L):
        p[f"layer{l}.norm1"] = 1 + rng.normal(0, .1, (1, h))
        p[f"layer{l}.norm2"] = 1 + rng.normal(0, .1, (1, h))
        p[f"layer{l}.wqkv"] = rng.normal(0, .2, (3 * h, h))
        p[f"layer{l}.wo"] = rng.normal(0, .2, (h, h))
        p[f"layer{l}.w1"] = rng.normal(0, .2, (fup, h))
        p[f"layer{l}.w2"] = rng.normal(0, .2, (h, F))
    return p


def autograd_step(family, p, tok, h, H, F, L):
    T = tok.shape[1] - 1
    tp = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
    hd = h // H
    pos = torch.arange(T, dtype=torch.float64)

    def norm(x, g):
        if family == LLAMA:
            return x * torch.rsqrt((x * x).mean(1, keepdim=True) + 1e-5) * g
        xc = x - x.mean(1, keepdim=True)
        return xc * torch.rsqrt((xc * xc).mean(1, keepdim=True) + 1e-5) * g

    def rope(x):
        j = torch.arange(hd // 2, dtype=torch.float64)
        ang = pos[:, None] * (10000.0 ** (-2 * j / hd))[None]
        c, s = torch.cos(ang), torch.sin(ang)
        xr = x.view(T, H, hd)
        a, b = xr[..., :hd // 2], xr[..., hd // 2:]
        return torch.cat([a * c[:, None] - b * s[:, None], a * s[:, None] + b * c[:, None]], -1).reshape(T, h)

    total = 0
    for mb in range(tok.shape[0]):
        t = torch.tensor(tok[mb].astype(np.int64))
        x = tp["embed"][t[:T]] + (tp["pos"][:T] if family == GPT else 0)
        for l in range(L):
            a = norm(x, tp[f"layer{l}.norm1"][0])
            qkv = a @ tp[f"layer{l}.wqkv"].T
            q, k, v = qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:]
            if family == LLAMA:
                q, k = rope(q), rope(k)
            qh, kh, vh = (z.view(T, H, hd).transpose(0, 1) for z in (q, k, v))
            S = (qh @ kh.transpose(1, 2) / np.sqrt(hd)).masked_fill(
                torch.triu(torch.ones(T, T, dtype=torch.bool), 1), float("-inf"))
            o = (torch.softmax(S, -1) @ vh).transpose(0, 1).reshape(T, h)
            xm = x + o @ tp[f"layer{l}.wo"].T
            u = norm(xm, tp[f"layer{l}.norm2"][0]) @ tp[f"layer{l}.w1"].T
            g = torch.nn.functional.gelu(u, approximate="tanh") if family == GPT else \
                torch.nn.functional.silu(u[:, :F]) * u[:, F:]
            x = xm + g @ tp[f"layer{l}.w2"].T
        logits = norm(x, tp["final_norm"][0]) @ tp["lm_head"].T
        total = total + torch.nn.functional.cross_entropy(logits, t[1:], reduction="sum")
    loss = total / (tok.shape[0] * T)
    loss.backward()
    return float(loss.detach()), {k: v.grad.numpy() for k, v in tp.items()}


@pytest.mark.parametrize("family", [GPT, LLAMA])
def test_oracle_matches_autograd_fp64(family):
    h, H, L, F, V, T = 64, 2, 2, 128, 97, 64
    p = params(family, V, h, L, F, T)
    tok = tokens_for(2, T, V)
    m = Model(family, V, h, L, H, h // H, F)
    loss, grads = m.step(p, tok, [T])
    l2, g2 = autograd_step(family, p, tok, h, H, F, L)
    assert abs(loss - l2) < 1e-12
    for k in grads:
        assert rel_l2(grads[k], g2[k]) < 1e-11, k


@pytest.mark.parametrize("family", [GPT, LLAMA])
@pytest.mark.parametrize("lengths", [[30, 20, 9, 5], [1, 1, 62], [64], [16, 16, 16, 16]])
def test_split_equals_unsplit(family, lengths):
    h, H, L, F, V, T = 64, 2, 2, 128, 97, 64
    p = params(family, V, h, L, F, T, seed=3)
    tok = tokens_for(2, T, V, seed=7)
    m = Model(family, V, h, L, H, h // H, F)
    l1, g1 = m.step(p, tok, [T])
    lk, gk = m.step(p, tok, lengths)
    assert abs(l1 - lk) < 1e-12
    assert max(rel_l2(gk[k], g1[k]) for k in g1) < 1e-12


@pytest.mark.parametrize("family", [GPT, LLAMA])
def test_torch_backend_and_head_chunking_match_numpy(family):
    """The oracle's torch-fp64 backend (used on the GPU box for the 32K-token parity
    checks) and its head-chunked attention give the numpy oracle's numbers."""
    from oracle.transformer import TorchOps
    h, H, L, F, V, T = 64, 4, 2, 128, 97, 64
    p = params(family, V, h, L, F, T, seed=5)
    tok = tokens_for(2, T, V, seed=9)
    l0, g0 = Model(family, V, h, L, H, h // H, F).step(p, tok, [30, 20, 14])
    l1, g1 = Model(family, V, h, L, H, h // H, F, ops=TorchOps("cpu"), head_chunk=1).step(p, tok, [30, 20, 14])
    assert abs(l0 - l1) < 1e-12
    assert max(rel_l2(g1[k], g0[k]) for k in g0) < 1e-12
