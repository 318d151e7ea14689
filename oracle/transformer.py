"""TEST INFRASTRUCTURE ONLY — CPU fp64 oracle for the execution half.

Parity status: the reference (/root/reference) has no tensor code
(SPEC.md:117, :434), so the loss/gradient numerics are NOT pinned by the
reference. This oracle restates PAPER.md:140-157 (Eq. 2 language-model
factorisation, Eq. 3 causal attention) for the two model families the engine
runs, and is itself pinned two ways (tests/test_oracle_transformer.py):
  * against torch.autograd in float64 on the same weights and tokens, and
  * split == unsplit: running the Seq1F1B segment loop (per-segment forward
    over the KV prefix, reverse-order backward accumulating dK/dV into earlier
    segments' rows — the dependency edges of sim.cpp:24-27 and :34-36) gives
    the same loss and gradients as the whole-sequence pass.

Model definitions (must match csrc/engine/stage.cpp):
  GPT   : x = E[tok] + Pos[t]; pre-LayerNorm (gain only); QKV/O/W1/W2 without
          bias; GeLU(tanh); final LayerNorm; untied LM head.
  LLaMA : x = E[tok]; RMSNorm; RoPE (rotate-half, global positions); SwiGLU with
          W1 = [gate; up] rows; final RMSNorm; untied LM head.
Loss = mean token cross-entropy over all M*T tokens of the step.
"""
from __future__ import annotations

import math

import numpy as np

GPT, LLAMA = 0, 1


class NumpyOps:
    """Array backend of the oracle: numpy float64 on the host (the default)."""

    def __init__(self):
        self.f = np.float64

    def asarray(self, x):
        return np.asarray(x, dtype=np.float64)

    def host(self, x):
        return np.asarray(x, dtype=np.float64)

    def ints(self, x):
        return np.asarray(x, dtype=np.int64)

    def zeros(self, shape):
        return np.zeros(shape)

    def zeros_like(self, x):
        return np.zeros_like(x)

    def arange(self, a, b=None):
        return np.arange(a) if b is None else np.arange(a, b)

    def cat(self, xs, axis):
        return np.concatenate(xs, axis=axis)

    def where(self, c, a, b):
        return np.where(c, a, b)

    def mean(self, x, axis):
        return x.mean(axis=axis, keepdims=True)

    def sum(self, x, axis, keepdims=True):
        return x.sum(axis=axis, keepdims=keepdims)

    def amax(self, x, axis):
        return x.max(axis=axis, keepdims=True)

    def heads(self, x, n, H, hd):  # [n, H*hd] -> [H, n, hd]
        return x.reshape(n, H, hd).transpose(1, 0, 2)

    def unheads(self, x, n):  # [H, n, hd] -> [n, H*hd]
        return x.transpose(1, 0, 2).reshape(n, -1)

    def swap(self, x):  # transpose of the last two axes
        return np.swapaxes(x, -1, -2)

    def index_add(self, dst, idx, src):
        np.add.at(dst, idx, src)

    exp, log, tanh, sqrt = staticmethod(np.exp), staticmethod(np.log), staticmethod(np.tanh), staticmethod(np.sqrt)


class TorchOps(NumpyOps):
    """The same oracle on torch float64 tensors (e.g. on a GPU, to check the engine at the
    benchmarked 32K-token shapes in seconds). Arithmetic is identical: fp64 throughout."""

    def __init__(self, device="cpu"):
        import torch
        self.t, self.device, self.f = torch, device, torch.float64

    def asarray(self, x):
        return self.t.as_tensor(np.asarray(x, dtype=np.float64), device=self.device)

    def host(self, x):
        return x.detach().cpu().numpy()

    def ints(self, x):
        return self.t.as_tensor(np.asarray(x, dtype=np.int64), device=self.device)

    def zeros(self, shape):
        return self.t.zeros(shape, dtype=self.f, device=self.device)

    def zeros_like(self, x):
        return self.t.zeros_like(x)

    def arange(self, a, b=None):
        return self.t.arange(a, device=self.device) if b is None else self.t.arange(a, b, device=self.device)

    def cat(self, xs, axis):
        return self.t.cat(xs, dim=axis)

    def where(self, c, a, b):
        return self.t.where(c, a, self.t.as_tensor(b, dtype=self.f, device=self.device))

    def mean(self, x, axis):
        return x.mean(dim=axis, keepdim=True)

    def sum(self, x, axis, keepdims=True):
        return x.sum(dim=axis, keepdim=keepdims)

    def amax(self, x, axis):
        return x.amax(dim=axis, keepdim=True)

    def heads(self, x, n, H, hd):
        return x.reshape(n, H, hd).permute(1, 0, 2)

    def unheads(self, x, n):
        return x.permute(1, 0, 2).reshape(n, -1)

    def swap(self, x):
        return x.transpose(-1, -2)

    def index_add(self, dst, idx, src):
        dst.index_add_(0, idx, src)

    def exp(self, x):
        return self.t.exp(x)

    def log(self, x):
        return self.t.log(x)

    def tanh(self, x):
        return self.t.tanh(x)

    def sqrt(self, x):
        return self.t.sqrt(x)


def _gelu(o, u):
    c = math.sqrt(2.0 / math.pi)
    return 0.5 * u * (1.0 + o.tanh(c * (u + 0.044715 * u ** 3)))


def _gelu_grad(o, u):
    c = math.sqrt(2.0 / math.pi)
    t = o.tanh(c * (u + 0.044715 * u ** 3))
    return 0.5 * (1 + t) + 0.5 * u * (1 - t * t) * c * (1 + 3 * 0.044715 * u * u)


def _sigmoid(o, x):
    return 1.0 / (1.0 + o.exp(-x))


def _norm_fwd(o, x, g, rms, eps):
    xc = x if rms else x - o.mean(x, 1)
    rstd = 1.0 / o.sqrt(o.mean(xc * xc, 1) + eps)
    xh = xc * rstd
    return xh * g, (xh, rstd)


def _norm_bwd(o, dy, g, cache, rms):
    xh, rstd = cache
    dxh = dy * g
    m2 = o.mean(dxh * xh, 1)
    if rms:
        dx = rstd * (dxh - xh * m2)
    else:
        dx = rstd * (dxh - o.mean(dxh, 1) - xh * m2)
    return dx, o.sum(dy * xh, 0, keepdims=False)


def _rope(o, x, H, hd, pos, theta, inverse=False):
    """x [n, H*hd] -> rotated copy (pairs j, j + hd/2 inside each head), global positions."""
    n = x.shape[0]
    j = np.arange(hd // 2)
    inv = theta ** (-2.0 * j / hd)
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv[None, :]
    c, s = o.asarray(np.cos(ang)), o.asarray(np.sin(ang))
    if inverse:
        s = -s
    xr = x.reshape(n, H, hd)
    a, b = xr[:, :, : hd // 2], xr[:, :, hd // 2:]
    out = o.cat([a * c[:, None, :] - b * s[:, None, :], a * s[:, None, :] + b * c[:, None, :]], 2)
    return out.reshape(n, H * hd)


class Model:
    """ops: NumpyOps() (default, host fp64) or TorchOps(device) (same arithmetic on torch
    fp64 tensors). head_chunk bounds the [heads, n, kv] score tiles the attention materialises
    (the probabilities are recomputed from the saved log-sum-exp in the backward, so memory
    stays O(chunk * n * kv) at the benchmarked 32K-token shapes)."""

    def __init__(self, family, vocab, hidden, layers, heads, head_dim, ffn, eps=1e-5, theta=10000.0, ops=None,
                 head_chunk=None):
        self.family, self.V, self.h, self.L, self.H, self.hd, self.F = family, vocab, hidden, layers, heads, head_dim, ffn
        self.eps, self.theta = eps, theta
        self.rms = family == LLAMA
        self.o = ops or NumpyOps()
        self.head_chunk = head_chunk or heads

    # ------------------------------------------------------------------ attention over a prefix
    def _scores(self, qh, kh, q_off):
        """Causal scaled scores of head chunk qh [c,n,hd] x kh [c,kv,hd] -> [c,n,kv]."""
        o = self.o
        n, kv = qh.shape[1], kh.shape[1]
        S = (qh @ o.swap(kh)) / math.sqrt(self.hd)
        mask = o.arange(kv)[None, :] > (q_off + o.arange(n))[:, None]
        return o.where(~mask[None], S, -np.inf)

    def _attn_fwd(self, q, k, v, q_off):
        """q [n, h] at positions q_off..; k, v [q_off+n, h]. Returns o [n,h] and the row
        log-sum-exp [H, n, 1] of the scaled causal scores (PAPER Eq. 3)."""
        o = self.o
        n, H, hd = q.shape[0], self.H, self.hd
        kv = k.shape[0]
        qh, kh, vh = o.heads(q, n, H, hd), o.heads(k, kv, H, hd), o.heads(v, kv, H, hd)
        outs, lses = [], []
        for c0 in range(0, H, self.head_chunk):
            c1 = min(H, c0 + self.head_chunk)
            S = self._scores(qh[c0:c1], kh[c0:c1], q_off)
            mx = o.amax(S, 2)
            P = o.exp(S - mx)
            z = o.sum(P, 2)
            outs.append((P @ vh[c0:c1]) / z)
            lses.append(mx + o.log(z))
        return o.unheads(o.cat(outs, 0), n), o.cat(lses, 0)

    def _attn_bwd(self, do, q, k, v, out, lse):
        """dq [n,h], dk, dv [kv,h] of the prefix attention, with P recomputed from lse."""
        o = self.o
        n, H, hd = q.shape[0], self.H, self.hd
        kv = k.shape[0]
        q_off = kv - n
        qh, kh, vh = o.heads(q, n, H, hd), o.heads(k, kv, H, hd), o.heads(v, kv, H, hd)
        doh, oh = o.heads(do, n, H, hd), o.heads(out, n, H, hd)
        dq, dk, dv = [], [], []
        for c0 in range(0, H, self.head_chunk):
            c1 = min(H, c0 + self.head_chunk)
            P = o.exp(self._scores(qh[c0:c1], kh[c0:c1], q_off) - lse[c0:c1])
            dP = doh[c0:c1] @ o.swap(vh[c0:c1])
            dv.append(o.swap(P) @ doh[c0:c1])
            delta = o.sum(doh[c0:c1] * oh[c0:c1], 2)  # rowsum(dP * P) == rowsum(dO * O)
            dS = P * (dP - delta) / math.sqrt(hd)
            dq.append(dS @ kh[c0:c1])
            dk.append(o.swap(dS) @ qh[c0:c1])
        return o.unheads(o.cat(dq, 0), n), o.unheads(o.cat(dk, 0), kv), o.unheads(o.cat(dv, 0), kv)

    # ------------------------------------------------------------------ one micro-batch, segmented
    def micro_batch(self, p, tok, lengths, grads, scale):
        """Forward + backward of one micro-batch split into `lengths` segments
        (Seq1F1B order: F(s=1..k) then B(s=k..1)). tok: [T+1] int. Accumulates
        into `grads`; returns the summed token loss."""
        o = self.o
        h, L, F = self.h, self.L, self.F
        T = int(sum(lengths))
        prefix = np.concatenate([[0], np.cumsum(lengths)]).astype(int)
        tok_d = o.ints(tok)
        K = [o.zeros((T, h)) for _ in range(L)]
        Vv = [o.zeros((T, h)) for _ in range(L)]
        caches, loss = [], 0.0
        for s in range(len(lengths)):
            p0, n = int(prefix[s]), int(lengths[s])
            pos = np.arange(p0, p0 + n)
            t_in = tok_d[p0:p0 + n]
            x = p["embed"][t_in]
            if self.family == GPT:
                x = x + p["pos"][p0:p0 + n]
            cache = {"layers": []}
            for l in range(L):
                pre = f"layer{l}."
                a, c1 = _norm_fwd(o, x, p[pre + "norm1"][0], self.rms, self.eps)
                qkv = a @ p[pre + "wqkv"].T
                q, k, v = qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:]
                if self.family == LLAMA:
                    q = _rope(o, q, self.H, self.hd, pos, self.theta)
                    k = _rope(o, k, self.H, self.hd, pos, self.theta)
                K[l][p0:p0 + n], Vv[l][p0:p0 + n] = k, v
                at, lse = self._attn_fwd(q, K[l][:p0 + n], Vv[l][:p0 + n], p0)
                xm = x + at @ p[pre + "wo"].T
                b, c2 = _norm_fwd(o, xm, p[pre + "norm2"][0], self.rms, self.eps)
                u = b @ p[pre + "w1"].T
                if self.family == GPT:
                    g = _gelu(o, u)
                else:
                    g = u[:, :F] * _sigmoid(o, u[:, :F]) * u[:, F:]
                y = xm + g @ p[pre + "w2"].T
                cache["layers"].append(dict(a=a, c1=c1, q=q, o=at, lse=lse, b=b, c2=c2, u=u, g=g))
                x = y
            xf, cf = _norm_fwd(o, x, p["final_norm"][0], self.rms, self.eps)
            logits = xf @ p["lm_head"].T
            mx = o.amax(logits, 1)
            e = o.exp(logits - mx)
            z = o.sum(e, 1)
            lab = tok_d[p0 + 1:p0 + n + 1]
            rows = o.arange(n)
            loss += float((o.log(z[:, 0]) + mx[:, 0] - logits[rows, lab]).sum())
            dlog = e / z
            dlog[rows, lab] -= 1.0
            dlog = dlog * scale
            grads["lm_head"] += dlog.T @ xf
            dxf = dlog @ p["lm_head"]
            dx, dgf = _norm_bwd(o, dxf, p["final_norm"][0], cf, self.rms)
            grads["final_norm"][0] += dgf
            cache["dy"] = dx
            caches.append(cache)
        dK = [o.zeros((T, h)) for _ in range(L)]
        dV = [o.zeros((T, h)) for _ in range(L)]
        for s in reversed(range(len(lengths))):
            p0, n = int(prefix[s]), int(lengths[s])
            pos = np.arange(p0, p0 + n)
            dy = caches[s]["dy"]
            for l in reversed(range(L)):
                pre = f"layer{l}."
                c = caches[s]["layers"][l]
                grads[pre + "w2"] += dy.T @ c["g"]
                dg = dy @ p[pre + "w2"]
                if self.family == GPT:
                    du = dg * _gelu_grad(o, c["u"])
                else:
                    a_, b_ = c["u"][:, :F], c["u"][:, F:]
                    sg = _sigmoid(o, a_)
                    du = o.cat([dg * b_ * sg * (1 + a_ * (1 - sg)), dg * a_ * sg], 1)
                grads[pre + "w1"] += du.T @ c["b"]
                db = du @ p[pre + "w1"]
                dxm, dg2 = _norm_bwd(o, db, p[pre + "norm2"][0], c["c2"], self.rms)
                dxm = dxm + dy
                grads[pre + "norm2"][0] += dg2
                grads[pre + "wo"] += dxm.T @ c["o"]
                do = dxm @ p[pre + "wo"]
                dq, dk, dv = self._attn_bwd(do, c["q"], K[l][:p0 + n], Vv[l][:p0 + n], c["o"], c["lse"])
                dK[l][:p0 + n] += dk
                dV[l][:p0 + n] += dv
                dks, dvs = dK[l][p0:p0 + n], dV[l][p0:p0 + n]  # complete: later segments already added
                if self.family == LLAMA:
                    dq = _rope(o, dq, self.H, self.hd, pos, self.theta, inverse=True)
                    dks = _rope(o, dks, self.H, self.hd, pos, self.theta, inverse=True)
                dqkv = o.cat([dq, dks, dvs], 1)
                grads[pre + "wqkv"] += dqkv.T @ c["a"]
                da = dqkv @ p[pre + "wqkv"]
                dx, dg1 = _norm_bwd(o, da, p[pre + "norm1"][0], c["c1"], self.rms)
                grads[pre + "norm1"][0] += dg1
                dy = dx + dxm
            caches[s] = None  # release the segment's activations
            o.index_add(grads["embed"], tok_d[p0:p0 + n], dy)
            if self.family == GPT:
                grads["pos"][p0:p0 + n] += dy
        return loss

    def step(self, params, tokens, lengths):
        """Whole step: every micro-batch (tokens [M, T+1]) with the given segment
        lengths. Returns (mean loss, grads dict of host float64 arrays)."""
        o = self.o
        p = {k: o.asarray(v) for k, v in params.items()}
        grads = {k: o.zeros_like(v) for k, v in p.items()}
        M, T1 = tokens.shape
        T = T1 - 1
        scale = 1.0 / (M * T)
        total = 0.0
        for m in range(M):
            total += self.micro_batch(p, tokens[m], list(lengths), grads, scale)
        return total * scale, {k: o.host(v) for k, v in grads.items()}


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def tokens_for(M, T, vocab, seed=1234):
    """Synthetic tokens, uniform in [0, V): counter-based (PCG64 with a fixed seed)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, vocab, size=(M, T + 1), dtype=np.int64).astype(np.int32)
