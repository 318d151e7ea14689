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

import numpy as np

GPT, LLAMA = 0, 1


def _gelu(u):
    c = np.sqrt(2.0 / np.pi)
    return 0.5 * u * (1.0 + np.tanh(c * (u + 0.044715 * u ** 3)))


def _gelu_grad(u):
    c = np.sqrt(2.0 / np.pi)
    t = np.tanh(c * (u + 0.044715 * u ** 3))
    return 0.5 * (1 + t) + 0.5 * u * (1 - t * t) * c * (1 + 3 * 0.044715 * u * u)


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _norm_fwd(x, g, rms, eps):
    mu = np.zeros((x.shape[0], 1)) if rms else x.mean(axis=1, keepdims=True)
    xc = x - mu
    rstd = 1.0 / np.sqrt((xc * xc).mean(axis=1, keepdims=True) + eps)
    xh = xc * rstd
    return xh * g, (xh, rstd)


def _norm_bwd(dy, g, cache, rms):
    xh, rstd = cache
    dxh = dy * g
    m2 = (dxh * xh).mean(axis=1, keepdims=True)
    if rms:
        dx = rstd * (dxh - xh * m2)
    else:
        dx = rstd * (dxh - dxh.mean(axis=1, keepdims=True) - xh * m2)
    return dx, (dy * xh).sum(axis=0)


def _rope_tables(pos, hd, theta):
    j = np.arange(hd // 2)
    inv = theta ** (-2.0 * j / hd)
    ang = pos[:, None].astype(np.float64) * inv[None, :]
    return np.cos(ang), np.sin(ang)


def _rope(x, H, hd, pos, theta, inverse=False):
    """x [n, H*hd] -> rotated copy (pairs j, j + hd/2 inside each head)."""
    n = x.shape[0]
    c, s = _rope_tables(pos, hd, theta)
    if inverse:
        s = -s
    xr = x.reshape(n, H, hd)
    a, b = xr[:, :, : hd // 2], xr[:, :, hd // 2:]
    out = np.concatenate([a * c[:, None, :] - b * s[:, None, :], a * s[:, None, :] + b * c[:, None, :]], axis=2)
    return out.reshape(n, H * hd)


class Model:
    def __init__(self, family, vocab, hidden, layers, heads, head_dim, ffn, eps=1e-5, theta=10000.0):
        self.family, self.V, self.h, self.L, self.H, self.hd, self.F = family, vocab, hidden, layers, heads, head_dim, ffn
        self.eps, self.theta = eps, theta
        self.rms = family == LLAMA

    # ------------------------------------------------------------------ attention over a prefix
    def _attn_fwd(self, q, k, v, q_off):
        """q [n, h] at positions q_off..; k, v [q_off+n, h]. Returns o [n,h], P [H,n,kv]."""
        n, H, hd = q.shape[0], self.H, self.hd
        kv = k.shape[0]
        qh = q.reshape(n, H, hd).transpose(1, 0, 2)
        kh = k.reshape(kv, H, hd).transpose(1, 0, 2)
        vh = v.reshape(kv, H, hd).transpose(1, 0, 2)
        S = qh @ kh.transpose(0, 2, 1) / np.sqrt(hd)
        mask = np.arange(kv)[None, :] > (q_off + np.arange(n))[:, None]
        S = np.where(mask[None], -np.inf, S)
        S = S - S.max(axis=2, keepdims=True)
        P = np.exp(S)
        P /= P.sum(axis=2, keepdims=True)
        o = (P @ vh).transpose(1, 0, 2).reshape(n, H * hd)
        return o, P

    def _attn_bwd(self, do, q, k, v, P):
        n, H, hd = q.shape[0], self.H, self.hd
        kv = k.shape[0]
        qh = q.reshape(n, H, hd).transpose(1, 0, 2)
        kh = k.reshape(kv, H, hd).transpose(1, 0, 2)
        vh = v.reshape(kv, H, hd).transpose(1, 0, 2)
        doh = do.reshape(n, H, hd).transpose(1, 0, 2)
        dP = doh @ vh.transpose(0, 2, 1)
        dvh = P.transpose(0, 2, 1) @ doh
        dS = P * (dP - (dP * P).sum(axis=2, keepdims=True)) / np.sqrt(hd)
        dqh = dS @ kh
        dkh = dS.transpose(0, 2, 1) @ qh
        back = lambda a, rows: a.transpose(1, 0, 2).reshape(rows, H * hd)
        return back(dqh, n), back(dkh, kv), back(dvh, kv)

    # ------------------------------------------------------------------ one micro-batch, segmented
    def micro_batch(self, p, tok, lengths, grads, scale):
        """Forward + backward of one micro-batch split into `lengths` segments
        (Seq1F1B order: F(s=1..k) then B(s=k..1)). tok: [T+1] int. Accumulates
        into `grads`; returns the summed token loss."""
        h, L, F = self.h, self.L, self.F
        T = int(sum(lengths))
        prefix = np.concatenate([[0], np.cumsum(lengths)]).astype(int)
        K = [np.zeros((T, h)) for _ in range(L)]
        Vv = [np.zeros((T, h)) for _ in range(L)]
        caches, loss = [], 0.0
        for s in range(len(lengths)):
            p0, n = prefix[s], lengths[s]
            pos = np.arange(p0, p0 + n)
            t_in = tok[p0:p0 + n]
            x = p["embed"][t_in].astype(np.float64)
            if self.family == GPT:
                x = x + p["pos"][pos]
            cache = {"x0": None, "layers": []}
            for l in range(L):
                pre = f"layer{l}."
                a, c1 = _norm_fwd(x, p[pre + "norm1"][0], self.rms, self.eps)
                qkv = a @ p[pre + "wqkv"].T
                q, k, v = qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:]
                if self.family == LLAMA:
                    q = _rope(q, self.H, self.hd, pos, self.theta)
                    k = _rope(k, self.H, self.hd, pos, self.theta)
                K[l][p0:p0 + n], Vv[l][p0:p0 + n] = k, v
                o, P = self._attn_fwd(q, K[l][:p0 + n], Vv[l][:p0 + n], p0)
                xm = x + o @ p[pre + "wo"].T
                b, c2 = _norm_fwd(xm, p[pre + "norm2"][0], self.rms, self.eps)
                u = b @ p[pre + "w1"].T
                if self.family == GPT:
                    g = _gelu(u)
                else:
                    g = u[:, :F] * _sigmoid(u[:, :F]) * u[:, F:]
                y = xm + g @ p[pre + "w2"].T
                cache["layers"].append(dict(x=x, a=a, c1=c1, q=q, o=o, P=P, xm=xm, b=b, c2=c2, u=u, g=g))
                x = y
            xf, cf = _norm_fwd(x, p["final_norm"][0], self.rms, self.eps)
            logits = xf @ p["lm_head"].T
            mx = logits.max(axis=1, keepdims=True)
            e = np.exp(logits - mx)
            z = e.sum(axis=1, keepdims=True)
            lab = tok[p0 + 1:p0 + n + 1]
            loss += float((np.log(z[:, 0]) + mx[:, 0] - logits[np.arange(n), lab]).sum())
            dlog = e / z
            dlog[np.arange(n), lab] -= 1.0
            dlog *= scale
            grads["lm_head"] += dlog.T @ xf
            dxf = dlog @ p["lm_head"]
            dx, dgf = _norm_bwd(dxf, p["final_norm"][0], cf, self.rms)
            grads["final_norm"][0] += dgf
            cache["dy"] = dx
            caches.append(cache)
        dK = [np.zeros((T, h)) for _ in range(L)]
        dV = [np.zeros((T, h)) for _ in range(L)]
        for s in reversed(range(len(lengths))):
            p0, n = prefix[s], lengths[s]
            pos = np.arange(p0, p0 + n)
            dy = caches[s]["dy"]
            for l in reversed(range(L)):
                pre = f"layer{l}."
                c = caches[s]["layers"][l]
                grads[pre + "w2"] += dy.T @ c["g"]
                dg = dy @ p[pre + "w2"]
                if self.family == GPT:
                    du = dg * _gelu_grad(c["u"])
                else:
                    a_, b_ = c["u"][:, :F], c["u"][:, F:]
                    sg = _sigmoid(a_)
                    du = np.concatenate([dg * b_ * sg * (1 + a_ * (1 - sg)), dg * a_ * sg], axis=1)
                grads[pre + "w1"] += du.T @ c["b"]
                db = du @ p[pre + "w1"]
                dxm, dg2 = _norm_bwd(db, p[pre + "norm2"][0], c["c2"], self.rms)
                dxm = dxm + dy
                grads[pre + "norm2"][0] += dg2
                grads[pre + "wo"] += dxm.T @ c["o"]
                do = dxm @ p[pre + "wo"]
                dq, dk, dv = self._attn_bwd(do, c["q"], K[l][:p0 + n], Vv[l][:p0 + n], c["P"])
                dK[l][:p0 + n] += dk
                dV[l][:p0 + n] += dv
                dks, dvs = dK[l][p0:p0 + n], dV[l][p0:p0 + n]  # complete: later segments already added
                if self.family == LLAMA:
                    dq = _rope(dq, self.H, self.hd, pos, self.theta, inverse=True)
                    dks = _rope(dks, self.H, self.hd, pos, self.theta, inverse=True)
                dqkv = np.concatenate([dq, dks, dvs], axis=1)
                grads[pre + "wqkv"] += dqkv.T @ c["a"]
                da = dqkv @ p[pre + "wqkv"]
                dx, dg1 = _norm_bwd(da, p[pre + "norm1"][0], c["c1"], self.rms)
                grads[pre + "norm1"][0] += dg1
                dy = dx + dxm
            t_in = tok[p0:p0 + n]
            np.add.at(grads["embed"], t_in, dy)
            if self.family == GPT:
                grads["pos"][pos] += dy
        return loss

    def step(self, params, tokens, lengths):
        """Whole step: every micro-batch (tokens [M, T+1]) with the given segment
        lengths. Returns (mean loss, grads dict) in float64."""
        p = {k: np.asarray(v, dtype=np.float64) for k, v in params.items()}
        grads = {k: np.zeros_like(v) for k, v in p.items()}
        M, T1 = tokens.shape
        T = T1 - 1
        scale = 1.0 / (M * T)
        total = 0.0
        for m in range(M):
            total += self.micro_batch(p, tokens[m], list(lengths), grads, scale)
        return total * scale, grads


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def tokens_for(M, T, vocab, seed=1234):
    """Synthetic tokens, uniform in [0, V): counter-based (PCG64 with a fixed seed)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, vocab, size=(M, T + 1), dtype=np.int64).astype(np.int32)
