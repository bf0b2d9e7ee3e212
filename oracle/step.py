"""ORACLE / TEST INFRASTRUCTURE — float64 numpy restatement of the training step.

The reference has no tensors: its device step is the closed form
`(compute_fixed + compute_per_batch * b)` (proj/core/src/hardware.cpp:160-167) and its
optimizer is the constant `optimizer_time` (hardware.cpp:168). Gradient / parameter parity
is therefore pinned by this independent float64 restatement of what the B200 step computes
(SURVEY.md §8c): a GPT-2-family decoder (pre-LN, learned positions, tied LM head, GELU-tanh)
with mean token cross-entropy over the GLOBAL batch of B samples, and AdamW.

Key invariant checked with it: the heterogeneous ZeRO step — any split of the B samples
into per-rank micro-batches b_i^s, any stage — equals this single-device B-sample step.
"""
from __future__ import annotations

import numpy as np

SQRT_2_OVER_PI = 0.7978845608028654
GELU_K = 0.044715


def gelu(u):
    return 0.5 * u * (1.0 + np.tanh(SQRT_2_OVER_PI * (u + GELU_K * u ** 3)))


def gelu_grad(u):
    t = np.tanh(SQRT_2_OVER_PI * (u + GELU_K * u ** 3))
    return 0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * SQRT_2_OVER_PI * (1.0 + 3.0 * GELU_K * u * u)


def ln_fwd(x, g, b, eps=1e-5):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    rs = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * rs
    return xh * g + b, (xh, rs)


def ln_bwd(dy, g, cache):
    xh, rs = cache
    gd = dy * g
    m1 = gd.mean(-1, keepdims=True)
    m2 = (gd * xh).mean(-1, keepdims=True)
    dx = rs * (gd - m1 - xh * m2)
    return dx, (dy * xh).sum(0), dy.sum(0)


def gpt_loss_and_grads(P: dict, tokens: np.ndarray, n_layer: int, n_head: int, vocab: int,
                       global_batch: int):
    """P: name -> float64 array (flat-layout names of zp_runtime_tensor_info; wte may carry
    padded rows). tokens: [b, s+1]. Returns (sum over these samples of CE / (B*s), grads)."""
    b, sp1 = tokens.shape
    s = sp1 - 1
    inp, tgt = tokens[:, :s], tokens[:, 1:]
    wte, wpe = P["wte"], P["wpe"]
    h = wte.shape[1]
    dh = h // n_head
    T = b * s
    x = wte[inp.reshape(-1)] + np.tile(wpe[:s], (b, 1))
    caches = []
    mask = np.triu(np.ones((s, s), dtype=bool), 1)
    for i in range(n_layer):
        p = lambda n: P[f"h{i}.{n}"]  # noqa: E731
        x_in = x
        ln1, c1 = ln_fwd(x_in, p("ln1_g")[0], p("ln1_b")[0])
        qkv = ln1 @ p("w_qkv").T + p("b_qkv")[0]
        q, k, v = (qkv[:, j * h:(j + 1) * h].reshape(b, s, n_head, dh).transpose(0, 2, 1, 3) for j in range(3))
        S = (q @ k.transpose(0, 1, 3, 2)) / np.sqrt(dh)
        S = np.where(mask, -np.inf, S)
        S = S - S.max(-1, keepdims=True)
        Pm = np.exp(S)
        Pm /= Pm.sum(-1, keepdims=True)
        o = (Pm @ v).transpose(0, 2, 1, 3).reshape(T, h)
        x_mid = x_in + o @ p("w_o").T + p("b_o")[0]
        ln2, c2 = ln_fwd(x_mid, p("ln2_g")[0], p("ln2_b")[0])
        u = ln2 @ p("w_fc").T + p("b_fc")[0]
        g = gelu(u)
        x = x_mid + g @ p("w_proj").T + p("b_proj")[0]
        caches.append((x_in, ln1, c1, q, k, v, Pm, o, x_mid, ln2, c2, u, g))
    lnf, cf = ln_fwd(x, P["lnf_g"][0], P["lnf_b"][0])
    logits = lnf @ wte[:vocab].T
    mx = logits.max(-1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(-1))
    t = tgt.reshape(-1)
    scale = 1.0 / (global_batch * s)
    loss = float((lse - logits[np.arange(T), t]).sum() * scale)
    dlog = np.exp(logits - lse[:, None])
    dlog[np.arange(T), t] -= 1.0
    dlog *= scale
    G = {k: np.zeros_like(v) for k, v in P.items()}
    G["wte"][:vocab] += dlog.T @ lnf
    dlnf = dlog @ wte[:vocab]
    dx, G["lnf_g"][0], G["lnf_b"][0] = ln_bwd(dlnf, P["lnf_g"][0], cf)
    for i in reversed(range(n_layer)):
        p = lambda n: P[f"h{i}.{n}"]  # noqa: E731
        x_in, ln1, c1, q, k, v, Pm, o, x_mid, ln2, c2, u, g = caches[i]
        G[f"h{i}.b_proj"][0] = dx.sum(0)
        G[f"h{i}.w_proj"] = dx.T @ g
        du = (dx @ p("w_proj")) * gelu_grad(u)
        G[f"h{i}.b_fc"][0] = du.sum(0)
        G[f"h{i}.w_fc"] = du.T @ ln2
        dln2 = du @ p("w_fc")
        d2, G[f"h{i}.ln2_g"][0], G[f"h{i}.ln2_b"][0] = ln_bwd(dln2, p("ln2_g")[0], c2)
        dx_mid = dx + d2
        G[f"h{i}.b_o"][0] = dx_mid.sum(0)
        G[f"h{i}.w_o"] = dx_mid.T @ o
        dO = (dx_mid @ p("w_o")).reshape(b, s, n_head, dh).transpose(0, 2, 1, 3)
        dV = Pm.transpose(0, 1, 3, 2) @ dO
        dP = dO @ v.transpose(0, 1, 3, 2)
        dS = Pm * (dP - (Pm * dP).sum(-1, keepdims=True)) / np.sqrt(dh)
        dQ = dS @ k
        dK = dS.transpose(0, 1, 3, 2) @ q
        dqkv = np.concatenate([a.transpose(0, 2, 1, 3).reshape(T, h) for a in (dQ, dK, dV)], axis=1)
        G[f"h{i}.b_qkv"][0] = dqkv.sum(0)
        G[f"h{i}.w_qkv"] = dqkv.T @ ln1
        dln1 = dqkv @ p("w_qkv")
        d1, G[f"h{i}.ln1_g"][0], G[f"h{i}.ln1_b"][0] = ln_bwd(dln1, p("ln1_g")[0], c1)
        dx = dx_mid + d1
    np.add.at(G["wte"], inp.reshape(-1), dx)
    G["wpe"][:s] += dx.reshape(b, s, h).sum(0)
    return loss, G


def adamw(p, m, v, g, t, lr, b1, b2, eps, wd):
    """One AdamW step in float64 (the update the B200 kernel fuses with the gradient sum)."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mhat = m / (1 - b1 ** t)
    vhat = v / (1 - b2 ** t)
    p = p - lr * (mhat / (np.sqrt(vhat) + eps) + wd * p)
    return p, m, v


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ----------------------------------------------------------------------------- Llama family
# RMSNorm (eps 1e-5), rotary Q/K (rotate-half, theta 1e4, any even head_dim), SwiGLU MLP whose fused
# gate/up weight interleaves 32-row blocks (rows r with r % 64 < 32 are gate rows), no biases,
# untied LM head. Same global-batch loss normalisation as the GPT step.

def rms_fwd(x, g, eps=1e-5):
    rs = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + eps)
    xh = x * rs
    return xh * g, (xh, rs)


def rms_bwd(dy, g, cache):
    xh, rs = cache
    gd = dy * g
    m2 = (gd * xh).mean(-1, keepdims=True)
    return rs * (gd - xh * m2), (dy * xh).sum(0)


def rope_tables(s, dh=64, theta=10000.0):
    j = np.arange(dh // 2, dtype=np.float64)
    inv = theta ** (-2.0 * j / dh)
    ang = np.arange(s, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope_apply(x, cos, sin, inverse=False):
    """x: [..., s, dh], rotate-half pairing (i, i + dh/2)."""
    sn = -sin if inverse else sin
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    return np.concatenate([a * cos - b * sn, b * cos + a * sn], axis=-1)


def causal_attention_fwd(q, k, v):
    """Causal softmax attention per (sample, head), one head at a time so no [b, H, s, s] array is
    ever held (the B200 kernel keeps scores on chip too). q, k, v: [b, H, s, dh].
    Returns o [b, H, s, dh] and the row log-sum-exp [b, H, s] of the scaled scores."""
    b, H, s, dh = q.shape
    mask = np.triu(np.ones((s, s), dtype=bool), 1)
    o = np.empty_like(q)
    lse = np.empty((b, H, s))
    for i in range(b):
        for j in range(H):
            S = (q[i, j] @ k[i, j].T) / np.sqrt(dh)
            S[mask] = -np.inf
            mx = S.max(-1, keepdims=True)
            E = np.exp(S - mx)
            l = E.sum(-1, keepdims=True)
            o[i, j] = (E / l) @ v[i, j]
            lse[i, j] = (mx + np.log(l))[:, 0]
    return o, lse


def causal_attention_bwd(q, k, v, o, lse, do):
    """Gradients of causal_attention_fwd, recomputing P from the saved log-sum-exp."""
    b, H, s, dh = q.shape
    mask = np.triu(np.ones((s, s), dtype=bool), 1)
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    for i in range(b):
        for j in range(H):
            S = (q[i, j] @ k[i, j].T) / np.sqrt(dh)
            S[mask] = -np.inf
            P = np.exp(S - lse[i, j][:, None])
            dv[i, j] = P.T @ do[i, j]
            dP = do[i, j] @ v[i, j].T
            D = (do[i, j] * o[i, j]).sum(-1, keepdims=True)
            dS = P * (dP - D) / np.sqrt(dh)
            dq[i, j] = dS @ k[i, j]
            dk[i, j] = dS.T @ q[i, j]
    return dq, dk, dv


def gu_split(w):
    r = np.arange(w.shape[0])
    return w[(r % 64) < 32], w[(r % 64) >= 32]


def gu_merge(dg, du):
    f = dg.shape[0]
    out = np.zeros((2 * f,) + dg.shape[1:], dtype=dg.dtype)
    r = np.arange(2 * f)
    out[(r % 64) < 32] = dg
    out[(r % 64) >= 32] = du
    return out


def llama_loss_and_grads(P: dict, tokens: np.ndarray, n_layer: int, n_head: int, vocab: int,
                         global_batch: int):
    b, sp1 = tokens.shape
    s = sp1 - 1
    inp, tgt = tokens[:, :s], tokens[:, 1:]
    h = P["wte"].shape[1]
    dh = h // n_head
    T = b * s
    cos, sin = rope_tables(s, dh)
    x = P["wte"][inp.reshape(-1)].copy()
    caches = []
    heads = lambda m: m.reshape(b, s, n_head, dh).transpose(0, 2, 1, 3)  # noqa: E731
    for i in range(n_layer):
        p = lambda n: P[f"h{i}.{n}"]  # noqa: E731
        x_in = x
        a, c1 = rms_fwd(x_in, p("ln1_g")[0])
        qkv = a @ p("w_qkv").T
        q = rope_apply(heads(qkv[:, :h]), cos, sin)
        k = rope_apply(heads(qkv[:, h:2 * h]), cos, sin)
        v = heads(qkv[:, 2 * h:])
        oh, lse_a = causal_attention_fwd(q, k, v)
        o = oh.transpose(0, 2, 1, 3).reshape(T, h)
        x_mid = x_in + o @ p("w_o").T
        m, c2 = rms_fwd(x_mid, p("ln2_g")[0])
        wg, wu = gu_split(p("w_gu"))
        ga, ub = m @ wg.T, m @ wu.T
        sg = 1.0 / (1.0 + np.exp(-ga))
        hh = ga * sg * ub
        x = x_mid + hh @ p("w_down").T
        caches.append((x_in, a, c1, q, k, v, (oh, lse_a), o, x_mid, m, c2, ga, ub, sg, hh))
    xf, cf = rms_fwd(x, P["lnf_g"][0])
    W = P["lm_head"][:vocab]
    logits = xf @ W.T
    mx = logits.max(-1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(-1))
    t = tgt.reshape(-1)
    scale = 1.0 / (global_batch * s)
    loss = float((lse - logits[np.arange(T), t]).sum() * scale)
    dlog = np.exp(logits - lse[:, None])
    dlog[np.arange(T), t] -= 1.0
    dlog *= scale
    G = {k_: np.zeros_like(v_) for k_, v_ in P.items()}
    G["lm_head"][:vocab] = dlog.T @ xf
    dx, G["lnf_g"][0] = rms_bwd(dlog @ W, P["lnf_g"][0], cf)
    unheads = lambda m: m.transpose(0, 2, 1, 3).reshape(T, h)  # noqa: E731
    for i in reversed(range(n_layer)):
        p = lambda n: P[f"h{i}.{n}"]  # noqa: E731
        x_in, a, c1, q, k, v, (oh, lse_a), o, x_mid, m, c2, ga, ub, sg, hh = caches[i]
        G[f"h{i}.w_down"] = dx.T @ hh
        dhh = dx @ p("w_down")
        silu = ga * sg
        dub = dhh * silu
        dga = dhh * ub * sg * (1.0 + ga * (1.0 - sg))
        wg, wu = gu_split(p("w_gu"))
        G[f"h{i}.w_gu"] = gu_merge(dga.T @ m, dub.T @ m)
        dm = dga @ wg + dub @ wu
        d2, G[f"h{i}.ln2_g"][0] = rms_bwd(dm, p("ln2_g")[0], c2)
        dx_mid = dx + d2
        G[f"h{i}.w_o"] = dx_mid.T @ o
        dO = heads(dx_mid @ p("w_o"))
        dQr, dKr, dV = causal_attention_bwd(q, k, v, oh, lse_a, dO)
        dQ = rope_apply(dQr, cos, sin, inverse=True)
        dK = rope_apply(dKr, cos, sin, inverse=True)
        dqkv = np.concatenate([unheads(dQ), unheads(dK), unheads(dV)], axis=1)
        G[f"h{i}.w_qkv"] = dqkv.T @ a
        d1, G[f"h{i}.ln1_g"][0] = rms_bwd(dqkv @ p("w_qkv"), p("ln1_g")[0], c1)
        dx = dx_mid + d1
    np.add.at(G["wte"], inp.reshape(-1), dx)
    return loss, G


def loss_and_grads(P, tokens, n_layer, n_head, vocab, global_batch, arch=0):
    f = llama_loss_and_grads if arch == 1 else gpt_loss_and_grads
    return f(P, tokens, n_layer, n_head, vocab, global_batch)
