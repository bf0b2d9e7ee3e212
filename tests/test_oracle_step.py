"""Pins the float64 step oracle (oracle/step.py) against torch autograd in float64 on CPU,
so the GPU parity tests compare against a checked restatement."""
import numpy as np
import pytest
import torch

from oracle import step as so


def torch_reference(P, tokens, n_layer, n_head, vocab, B):
    T = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in P.items()}
    tok = torch.tensor(tokens, dtype=torch.long)
    b, sp1 = tok.shape
    s = sp1 - 1
    inp, tgt = tok[:, :s], tok[:, 1:]
    h = T["wte"].shape[1]
    x = T["wte"][inp] + T["wpe"][:s][None]
    for i in range(n_layer):
        p = lambda n: T[f"h{i}.{n}"]  # noqa: E731
        a = torch.nn.functional.layer_norm(x, (h,), p("ln1_g")[0], p("ln1_b")[0], 1e-5)
        qkv = a @ p("w_qkv").T + p("b_qkv")[0]
        q, k, v = (qkv[..., j * h:(j + 1) * h].view(b, s, n_head, h // n_head).transpose(1, 2) for j in range(3))
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + o.transpose(1, 2).reshape(b, s, h) @ p("w_o").T + p("b_o")[0]
        a = torch.nn.functional.layer_norm(x, (h,), p("ln2_g")[0], p("ln2_b")[0], 1e-5)
        u = a @ p("w_fc").T + p("b_fc")[0]
        x = x + torch.nn.functional.gelu(u, approximate="tanh") @ p("w_proj").T + p("b_proj")[0]
    a = torch.nn.functional.layer_norm(x, (h,), T["lnf_g"][0], T["lnf_b"][0], 1e-5)
    logits = a @ T["wte"][:vocab].T
    loss = torch.nn.functional.cross_entropy(logits.reshape(-1, vocab), tgt.reshape(-1), reduction="sum") / (B * s)
    loss.backward()
    return loss.item(), {k: v.grad.numpy() for k, v in T.items()}


def random_params(rng, n_layer, h, ff, vocab_pad, s):
    P = {"wte": rng.normal(0, 0.1, (vocab_pad, h)), "wpe": rng.normal(0, 0.1, (s, h)),
         "lnf_g": 1 + rng.normal(0, 0.1, (1, h)), "lnf_b": rng.normal(0, 0.1, (1, h))}
    for i in range(n_layer):
        P.update({f"h{i}.ln1_g": 1 + rng.normal(0, 0.1, (1, h)), f"h{i}.ln1_b": rng.normal(0, 0.1, (1, h)),
                  f"h{i}.w_qkv": rng.normal(0, 0.1, (3 * h, h)), f"h{i}.b_qkv": rng.normal(0, 0.1, (1, 3 * h)),
                  f"h{i}.w_o": rng.normal(0, 0.1, (h, h)), f"h{i}.b_o": rng.normal(0, 0.1, (1, h)),
                  f"h{i}.ln2_g": 1 + rng.normal(0, 0.1, (1, h)), f"h{i}.ln2_b": rng.normal(0, 0.1, (1, h)),
                  f"h{i}.w_fc": rng.normal(0, 0.1, (ff, h)), f"h{i}.b_fc": rng.normal(0, 0.1, (1, ff)),
                  f"h{i}.w_proj": rng.normal(0, 0.1, (h, ff)), f"h{i}.b_proj": rng.normal(0, 0.1, (1, h))})
    return P


@pytest.mark.parametrize("b,B", [(2, 2), (2, 5)])
def test_step_oracle_matches_autograd(b, B):
    rng = np.random.default_rng(0)
    L, h, H, ff, V, Vp, s = 2, 32, 4, 64, 50, 64, 16
    P = random_params(rng, L, h, ff, Vp, s)
    tokens = rng.integers(0, V, (b, s + 1))
    loss, G = so.gpt_loss_and_grads(P, tokens, L, H, V, B)
    tl, TG = torch_reference(P, tokens, L, H, V, B)
    assert abs(loss - tl) <= 1e-12 * max(1.0, abs(tl))
    for k in P:
        assert so.rel_err(G[k], TG[k]) < 1e-10, k


def test_split_batch_invariance():
    """Sum of per-micro-batch grads (each scaled by 1/(B*s)) == full-batch grads: the
    b_i/B weighting that the heterogeneous plan relies on."""
    rng = np.random.default_rng(1)
    L, h, H, ff, V, Vp, s = 1, 32, 2, 64, 40, 64, 8
    P = random_params(rng, L, h, ff, Vp, s)
    tokens = rng.integers(0, V, (7, s + 1))
    l_all, G_all = so.gpt_loss_and_grads(P, tokens, L, H, V, 7)
    acc, lsum = None, 0.0
    for lo, hi in ((0, 3), (3, 4), (4, 7)):
        l, G = so.gpt_loss_and_grads(P, tokens[lo:hi], L, H, V, 7)
        lsum += l
        acc = G if acc is None else {k: acc[k] + G[k] for k in G}
    assert abs(lsum - l_all) < 1e-12
    for k in P:
        assert so.rel_err(acc[k], G_all[k]) < 1e-12


def torch_llama(P, tokens, n_layer, n_head, vocab, B):
    T = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in P.items()}
    tok = torch.tensor(tokens, dtype=torch.long)
    b, sp1 = tok.shape
    s = sp1 - 1
    inp, tgt = tok[:, :s], tok[:, 1:]
    h = T["wte"].shape[1]
    dh = h // n_head
    half = dh // 2
    j = torch.arange(half, dtype=torch.float64)
    ang = torch.arange(s, dtype=torch.float64)[:, None] * (10000.0 ** (-2.0 * j / dh))[None]
    cos, sin = torch.cos(ang), torch.sin(ang)

    def rope(x):
        a, b_ = x[..., :half], x[..., half:]
        return torch.cat([a * cos - b_ * sin, b_ * cos + a * sin], -1)

    def rms(x, g):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-5) * g

    x = T["wte"][inp]
    for i in range(n_layer):
        p = lambda n: T[f"h{i}.{n}"]  # noqa: E731
        a = rms(x, p("ln1_g")[0])
        qkv = a @ p("w_qkv").T
        q, k, v = (qkv[..., m * h:(m + 1) * h].view(b, s, n_head, dh).transpose(1, 2) for m in range(3))
        o = torch.nn.functional.scaled_dot_product_attention(rope(q), rope(k), v, is_causal=True)
        x = x + o.transpose(1, 2).reshape(b, s, h) @ p("w_o").T
        m_ = rms(x, p("ln2_g")[0])
        w = p("w_gu")
        r = torch.arange(w.shape[0])
        wg, wu = w[(r % 64) < 32], w[(r % 64) >= 32]
        x = x + (torch.nn.functional.silu(m_ @ wg.T) * (m_ @ wu.T)) @ p("w_down").T
    xf = rms(x, T["lnf_g"][0])
    logits = xf @ T["lm_head"][:vocab].T
    loss = torch.nn.functional.cross_entropy(logits.reshape(-1, vocab), tgt.reshape(-1), reduction="sum") / (B * s)
    loss.backward()
    return loss.item(), {k: v.grad.numpy() for k, v in T.items()}


@pytest.mark.parametrize("H", [2, 1])  # head_dim 64 and 128
def test_llama_oracle_matches_autograd(H):
    rng = np.random.default_rng(4)
    L, h, ff, V, Vp, s = 2, 128, 64, 50, 64, 16
    P = {"wte": rng.normal(0, 0.1, (Vp, h)), "lnf_g": 1 + rng.normal(0, 0.1, (1, h)),
         "lm_head": rng.normal(0, 0.1, (Vp, h))}
    for i in range(L):
        P.update({f"h{i}.ln1_g": 1 + rng.normal(0, 0.1, (1, h)), f"h{i}.w_qkv": rng.normal(0, 0.1, (3 * h, h)),
                  f"h{i}.w_o": rng.normal(0, 0.1, (h, h)), f"h{i}.ln2_g": 1 + rng.normal(0, 0.1, (1, h)),
                  f"h{i}.w_gu": rng.normal(0, 0.1, (2 * ff, h)), f"h{i}.w_down": rng.normal(0, 0.1, (h, ff))})
    tokens = rng.integers(0, V, (3, s + 1))
    loss, G = so.llama_loss_and_grads(P, tokens, L, H, V, 5)
    tl, TG = torch_llama(P, tokens, L, H, V, 5)
    assert abs(loss - tl) <= 1e-12 * max(1.0, abs(tl))
    for k in P:
        assert so.rel_err(G[k], TG[k]) < 1e-10, k
