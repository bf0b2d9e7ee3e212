"""Plain PyTorch fp32 references of the two decoder families the runtime trains (the numerics
reference for the GPU parity tests at the benchmarked shapes; float64 restatements of the same
maths live in oracle/step.py and are pinned to autograd by tests/test_oracle_step.py).

Parameters are a dict name -> fp32 tensor in the runtime's flat-layout shapes
(zp_runtime_tensor_info): wte / lm_head may carry padded vocabulary rows, Llama's w_gu interleaves
gate / up rows in 32-row blocks, qkv is [Q | K | V]. The loss is the sum over the batch's tokens
of cross-entropy / (B * s) (B = global batch), as the runtime scales it. The LM head + loss is
evaluated in row chunks under activation checkpointing so the [T, V] logits never exist at once.
"""
import torch
import torch.nn.functional as F
from torch.utils.checkpoint import checkpoint


def _head_ce(x, W, t, vocab):
    return F.cross_entropy(x @ W[:vocab].T, t, reduction="sum")


def chunked_ce(x, W, tgt, vocab, denom, chunk=8192):
    total = x.new_zeros(())
    for i in range(0, x.shape[0], chunk):
        total = total + checkpoint(_head_ce, x[i:i + chunk], W, tgt[i:i + chunk], vocab, use_reentrant=False)
    return total / denom


def gpt_loss(P, tok, n_layer, n_head, vocab, B):
    b, s1 = tok.shape
    s = s1 - 1
    inp, tgt = tok[:, :s], tok[:, 1:]
    h = P["wte"].shape[1]
    x = P["wte"][inp] + P["wpe"][:s][None]
    for i in range(n_layer):
        p = lambda n: P[f"h{i}.{n}"]  # noqa: E731
        a = F.layer_norm(x, (h,), p("ln1_g")[0], p("ln1_b")[0], 1e-5)
        qkv = a @ p("w_qkv").T + p("b_qkv")[0]
        q, k, v = (qkv[..., j * h:(j + 1) * h].view(b, s, n_head, h // n_head).transpose(1, 2) for j in range(3))
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + o.transpose(1, 2).reshape(b, s, h) @ p("w_o").T + p("b_o")[0]
        a = F.layer_norm(x, (h,), p("ln2_g")[0], p("ln2_b")[0], 1e-5)
        u = a @ p("w_fc").T + p("b_fc")[0]
        x = x + F.gelu(u, approximate="tanh") @ p("w_proj").T + p("b_proj")[0]
    a = F.layer_norm(x, (h,), P["lnf_g"][0], P["lnf_b"][0], 1e-5)
    return chunked_ce(a.reshape(b * s, h), P["wte"], tgt.reshape(-1), vocab, B * s)


def _rms(x, g):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-5) * g


def llama_loss(P, tok, n_layer, n_head, vocab, B):
    b, s1 = tok.shape
    s = s1 - 1
    inp, tgt = tok[:, :s], tok[:, 1:]
    h = P["wte"].shape[1]
    dh = h // n_head
    half = dh // 2
    j = torch.arange(half, dtype=torch.float64, device=tok.device)
    ang = torch.arange(s, dtype=torch.float64, device=tok.device)[:, None] * (10000.0 ** (-2.0 * j / dh))[None]
    cos, sin = torch.cos(ang).float(), torch.sin(ang).float()

    def rope(x):
        a, b_ = x[..., :half], x[..., half:]
        return torch.cat([a * cos - b_ * sin, b_ * cos + a * sin], -1)

    x = P["wte"][inp]
    for i in range(n_layer):
        p = lambda n: P[f"h{i}.{n}"]  # noqa: E731
        a = _rms(x, p("ln1_g")[0])
        qkv = a @ p("w_qkv").T
        q, k, v = (qkv[..., m * h:(m + 1) * h].view(b, s, n_head, dh).transpose(1, 2) for m in range(3))
        o = F.scaled_dot_product_attention(rope(q), rope(k), v, is_causal=True)
        x = x + o.transpose(1, 2).reshape(b, s, h) @ p("w_o").T
        m_ = _rms(x, p("ln2_g")[0])
        w = p("w_gu")
        r = torch.arange(w.shape[0], device=w.device)
        wg, wu = w[(r % 64) < 32], w[(r % 64) >= 32]
        x = x + (F.silu(m_ @ wg.T) * (m_ @ wu.T)) @ p("w_down").T
    xf = _rms(x, P["lnf_g"][0])
    return chunked_ce(xf.reshape(b * s, h), P["lm_head"], tgt.reshape(-1), vocab, B * s)


def loss_fn(arch):
    return llama_loss if arch == 1 else gpt_loss
