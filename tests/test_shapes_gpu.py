"""Parity at the benchmarked shapes (BASELINE.json configs C2-C5): one real iteration of the
runtime (tcgen05 GEMMs with their CTA-pair / split-K / TMA-epilogue paths, fused attention at the
configs' sequence lengths, the full LM head and cross-entropy) against a plain PyTorch fp32
reference of the same step (tests/torch_ref.py) on the same bf16 parameters and tokens.

Models are cut to two layers (every layer of a config has the same shapes); widths, heads,
vocabularies, sequence lengths and per-rank micro-batches are the configs' own:
  C2 GPT-2 small  h768  H12 V50257 s1024, b=128 (T=131072 tokens), ZeRO-2
  C3 GPT-2 medium h1024 H16 V50257 s1024, b=32, ZeRO-3
  C4 Llama 1.3B   h2048 ff5504 V32000 s2048, b=4, ZeRO-3
  C5 Llama 7B     h4096 ff11008 V32000 s4096, b=2, ZeRO-3
Tolerance (north star, bf16 path): every parameter's gradient within rel 2e-2 (Frobenius), the
loss within rel 5e-3. At the C5 width (h = 4096) a standard bf16 implementation of the same step
(the PyTorch reference under bf16 autocast) is itself 2.7-2.9e-2 away from fp32 on the last layer's
attention-input gradients (profiles/r2_bf16_yardstick.md), so there a gradient may exceed 2e-2
only if it is no further from fp32 than that bf16 yardstick (x 1.02).
Large standalone GEMM and attention shapes of the same configs follow.
"""
import numpy as np
import pytest
import torch

from tests import torch_ref

pytestmark = pytest.mark.gpu


def _plan(stage, b):
    return dict(stage=stage, gbs=b, gas=1, devices=[dict(device_id=0, b=b, gmbs=b, lbs=b, predicted_time=0.0)],
                iteration_time=0.0, idle=[0.0], under_utilization=[0.0], objective=0.0, weights=[1.0],
                predicted_wall_time=0.0)


def _relerr(a, b):
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


CASES = {
    "c2-gpt2-small-b128": (dict(n_layer=2, d_model=768, n_head=12, vocab=50257, seq_len=1024), 128, 2),
    "c3-gpt2-medium-b32": (dict(n_layer=2, d_model=1024, n_head=16, vocab=50257, seq_len=1024), 32, 3),
    "c4-llama1.3b-b4": (dict(n_layer=2, d_model=2048, n_head=16, vocab=32000, seq_len=2048, d_ff=5504, arch=1), 4, 3),
    "c5-llama7b-b2": (dict(n_layer=2, d_model=4096, n_head=32, vocab=32000, seq_len=4096, d_ff=11008, arch=1), 2, 3),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_step_at_benchmark_shape(cuda, case):
    from paper_2408_12596_b200.models import MODELS, GPT
    from paper_2408_12596_b200.runtime import Runtime, bf16_to_f32
    shape, b, stage = CASES[case]
    full = next(m for m in MODELS.values() if m.d_model == shape["d_model"] and m.vocab == shape["vocab"])
    shape = dict(shape, n_head=full.n_head, d_ff=full.d_ff)  # the configs' own head layout
    cfg = GPT(**shape)
    rt = Runtime(cfg, seed=11, lr=1e-4, hbm_cap_bytes=70 << 30)
    rt.keep_grads(True)
    rt.resident_bytes(stage)
    flat = bf16_to_f32(rt.params_bf16())
    names = rt.tensor_names()
    info = {n: rt.tensor_info(n) for n in names}
    rng = np.random.default_rng(5)
    tok = rng.integers(0, cfg.vocab, (b, cfg.seq_len + 1)).astype(np.int32)
    rt.load_tokens(tok)
    t = rt.execute_iteration(_plan(stage, b), stage)
    g, _ = rt.state_flat(3)
    rt.close()

    tt = torch.tensor(tok, dtype=torch.long, device=cuda)

    def reference(bf16):
        P = {n: torch.tensor(flat[o:o + r * c].reshape(r, c), device=cuda, requires_grad=True)
             for n, (o, r, c) in info.items()}
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=bf16):
            loss = torch_ref.loss_fn(cfg.arch)(P, tt, cfg.n_layer, cfg.n_head, cfg.vocab, b)
        loss.backward()
        return loss.item(), {n: P[n].grad for n in P}

    loss, G = reference(False)
    assert abs(t["loss_sum"] - loss) <= 5e-3 * abs(loss), (t["loss_sum"], loss)
    h = cfg.d_model
    G16 = None
    worst = (0.0, "")
    for n, (o, r, c) in info.items():
        got = torch.tensor(g[o:o + r * c].reshape(r, c), device=cuda)
        ref = G[n]
        if n.endswith("b_qkv"):  # the key bias has a zero gradient (softmax shift invariance)
            got = torch.cat([got[:, :h], got[:, 2 * h:]], 1)
            ref = torch.cat([ref[:, :h], ref[:, 2 * h:]], 1)
        e = _relerr(got, ref)
        worst = max(worst, (e, n))
        if e >= 2e-2:
            if G16 is None:
                G16 = reference(True)[1]
            yard = _relerr(G16[n], G[n])
            assert e <= 1.02 * yard, (n, e, "bf16 yardstick", yard)
    print(f"\n[{case}] loss {t['loss_sum']:.5f} vs {loss:.5f}; worst grad rel err {worst[0]:.2e} ({worst[1]})")


# ---------------------------------------------------------------- GEMMs at the configs' shapes
def _gemm():
    from tests.test_gemm_gpu import run_gemm
    return run_gemm


@pytest.mark.parametrize("M,N,K,what", [
    (131072, 3072, 768, "C2 fc + bias + GELU, T=131072"),
    (8192, 32000, 4096, "C5 LM head"),
    (8192, 4096, 11008, "C5 down projection"),
    (16384, 6144, 2048, "C4 QKV"),
])
def test_gemm_forward_shapes(cuda, M, N, K, what):
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).to(cuda)
    B = (torch.randn(N, K, generator=g) / K ** 0.5).to(torch.bfloat16).to(cuda)
    ref = A.float() @ B.float().t()
    if "GELU" in what:
        bias = torch.randn(N, device=cuda).to(torch.bfloat16)
        gp = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
        C = _gemm()(A, 0, B, 0, M, N, K, out_dtype=torch.bfloat16, epilogue=5, bias=bias, aux_out=gp).view(M, N)
        ref = torch.nn.functional.gelu(ref + bias.float(), approximate="tanh")
        assert _relerr(C.float(), ref) < 1e-2, what
    else:
        C = _gemm()(A, 0, B, 0, M, N, K, out_dtype=torch.bfloat16, epilogue=0).view(M, N)
        assert _relerr(C.float(), ref) < 8e-3, what


@pytest.mark.parametrize("M,N,T,what", [
    (4096, 11008, 8192, "C5 w_down weight gradient (split-K)"),
    (22016, 4096, 8192, "C5 w_gu weight gradient"),
    (3072, 768, 131072, "C2 w_qkv weight gradient, T=131072"),
])
def test_gemm_weight_gradient_shapes(cuda, M, N, T, what):
    g = torch.Generator(device="cpu").manual_seed(M + N + T)
    dY = (0.1 * torch.randn(T, M, generator=g)).to(torch.bfloat16).to(cuda)
    X = torch.randn(T, N, generator=g).to(torch.bfloat16).to(cuda)
    C = torch.zeros(M * N, device=cuda)
    _gemm()(dY, 1, X, 1, M, N, T, epilogue=7, c=C, ldc=N, split_k=-1)
    # fp32 tensor-core accumulation error grows with the reduction length: 1e-5 per 8192 tokens
    assert _relerr(C.view(M, N), dY.float().t() @ X.float()) < 1e-5 * max(1, T // 8192), what


def test_gemm_swiglu_c5_shape(cuda):
    M, f, K = 8192, 11008, 4096
    A = torch.randn(M, K, device=cuda).to(torch.bfloat16)
    B = (torch.randn(2 * f, K, device=cuda) / K ** 0.5).to(torch.bfloat16)
    H = torch.empty(M, f, device=cuda, dtype=torch.bfloat16)
    C = _gemm()(A, 0, B, 0, M, 2 * f, K, out_dtype=torch.bfloat16, epilogue=8, aux_out=H).view(M, 2 * f)
    acc = A.float() @ B.float().t()
    assert _relerr(C.float(), acc) < 8e-3
    cols = torch.arange(2 * f, device=cuda)
    gate, up = acc[:, (cols % 64) < 32], acc[:, (cols % 64) >= 32]
    assert _relerr(H.float(), torch.nn.functional.silu(gate) * up) < 1e-2


# ---------------------------------------------------------------- attention at the configs' lengths
@pytest.mark.parametrize("b,s,H,d", [(2, 2048, 32, 64), (1, 4096, 64, 64), (2, 2048, 16, 128), (1, 4096, 32, 128)])
def test_attention_long_sequences(cuda, b, s, H, d):
    from tests.test_attention_gpu import check_attention
    check_attention(cuda, b, s, H, 0, d=d)
