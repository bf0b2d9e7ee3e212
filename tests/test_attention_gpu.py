"""Fused tcgen05 causal attention vs a PyTorch fp32 reference of the same op (autograd for the
gradients). Inputs are exact bf16; P is rounded to bf16 before the P*V / dV / dK products on the
GPU, so tolerance is the bf16 path's rel 2e-2 (Frobenius); LSE rel 1e-5 (fp32 path)."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def ref_attention(qkv, b, s, H):
    h = qkv.shape[1] // 3
    d = h // H
    q, k, v = (qkv[:, j * h:(j + 1) * h].float().view(b, s, H, d).transpose(1, 2) for j in range(3))
    S = (q @ k.transpose(-1, -2)) / math.sqrt(d)
    S = S.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool, device=qkv.device), 1), float("-inf"))
    lse = torch.logsumexp(S, -1)
    o = torch.softmax(S, -1) @ v
    return o.transpose(1, 2).reshape(b * s, h), lse.reshape(-1)


def relerr(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


@pytest.mark.parametrize("b,s,H,ctas", [(1, 128, 1, 0), (2, 256, 2, 0), (2, 1024, 12, 0), (3, 512, 4, 37)])
def test_attention_fwd_bwd(cuda, b, s, H, ctas):
    check_attention(cuda, b, s, H, ctas)


def check_attention(cuda, b, s, H, ctas, d=64):
    from paper_2408_12596_b200 import _lib
    L = _lib.lib
    h = H * d
    T = b * s
    g = torch.Generator(device="cpu").manual_seed(b * 1000 + s + H)
    qkv = torch.randn(T, 3 * h, generator=g).to(torch.bfloat16).to(cuda)
    out = torch.empty(T, h, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(b * H * s, dtype=torch.float32, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    assert L.zp_attention_fwd_hd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), b, s, H, d, ctas, st) == 0
    torch.cuda.synchronize()
    ro, rl = ref_attention(qkv, b, s, H)
    assert relerr(lse, rl) < 1e-5
    assert relerr(out, ro) < 2e-2
    # backward
    dout = torch.randn(T, h, generator=g).to(torch.bfloat16).to(cuda)
    dvec = torch.empty(b * H * s, dtype=torch.float32, device=cuda)
    dq32 = torch.empty(T, h, dtype=torch.float32, device=cuda)
    dqkv = torch.zeros(T, 3 * h, dtype=torch.bfloat16, device=cuda)
    assert L.zp_attention_bwd_hd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dvec.data_ptr(),
                                 dq32.data_ptr(), dqkv.data_ptr(), b, s, H, d, ctas, st) == 0
    torch.cuda.synchronize()
    x = qkv.float().requires_grad_(True)
    o, _ = ref_attention(x, b, s, H)
    (gx,) = torch.autograd.grad(o, x, dout.float())
    for j, name in enumerate("QKV"):
        e = relerr(dqkv[:, j * h:(j + 1) * h], gx[:, j * h:(j + 1) * h])
        assert e < 2e-2, (name, e)


def test_attention_perf_smoke(cuda):
    """Not a gate: prints fused attention fwd/bwd time at GPT-2-small shapes (b=16)."""
    from paper_2408_12596_b200 import _lib
    L = _lib.lib
    b, s, H = 16, 1024, 12
    h, T = H * 64, b * s
    qkv = torch.randn(T, 3 * h, device=cuda).to(torch.bfloat16)
    out = torch.empty(T, h, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(b * H * s, device=cuda)
    dout = torch.randn(T, h, device=cuda).to(torch.bfloat16)
    dvec = torch.empty(b * H * s, device=cuda)
    dq32 = torch.empty(T, h, device=cuda)
    dqkv = torch.empty(T, 3 * h, dtype=torch.bfloat16, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for rep in range(3):
        ev[0].record()
        L.zp_attention_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), b, s, H, 0, st)
        ev[1].record()
        L.zp_attention_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dvec.data_ptr(),
                           dq32.data_ptr(), dqkv.data_ptr(), b, s, H, 0, st)
        ev[2].record()
    torch.cuda.synchronize()
    f = ev[0].elapsed_time(ev[1])
    bw = ev[1].elapsed_time(ev[2])
    flops = 4.0 * b * H * s * s * 64 / 2  # causal half of QK^T + PV
    print(f"\n[attention b={b} s={s} H={H}] fwd {f:.3f} ms ({flops / f / 1e9:.0f} TFLOP/s) "
          f"bwd {bw:.3f} ms ({2.5 * flops / bw / 1e9:.0f} TFLOP/s)")


@pytest.mark.parametrize("b,s,H,ctas", [(1, 128, 1, 0), (1, 256, 2, 0), (2, 384, 3, 0), (2, 1024, 8, 0),
                                        (1, 2048, 16, 37), (1, 4096, 32, 0)])
def test_attention_fwd_head_dim_128(cuda, b, s, H, ctas):
    """head_dim 128 forward (two query tiles per CTA sharing K/V; P over the S columns in TMEM)."""
    from paper_2408_12596_b200 import _lib
    L = _lib.lib
    d = 128
    h, T = H * d, b * s
    g = torch.Generator(device="cpu").manual_seed(b * 1000 + s + H + 7)
    qkv = torch.randn(T, 3 * h, generator=g).to(torch.bfloat16).to(cuda)
    out = torch.empty(T, h, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(b * H * s, dtype=torch.float32, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    assert L.zp_attention_fwd_hd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), b, s, H, d, ctas, st) == 0
    torch.cuda.synchronize()
    ro, rl = ref_attention(qkv, b, s, H)
    assert relerr(lse, rl) < 1e-5
    assert relerr(out, ro) < 2e-2


def test_attention_d128_perf_smoke(cuda):
    """Not a gate: fused attention forward at the Llama-7B shape with head_dim 128 (32 heads)."""
    from paper_2408_12596_b200 import _lib
    L = _lib.lib
    b, s, H, d = 2, 4096, 32, 128
    h, T = H * d, b * s
    qkv = torch.randn(T, 3 * h, device=cuda).to(torch.bfloat16)
    out = torch.empty(T, h, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(b * H * s, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for rep in range(3):
        ev[0].record()
        L.zp_attention_fwd_hd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), b, s, H, d, 0, st)
        ev[1].record()
    torch.cuda.synchronize()
    f = ev[0].elapsed_time(ev[1])
    flops = 4.0 * b * H * s * s * d / 2
    print(f"\n[attention d128 b={b} s={s} H={H}] fwd {f:.3f} ms ({flops / f / 1e9:.0f} TFLOP/s causal)")


@pytest.mark.parametrize("b,s,H,ctas", [(1, 128, 1, 0), (1, 256, 2, 0), (2, 384, 3, 0), (2, 1024, 8, 0),
                                        (1, 2048, 16, 37), (1, 4096, 32, 0)])
def test_attention_fwd_bwd_head_dim_128(cuda, b, s, H, ctas):
    """head_dim 128 backward (transposed, S^T / dP^T regions reused for P^T, dS'^T and dQ)."""
    check_attention(cuda, b, s, H, ctas, d=128)


def test_attention_d128_bwd_perf_smoke(cuda):
    """Not a gate: fused attention backward at the Llama-7B shape with head_dim 128."""
    from paper_2408_12596_b200 import _lib
    L = _lib.lib
    b, s, H, d = 2, 4096, 32, 128
    h, T = H * d, b * s
    qkv = torch.randn(T, 3 * h, device=cuda).to(torch.bfloat16)
    out = torch.empty(T, h, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(b * H * s, device=cuda)
    dout = torch.randn(T, h, device=cuda).to(torch.bfloat16)
    dvec = torch.empty(b * H * s, device=cuda)
    dq32 = torch.empty(T, h, device=cuda)
    dqkv = torch.empty(T, 3 * h, dtype=torch.bfloat16, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    L.zp_attention_fwd_hd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), b, s, H, d, 0, st)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for rep in range(3):
        ev[0].record()
        L.zp_attention_bwd_hd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dvec.data_ptr(),
                              dq32.data_ptr(), dqkv.data_ptr(), b, s, H, d, 0, st)
        ev[1].record()
    torch.cuda.synchronize()
    bw = ev[0].elapsed_time(ev[1])
    flops = 10.0 * b * H * s * s * d / 2
    print(f"\n[attention d128 b={b} s={s} H={H}] bwd {bw:.3f} ms ({flops / bw / 1e9:.0f} TFLOP/s causal)")
