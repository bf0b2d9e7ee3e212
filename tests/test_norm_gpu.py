"""LayerNorm / RMSNorm backward (kernels.cu: ln_bwd_fused_k for narrow rows, ln_bwd_rows_k for
h = 2048 / 4096) through the C ABI (zp_norm_bwd) vs a PyTorch fp32 reference of the same formula:
dx (bf16 output: rel 1e-2 Frobenius, from exact bf16 inputs and the forward's fp32 statistics),
the summed dgamma / dbeta / dx column partials (fp32: rel 1e-4)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


@pytest.mark.parametrize("rows,h,rms,res,cs", [
    (1000, 768, False, True, True),     # GPT-2 small: warp-per-row kernel, LN + dx column sums
    (517, 1024, False, False, False),
    (4096, 2048, True, True, False),    # Llama-1.3B: row-per-CTA kernel
    (333, 2048, False, True, True),
    (8192, 4096, True, True, False),    # Llama-7B (C5 micro-step rows)
    (129, 4096, True, False, False),
    (300, 4096, False, True, False),    # h = 4096 LayerNorm: rows kernel + column kernel (smem > 200 KB)
])
def test_norm_bwd_matches_fp32(cuda, rows, h, rms, res, cs):
    from paper_2408_12596_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(rows + h)
    x = torch.randn(rows, h, generator=g).to(torch.bfloat16).to(cuda)
    dy = torch.randn(rows, h, generator=g).to(torch.bfloat16).to(cuda)
    gamma = (1 + 0.1 * torch.randn(h, generator=g)).to(torch.bfloat16).to(cuda)
    dres = torch.randn(rows, h, generator=g).to(torch.bfloat16).to(cuda) if res else None
    xf = x.float()
    mean = torch.zeros(rows, device=cuda) if rms else xf.mean(1)
    var = (xf * xf).mean(1) if rms else ((xf - mean[:, None]) ** 2).mean(1)
    rstd = torch.rsqrt(var + 1e-5)
    dx = torch.empty(rows, h, dtype=torch.bfloat16, device=cuda)
    part = torch.zeros(2 * 592 * h, device=cuda)
    csp = torch.zeros(592 * h, device=cuda) if cs else None
    nparts = torch.zeros(1, dtype=torch.int32)
    st = torch.cuda.current_stream().cuda_stream
    rc = _lib.lib.zp_norm_bwd(dy.data_ptr(), x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), gamma.data_ptr(),
                              dres.data_ptr() if res else None, dx.data_ptr(), part.data_ptr(), part.numel(),
                              csp.data_ptr() if cs else None, csp.numel() if cs else 0, nparts.data_ptr(), rows, h,
                              int(rms), 0, st)
    assert rc == 0
    torch.cuda.synchronize()
    n = int(nparts.item())
    xh = (xf - mean[:, None]) * rstd[:, None]
    gd = gamma.float()[None, :] * dy.float()
    m1 = torch.zeros(rows, 1, device=cuda) if rms else gd.mean(1, keepdim=True)
    m2 = (gd * xh).mean(1, keepdim=True)
    ref = rstd[:, None] * (gd - m1 - xh * m2)
    if res:
        ref = ref + dres.float()
    assert relerr(dx, ref) < 1e-2
    dgamma = part[:n * h].view(n, h).sum(0)
    assert relerr(dgamma, (xh * dy.float()).sum(0)) < 1e-4
    if not rms:
        assert relerr(part[n * h:2 * n * h].view(n, h).sum(0), dy.float().sum(0)) < 1e-4
    if cs:
        assert relerr(csp[:n * h].view(n, h).sum(0), ref.sum(0)) < 1e-4


def test_norm_bwd_rejects_bad_arguments(cuda):
    from paper_2408_12596_b200 import _lib
    part = torch.zeros(2 * 592 * 256, device=cuda)
    n = torch.zeros(1, dtype=torch.int32)
    x = torch.zeros(4, 300, dtype=torch.bfloat16, device=cuda)
    # h not a multiple of 256
    assert _lib.lib.zp_norm_bwd(x.data_ptr(), x.data_ptr(), part.data_ptr(), part.data_ptr(), x.data_ptr(), None,
                                x.data_ptr(), part.data_ptr(), part.numel(), None, 0, n.data_ptr(), 4, 300, 1, 0,
                                None) == 1


def test_norm_bwd_perf_smoke(cuda):
    """C5 shape (8192 rows x 4096, RMSNorm with the residual gradient): bytes = x, dy, dres read +
    dx written (bf16), against the measured HBM peak."""
    import json
    import os
    from paper_2408_12596_b200 import _lib
    rows, h = 8192, 4096
    x, dy, dres = (torch.randn(rows, h, device=cuda).to(torch.bfloat16) for _ in range(3))
    gamma = torch.ones(h, dtype=torch.bfloat16, device=cuda)
    mean, rstd = torch.zeros(rows, device=cuda), torch.ones(rows, device=cuda)
    dx = torch.empty_like(x)
    part = torch.zeros(2 * 592 * h, device=cuda)
    n = torch.zeros(1, dtype=torch.int32)
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=cuda)

    def run():
        assert _lib.lib.zp_norm_bwd(dy.data_ptr(), x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), gamma.data_ptr(),
                                    dres.data_ptr(), dx.data_ptr(), part.data_ptr(), part.numel(), None, 0,
                                    n.data_ptr(), rows, h, 1, 0, st) == 0
    run()
    best = 1e9
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    gbs = 4 * rows * h * 2 / best / 1e9
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "MEASURED_PEAKS.json")))
    peak = peak.get("hbm_gbs", 6547.8) if isinstance(peak, dict) else 6547.8
    print(f"[rmsnorm bwd {rows}x{h}] {best * 1e6:.1f} us, {gbs:.0f} GB/s = {gbs / peak:.2f} of HBM")
    assert gbs > 0.3 * peak
