import os, sys, torch
sys.path.insert(0, os.getcwd())
from tests.test_gemm_gpu import run_gemm
from tools.gemm_bench import timeit
dev = torch.device("cuda:0")
M, f, K = 16384, 5504, 2048
A = (torch.randn(M, K, device=dev) * 0.1).to(torch.bfloat16)
B = (torch.randn(2 * f, K, device=dev) * 0.1).to(torch.bfloat16)
C = torch.empty(M * 2 * f, device=dev, dtype=torch.bfloat16)
H = torch.empty(M * f, device=dev, dtype=torch.bfloat16)
for rep in range(2):
    t0 = timeit(lambda: run_gemm(A, 0, B, 0, M, 2 * f, K, c=C, ldc=2 * f, epilogue=0, sync=False))
    t8 = timeit(lambda: run_gemm(A, 0, B, 0, M, 2 * f, K, c=C, ldc=2 * f, epilogue=8, aux_out=H, sync=False))
    gu = C.view(M, 2 * f)
    ts = timeit(lambda: torch.nn.functional.silu(gu[:, :f]) * gu[:, f:])  # torch reference elementwise cost (2 reads + write)
    print(f"gate/up GEMM plain {t0:.3f} ms, with fused SwiGLU {t8:.3f} ms (delta {t8 - t0:.3f}); torch silu*up {ts:.3f} ms")
