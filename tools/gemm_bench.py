"""Throughput of the tcgen05 GEMM on the GPT-2-small step shapes (T = b*s tokens) next to
torch.matmul (cuBLAS) on the same shapes, CUDA-event timed, full SM count and a 132-SM cap.

    python tools/gemm_bench.py [--T 65536]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gemm_gpu import run_gemm  # noqa: E402


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=65536)
    a = ap.parse_args()
    T, h, f, V = a.T, 768, 3072, 50304
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    # name, M, N, K, a_major, b_major, epilogue
    shapes = [("fwd qkv", T, 3 * h, h, 0, 0, 0), ("fwd fc", T, f, h, 0, 0, 0), ("fwd proj", T, h, f, 0, 0, 0),
              ("fwd fc +bias", T, f, h, 0, 0, 3),
              ("fwd fc +bias+GELU(+U)", T, f, h, 0, 0, 5), ("fwd proj +bias+resid", T, h, f, 0, 0, 4),
              ("dgrad fc +GELU'", T, f, h, 0, 1, 6),
              ("lm head", T, V, h, 0, 0, 0), ("dgrad proj", T, f, h, 0, 1, 0), ("dgrad fc", T, h, f, 0, 1, 0),
              ("wgrad fc", f, h, T, 1, 1, 7), ("wgrad qkv", 3 * h, h, T, 1, 1, 7)]
    print(f"| shape | M | N | K | ours 148 SM TF/s | ours 132 SM TF/s | cuBLAS 148 SM TF/s |")
    print("|---|---:|---:|---:|---:|---:|---:|")
    for name, M, N, K, am, bm, epi in shapes:
        A = (torch.randn(M * K, device=dev) * 0.1).to(torch.bfloat16)
        B = (torch.randn(N * K, device=dev) * 0.1).to(torch.bfloat16)
        if epi == 7:
            C = torch.zeros(M * N, device=dev)
        else:
            C = torch.empty(M * N, device=dev, dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        res = []
        extra = {}
        if epi == 3:
            extra["bias"] = (torch.randn(N, device=dev) * 0.1).to(torch.bfloat16)
        if epi in (4, 5, 6):
            extra["bias"] = (torch.randn(N, device=dev) * 0.1).to(torch.bfloat16) if epi in (4, 5) else None
            aux = (torch.randn(M * N, device=dev) * 0.1).to(torch.bfloat16)
            if epi == 5:
                extra["aux_out"] = aux
            else:
                extra["aux"] = aux
        for cap in (0, 132):
            kw = dict(c=C, ldc=N, epilogue=epi, sync=False, max_ctas=cap, split_k=-1 if epi == 7 else 1, **extra)
            ms = timeit(lambda: run_gemm(A, am, B, bm, M, N, K, **kw))
            res.append(fl / ms / 1e9)
        At = A.view(M, K) if am == 0 else A.view(K, M).t()
        Bt = B.view(N, K).t() if bm == 0 else B.view(K, N)
        ms = timeit(lambda: torch.matmul(At, Bt))
        res.append(fl / ms / 1e9)
        print(f"| {name} | {M} | {N} | {K} | {res[0]:.0f} | {res[1]:.0f} | {res[2]:.0f} |", flush=True)


if __name__ == "__main__":
    main()
