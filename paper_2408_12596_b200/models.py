"""Model shapes of the benchmark configurations (BASELINE.json configs).

Pure Python on purpose: importing this module never loads libzp.so, so the reference arm of
bench.py (`--impl reference`) and the CPU baseline can name the workload without mapping the
product library.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class GPT:
    n_layer: int
    d_model: int
    n_head: int
    vocab: int
    seq_len: int
    d_ff: int = 0
    arch: int = 0  # 0 = GPT-2 family, 1 = Llama family

    def __post_init__(self):
        if not self.d_ff:
            self.d_ff = 4 * self.d_model

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_head

    def matmul_params(self) -> int:
        """Parameters that enter a GEMM per token (every linear layer + the LM head)."""
        h, f, L = self.d_model, self.d_ff, self.n_layer
        mlp = 3 * h * f if self.arch == 1 else 2 * h * f
        return L * (4 * h * h + mlp) + self.vocab * h

    def flops_per_sample(self) -> float:
        """Training FLOPs of one sample: 6 * N_matmul * s + 12 * L * h * s^2 (dense attention
        accounting)."""
        h, L, s = self.d_model, self.n_layer, self.seq_len
        return 6.0 * self.matmul_params() * s + 12.0 * L * h * s * s


MODELS = {
    "gpt-tiny": GPT(4, 256, 4, 8192, 256, 1024),
    "gpt2-small": GPT(12, 768, 12, 50257, 1024),
    "gpt2-medium": GPT(24, 1024, 16, 50257, 1024),
    # Llama-style configs of BASELINE.json with the standard head layout (head_dim 128: 16 heads at
    # h=2048, 32 heads at h=4096)
    "llama-1.3b": GPT(24, 2048, 16, 32000, 2048, 5504, arch=1),
    "llama-7b": GPT(32, 4096, 32, 32000, 4096, 11008, arch=1),
}
