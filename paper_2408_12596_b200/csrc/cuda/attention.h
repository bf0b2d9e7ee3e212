// Fused causal attention (head_dim 64 or 128) on tcgen05: the s x s scores never reach HBM.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace zp {

using bf16 = __nv_bfloat16;

// qkv: [batch*seq, 3h] (Q | K | V, heads of head_dim contiguous); out: [batch*seq, h];
// lse: [batch*heads*seq] fp32 natural-log row log-sum-exp of the scaled scores.
cudaError_t attention_fwd(const bf16* qkv, bf16* out, float* lse, int64_t batch, int seq, int heads,
                          int ctas, cudaStream_t s, int head_dim = 64);

// dout: [batch*seq, h]; writes dqkv [batch*seq, 3h]. Workspaces: dvec [batch*heads*seq] fp32,
// dq32 [batch*seq, h] fp32. rope_tab (head_dim 128 only; float2 [seq][64], kernels.h rope_table):
// dQ and dK are written through the inverse rotary embedding (the Q, K of qkv are rotated).
// dvec_ready (head_dim 128 only): dvec already holds D = rowsum(dout * out) per head and dq32 is
// zero (the GEMM epilogue kEpiDvecBf16 that produced dout did both).
cudaError_t attention_bwd(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, float* dvec,
                          float* dq32, bf16* dqkv, int64_t batch, int seq, int heads, int ctas, cudaStream_t s,
                          int head_dim = 64, const float2* rope_tab = nullptr, bool dvec_ready = false);

}  // namespace zp
