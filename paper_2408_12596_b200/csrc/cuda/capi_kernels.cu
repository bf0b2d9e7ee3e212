// extern "C" wrappers of the individual kernels (include/zp_kernels.h).
#include "../../../include/zp_kernels.h"
#include "attention.h"
#include "gemm.h"
#include "kernels.h"

extern "C" int zp_gemm(const zp_gemm_desc* d, void* stream) {
  if (!d) return 1;
  zp::GemmArgs a;
  a.M = d->M; a.N = d->N; a.K = d->K; a.nb1 = d->nb1; a.nb2 = d->nb2;
  a.a.ptr = d->a; a.a.major = d->a_major; a.a.ld = d->lda; a.a.bs1 = d->a_bs1; a.a.bs2 = d->a_bs2;
  a.b.ptr = d->b; a.b.major = d->b_major; a.b.ld = d->ldb; a.b.bs1 = d->b_bs1; a.b.bs2 = d->b_bs2;
  a.c = d->c; a.ldc = d->ldc; a.cs1 = d->c_bs1; a.cs2 = d->c_bs2;
  a.alpha = d->alpha;
  a.epilogue = d->epilogue;
  a.causal = d->causal;
  a.bias = d->bias;
  a.aux = d->aux;
  a.aux_out = d->aux_out;
  a.max_ctas = d->max_ctas;
  a.split_k = d->split_k;
  a.colsum = d->colsum;
  const cudaError_t e = zp::gemm(a, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : 5;
}

extern "C" int64_t zp_launch_count(void) { return zp::launch_count(); }

extern "C" int zp_attention_fwd(const void* qkv, void* out, float* lse, int64_t batch, int32_t seq,
                                int32_t heads, int32_t max_ctas, void* stream) {
  const cudaError_t e = zp::attention_fwd(static_cast<const zp::bf16*>(qkv), static_cast<zp::bf16*>(out), lse,
                                          batch, seq, heads, max_ctas, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : 5;
}

extern "C" int zp_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                                float* dvec, float* dq32, void* dqkv, int64_t batch, int32_t seq,
                                int32_t heads, int32_t max_ctas, void* stream) {
  const cudaError_t e = zp::attention_bwd(static_cast<const zp::bf16*>(qkv), static_cast<const zp::bf16*>(out),
                                          static_cast<const zp::bf16*>(dout), lse, dvec, dq32,
                                          static_cast<zp::bf16*>(dqkv), batch, seq, heads, max_ctas,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : 5;
}
