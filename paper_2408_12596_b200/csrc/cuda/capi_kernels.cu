// extern "C" wrappers of the individual kernels (include/zp_kernels.h).
#include "../../../include/zp_kernels.h"
#include "attention.h"
#include "gemm.h"
#include "kernels.h"
#include "peer.h"

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

extern "C" int zp_synth_tokens(int32_t* out, int64_t first, int64_t count, int32_t seq_plus1, int32_t vocab,
                               uint64_t seed, uint64_t iteration, void* stream) {
  if (!out || first < 0 || count < 1 || seq_plus1 < 2 || vocab < 1) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  zp::synth_tokens(out, first, count, seq_plus1, vocab, seed, iteration, sms, static_cast<cudaStream_t>(stream));
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

extern "C" int zp_attention_fwd(const void* qkv, void* out, float* lse, int64_t batch, int32_t seq,
                                int32_t heads, int32_t max_ctas, void* stream) {
  const cudaError_t e = zp::attention_fwd(static_cast<const zp::bf16*>(qkv), static_cast<zp::bf16*>(out), lse,
                                          batch, seq, heads, max_ctas, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : 5;
}

extern "C" int zp_attention_fwd_hd(const void* qkv, void* out, float* lse, int64_t batch, int32_t seq,
                                   int32_t heads, int32_t head_dim, int32_t max_ctas, void* stream) {
  const cudaError_t e = zp::attention_fwd(static_cast<const zp::bf16*>(qkv), static_cast<zp::bf16*>(out), lse,
                                          batch, seq, heads, max_ctas, static_cast<cudaStream_t>(stream), head_dim);
  return e == cudaSuccess ? 0 : (e == cudaErrorInvalidValue ? 1 : 5);
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

extern "C" int zp_norm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const void* gamma,
                           const void* dres, void* dx, float* part, int64_t part_capacity, float* colsum_part,
                           int64_t colsum_capacity, int32_t* nparts, int64_t rows, int32_t h, int32_t rms,
                           int32_t max_ctas, void* stream) {
  if (!dy || !x || !mean || !rstd || !gamma || !dx || !part || !nparts || rows < 1 || h < 256 || h % 256 ||
      part_capacity < int64_t(2) * 592 * h || (colsum_part && colsum_capacity < int64_t(592) * h))
    return 1;
  int dev = 0, ctas = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&ctas, cudaDevAttrMultiProcessorCount, dev);
  if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
  int nb = 0;
  const cudaError_t e =
      zp::layernorm_bwd(static_cast<const zp::bf16*>(dy), static_cast<const zp::bf16*>(x), mean, rstd,
                        static_cast<const zp::bf16*>(gamma), static_cast<const zp::bf16*>(dres),
                        static_cast<zp::bf16*>(dx), part, &nb, rows, h, ctas, static_cast<cudaStream_t>(stream),
                        rms != 0, colsum_part);
  *nparts = nb;
  return e == cudaSuccess ? 0 : (e == cudaErrorInvalidValue ? 1 : 5);
}

// ---- peer-memory collectives, all ranks of a group emulated on one device (include/zp_kernels.h)
struct zp_peer_group {
  zp::PeerView pv;  // rank 0's view; the emulated launch derives every rank's
  zp::PeerFlags* flags = nullptr;
  char* base = nullptr;
  int64_t arena = 0;
};

extern "C" int zp_peer_group_create(int32_t n, void* base, int64_t arena_bytes, zp_peer_group** out) {
  if (!out || !base || n < 1 || n > zp::kMaxPeers || arena_bytes <= 0) return 1;
  auto* g = new zp_peer_group();
  if (cudaMalloc(&g->flags, sizeof(zp::PeerFlags) * n) != cudaSuccess ||
      cudaMemset(g->flags, 0, sizeof(zp::PeerFlags) * n) != cudaSuccess) {
    delete g;
    return 5;
  }
  g->base = static_cast<char*>(base);
  g->arena = arena_bytes;
  g->pv.n = n;
  g->pv.rank = 0;
  for (int j = 0; j < n; ++j) {
    g->pv.base[j] = g->base + arena_bytes * j;
    g->pv.flags[j] = g->flags + j;
  }
  *out = g;
  return 0;
}

extern "C" int zp_peer_group_destroy(zp_peer_group* g) {
  if (!g) return 0;
  cudaFree(g->flags);
  delete g;
  return 0;
}

static int peer_rc(cudaError_t e) { return e == cudaSuccess ? 0 : (e == cudaErrorInvalidValue ? 1 : 5); }

template <class T>
static T* at(const zp_peer_group* g, int64_t off) {  // rank 0's buffer at `off` (nullptr if off < 0)
  return off < 0 ? nullptr : reinterpret_cast<T*>(g->base + off);
}

extern "C" int zp_peer_rs_accumulate(zp_peer_group* g, int64_t src_off, int64_t len, int64_t acc_off,
                                     int32_t overwrite, uint32_t epoch, int32_t ctas, void* stream) {
  if (!g || acc_off < 0) return 1;
  zp::PeerEmu emu;
  emu.g = 1;  // set to the per-rank grid by the launcher
  emu.stride = g->arena;
  emu.shard = len;
  return peer_rc(zp::peer_rs_accumulate(g->pv, src_off, 0, at<float>(g, acc_off), len, overwrite != 0, epoch, ctas,
                                        static_cast<cudaStream_t>(stream), emu));
}

extern "C" int zp_peer_rs_adam_ag(zp_peer_group* g, int64_t src_off, int32_t src_f32, int64_t len, int64_t acc_off,
                                  int64_t p32_off, int64_t m_off, int64_t v_off, int64_t p16_off, int64_t gout_off,
                                  const zp_adam_params* ap, uint32_t epoch, int32_t ctas, void* stream) {
  if (!g || !ap || p32_off < 0 || m_off < 0 || v_off < 0) return 1;
  zp::AdamParams a;
  a.lr = ap->lr; a.beta1 = ap->beta1; a.beta2 = ap->beta2; a.eps = ap->eps; a.weight_decay = ap->weight_decay;
  a.bc1 = ap->bc1; a.bc2 = ap->bc2;
  zp::PeerEmu emu;
  emu.g = 1;
  emu.stride = g->arena;
  emu.shard = len;
  return peer_rc(zp::peer_rs_adam_ag(g->pv, src_off, src_f32 != 0, 0, at<float>(g, acc_off), at<float>(g, p32_off),
                                     at<float>(g, m_off), at<float>(g, v_off), p16_off, at<float>(g, gout_off), len, a,
                                     epoch, ctas, static_cast<cudaStream_t>(stream), emu));
}

extern "C" int zp_peer_all_gather(zp_peer_group* g, int64_t shard_src_off, int64_t dst_off, int64_t len,
                                  uint32_t epoch, int32_t ctas, void* stream) {
  if (!g || dst_off < 0) return 1;
  zp::PeerEmu emu;
  emu.g = 1;
  emu.stride = g->arena;
  return peer_rc(zp::peer_all_gather(g->pv, shard_src_off, at<zp::bf16>(g, dst_off), len, epoch, ctas,
                                     static_cast<cudaStream_t>(stream), emu));
}

extern "C" int zp_attention_bwd_hd(const void* qkv, const void* out, const void* dout, const float* lse,
                                   float* dvec, float* dq32, void* dqkv, int64_t batch, int32_t seq,
                                   int32_t heads, int32_t head_dim, int32_t max_ctas, void* stream) {
  const cudaError_t e = zp::attention_bwd(static_cast<const zp::bf16*>(qkv), static_cast<const zp::bf16*>(out),
                                          static_cast<const zp::bf16*>(dout), lse, dvec, dq32,
                                          static_cast<zp::bf16*>(dqkv), batch, seq, heads, max_ctas,
                                          static_cast<cudaStream_t>(stream), head_dim);
  return e == cudaSuccess ? 0 : (e == cudaErrorInvalidValue ? 1 : 5);
}
