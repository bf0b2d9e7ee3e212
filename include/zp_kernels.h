/*
 * zp_kernels.h — C ABI of the individual sm_100a kernels of the heterogeneous-ZeRO step.
 *
 * These entry points are what the step driver (zp_runtime.h) launches; they are exported
 * separately so parity tests can drive each kernel on device buffers. All pointers are
 * device pointers; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Every function returns 0 on success or a ZP_E* code (zp_host.h) and never throws.
 *
 * Reference counterpart: none of these exist in the reference, which models the whole
 * device step as the closed form `compute_fixed + compute_per_batch * b`
 * (proj/core/src/hardware.cpp:160-167) and `optimizer_time` (hardware.cpp:168).
 */
#ifndef ZP_KERNELS_H_
#define ZP_KERNELS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GEMM: C[z][m,n] = epilogue(alpha * sum_k A[z][m,k] * B[z][n,k]), bf16 in, fp32 accumulate.
 * major: 0 = K-major (elem (r,k) at ptr[r*ld+k]), 1 = MN-major (elem (r,k) at ptr[k*ld+r]).
 * epilogue: 0 store bf16, 1 store f32, 2 accumulate f32, 3 +bias bf16, 4 +bias+residual bf16,
 *           5 +bias then GELU bf16 (GELU'(pre-activation) to aux_out), 6 times aux (= GELU') bf16,
 *           7 fp32 atomic add (split-K partial sums),
 *           8 bf16 store + SwiGLU: aux_out[m, j] = silu(gate_j) * up_j, gate/up interleaved in
 *             32-column blocks of C, aux_out row stride ldc / 2 (N % 64 == 0).
 * causal:   0 none, 1 skip tiles above the diagonal, 2 k <= tile last row, 3 k >= tile first row.
 */
typedef struct zp_gemm_desc {
  int32_t M, N, K, nb1, nb2;
  const void* a; int32_t a_major; int64_t lda, a_bs1, a_bs2;
  const void* b; int32_t b_major; int64_t ldb, b_bs1, b_bs2;
  void* c; int64_t ldc, c_bs1, c_bs2;
  float alpha;
  int32_t epilogue;
  int32_t causal;
  const void* bias;
  const void* aux;
  void* aux_out;
  int32_t max_ctas;
  int32_t split_k;  /* > 1 splits the K range across CTAs, -1 picks the split for full waves; needs epilogue 7 (fp32 atomic add) */
  float* colsum;    /* optional, bf16 epilogues of unbatched GEMMs: colsum[n] += sum over m of C[m, n]
                       (fp32 [N], caller-zeroed; the bias gradient when C is an output gradient) */
} zp_gemm_desc;

int zp_gemm(const zp_gemm_desc* d, void* stream);

/* Fused causal attention, head_dim 64 (tcgen05; scores never reach HBM).
 * qkv [batch*seq, 3*heads*64] bf16 (Q | K | V); out [batch*seq, heads*64] bf16;
 * lse [batch*heads*seq] fp32 (natural log of the row sum of exp(scores / 8)). */
int zp_attention_fwd(const void* qkv, void* out, float* lse, int64_t batch, int32_t seq, int32_t heads,
                     int32_t max_ctas, void* stream);
/* Same with an explicit head_dim (64 or 128; qkv heads of head_dim contiguous, lse scale
 * 1/sqrt(head_dim)). head_dim 128: two 128-query tiles per CTA sharing every K/V tile. */
int zp_attention_fwd_hd(const void* qkv, void* out, float* lse, int64_t batch, int32_t seq, int32_t heads,
                        int32_t head_dim, int32_t max_ctas, void* stream);
/* Gradients of the above: dout [batch*seq, heads*64] -> dqkv [batch*seq, 3*heads*64] bf16.
 * Workspaces: dvec [batch*heads*seq] fp32, dq32 [batch*seq, heads*64] fp32. */
int zp_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* dvec,
                     float* dq32, void* dqkv, int64_t batch, int32_t seq, int32_t heads, int32_t max_ctas,
                     void* stream);
/* Same with an explicit head_dim (64 or 128; dq32 [batch*seq, heads*head_dim]). */
int zp_attention_bwd_hd(const void* qkv, const void* out, const void* dout, const float* lse, float* dvec,
                        float* dq32, void* dqkv, int64_t batch, int32_t seq, int32_t heads, int32_t head_dim,
                        int32_t max_ctas, void* stream);

/* LayerNorm (rms = 0) / RMSNorm (rms = 1) backward over `rows` rows of h (a multiple of 256)
 * columns, bf16 in / out, given the forward's per-row mean and rstd (fp32; RMS: mean = 0):
 * dx = dres + rstd * (gamma * dy - mean(gamma * dy) - xhat * mean(gamma * dy * xhat)), the
 * mean(gamma * dy) term only for LayerNorm; dres optional (NULL = 0). Column partials (fp32,
 * summed over the row chunk of each of *nparts CTAs): part[k*h + c] = dgamma, part[(*nparts + k)*h
 * + c] = dbeta (LayerNorm), colsum_part[k*h + c] (optional) = sum of dx. Capacities in floats:
 * part >= 2 * 592 * h, colsum_part >= 592 * h (592 = 4 x 148 CTAs, the largest split). */
int zp_norm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const void* gamma,
                const void* dres, void* dx, float* part, int64_t part_capacity, float* colsum_part,
                int64_t colsum_capacity, int32_t* nparts, int64_t rows, int32_t h, int32_t rms, int32_t max_ctas,
                void* stream);

/* ---- NVLink peer-memory collectives (csrc/cuda/peer.cu), emulated on ONE device for parity.
 * A peer group is n "rank arenas": n equal regions of `arena_bytes` starting at `base` (device
 * memory), plus n flag blocks the group allocates (zeroed). Every call runs ALL n rank instances
 * of the kernel in ONE cooperative launch (blocks [r*G, (r+1)*G) are rank r), so instances that
 * wait on one another through the epoch-stamped flags are co-resident by construction; epochs
 * must increase by one per call. Every buffer is given as a byte offset inside the arenas, the
 * same for every rank (rank r's lives at base + r*arena_bytes + offset), exactly as the runtime
 * lays them out. Rank r owns shard r: elements [r*len, (r+1)*len) of the full-size buffers.
 * Reference counterpart: none (the reference models these collectives as
 * collective_time(param_count * bytes_per_param), proj/core/src/comm.cpp:88-99). */
typedef struct zp_peer_group zp_peer_group;
typedef struct zp_adam_params {
  float lr, beta1, beta2, eps, weight_decay;
  float bc1, bc2; /* 1 - beta^t */
} zp_adam_params;
int zp_peer_group_create(int32_t n, void* base, int64_t arena_bytes, zp_peer_group** out);
int zp_peer_group_destroy(zp_peer_group* g);
/* rank r: acc_r[i] = (overwrite ? 0 : acc_r[i]) + sum_{j=0..n-1} bf16 src_j[r*len + i] (fp32, rank
 * order); src: bf16 [n*len] at src_off; acc: fp32 [len] at acc_off */
int zp_peer_rs_accumulate(zp_peer_group* g, int64_t src_off, int64_t len, int64_t acc_off, int32_t overwrite,
                          uint32_t epoch, int32_t ctas, void* stream);
/* rank r: grad[i] = (acc_off >= 0 ? acc_r[i] : 0) + sum_j src_j[r*len + i] (bf16, or fp32 when
 * src_f32); AdamW on (p32, m, v)_r[i] (fp32 [len] each); bf16(p32_r[i]) pushed to element
 * r*len + i of EVERY rank's p16 [n*len]; gout_r (fp32 [len], optional: gout_off >= 0) gets grad */
int zp_peer_rs_adam_ag(zp_peer_group* g, int64_t src_off, int32_t src_f32, int64_t len, int64_t acc_off,
                       int64_t p32_off, int64_t m_off, int64_t v_off, int64_t p16_off, int64_t gout_off,
                       const zp_adam_params* ap, uint32_t epoch, int32_t ctas, void* stream);
/* rank r: dst_r[j*len + e] = src_j[e] (bf16 [len] at shard_src_off in every arena; dst [n*len]) */
int zp_peer_all_gather(zp_peer_group* g, int64_t shard_src_off, int64_t dst_off, int64_t len, uint32_t epoch,
                       int32_t ctas, void* stream);

/* On-device synthetic token rows (the loader's synthetic data, zp_runtime_load_tokens with
 * from_host = 0): out[i * seq_plus1 + t] for samples j = first + i, i < count, is a fixed function
 * of (seed, iteration, j, t): splitmix64 finaliser chain, modulo vocab. A sample's row does not
 * depend on which rank or slice loads it. out: device int32 [count * seq_plus1]. */
int zp_synth_tokens(int32_t* out, int64_t first, int64_t count, int32_t seq_plus1, int32_t vocab, uint64_t seed,
                    uint64_t iteration, void* stream);

/* Number of kernels launched by this library since load (all entry points). */
int64_t zp_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* ZP_KERNELS_H_ */
