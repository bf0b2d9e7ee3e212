// HBM-bound kernels of the GPT training step and of the ZeRO reduce/update path.
// All launchers take the rank's CTA cap (`ctas`, its emulated SM budget) and a stream.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace zp {

using bf16 = __nv_bfloat16;

// Count of kernels this library has launched (bench.py's gpu_launches claim).
void note_launch(int64_t k = 1);
// True the first time it is called on the calling thread's current device for this flag word:
// per-device one-time setup (cudaFuncSetAttribute applies to the current device only, and one
// process may drive several GPUs, e.g. the single-process device-seam backend).
inline bool first_on_device(std::atomic<uint64_t>& flags) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  return !(flags.fetch_or(bit) & bit);
}
int64_t launch_count();

// ---- initialisation / data
void init_normal(float* p32, bf16* p16, int64_t n, float stdv, uint64_t seed, uint64_t offset,
                 int ctas, cudaStream_t s);
void init_const(float* p32, bf16* p16, int64_t n, float value, int ctas, cudaStream_t s);
// tokens[j, t] for sample j of [first, first+count) of iteration `it`: uniform in [0, vocab).
void synth_tokens(int32_t* tokens, int64_t first, int64_t count, int seq_plus1, int vocab,
                  uint64_t seed, uint64_t it, int ctas, cudaStream_t s);

// ---- forward
void embed_fwd(const int32_t* tokens, int seq, const bf16* wte, const bf16* wpe, bf16* x,
               int64_t rows, int h, int ctas, cudaStream_t s);
// LayerNorm, or RMSNorm when b == nullptr (mean written as 0).
cudaError_t layernorm_fwd(const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mean,
                          float* rstd, int64_t rows, int h, int ctas, cudaStream_t s);
// per-row CE on bf16 logits [rows, ldv] (first `vocab` columns valid); overwrites logits with
// dlogits * grad_scale, writes per-row loss.
void cross_entropy_fwd_bwd(bf16* logits, const int32_t* tokens, int seq, int64_t rows, int vocab,
                           int ldv, float grad_scale, float* row_loss, int ctas, cudaStream_t s);

// ---- backward
// dx = dres + LN_bwd(dy); dgamma/dbeta partials per block into part[2][nblk][h] (RMS: dgamma
// only); with cs, column partials of dx itself into cs[nblk][h]; returns nblk (<= 4 * 148).
cudaError_t layernorm_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd,
                          const bf16* g, const bf16* dres, bf16* dx, float* part, int* nblk,
                          int64_t rows, int h, int ctas, cudaStream_t s, bool rms = false,
                          float* cs = nullptr);
// Rotary embedding (rotate-half pairs (i, i + dh/2), any head_dim dh multiple of 16) on the Q and K
// blocks of qkv [T, 3h], in place.
void rope(bf16* qkv, int64_t tokens, int seq, int h, float theta, bool inverse, int ctas, cudaStream_t s,
          int dh = 64);
// The (cos, sin) table it uses: float2 [seq][dh / 2], per device, built on first use (nullptr on
// allocation failure). The QKV GEMM's kEpiRopeBf16 epilogue reads the same table.
const float2* rope_table(int seq, int dh, float theta, cudaStream_t s);
// SwiGLU with gate/up interleaved in 32-column blocks of gu [T, 2f]: out [T, f].
void swiglu_fwd(const bf16* gu, bf16* out, int64_t tokens, int f, int ctas, cudaStream_t s);
void swiglu_bwd(const bf16* gu, const bf16* dh, bf16* dgu, int64_t tokens, int f, int ctas, cudaStream_t s);
void embed_bwd(const int32_t* tokens, int seq, const bf16* dx, float* dwte32, float* dwpe32,
               int64_t rows, int h, int ctas, cudaStream_t s);
// out[n] = sum over rows of X[r, n] (X bf16 [rows, ld]); partial workspace [chunks][N] f32.
// out32 (optional): write / add (acc32) the fp32 sums there instead of bf16 to out
void colsum_bf16(const bf16* X, int64_t rows, int N, int ld, float* work, bf16* out, int ctas,
                 cudaStream_t s, float* out32 = nullptr, bool acc32 = false);
// out[n] = sum over k of part[k, n] (f32), written as bf16.
void sum_partials(const float* part, int nparts, int N, bf16* out, cudaStream_t s, float* out32 = nullptr,
                  bool acc32 = false);
void cast_f32_bf16(const float* in, bf16* out, int64_t n, int ctas, cudaStream_t s);

// ---- ZeRO reduce / update
// acc (=|+=) src; bf16 source.
void accumulate_bf16(float* acc, const bf16* src, int64_t n, bool overwrite, int ctas,
                     cudaStream_t s);
struct AdamParams {
  float lr, beta1, beta2, eps, weight_decay, bc1, bc2;  // bc = 1 - beta^t
};
// g = (acc ? acc : 0) + (g16 ? g16 : 0) + (g32 ? g32 : 0); AdamW on (p32, m, v); p16 = bf16(p32).
void adam_update(float* p32, float* m, float* v, bf16* p16, const float* acc, const bf16* g16,
                 const float* g32, int64_t n, const AdamParams& ap, int ctas, cudaStream_t s);
void reduce_sum_f32(const float* x, int64_t n, float* out, cudaStream_t s);
// dst += src (fp32)
void add_f32(float* dst, const float* src, int64_t n, int ctas, cudaStream_t s);
// acc = (first ? 0 : acc) + sum_j srcs[j] (bf16, j in order, n <= 8; len a multiple of 8)
void reduce_slices(float* acc, const bf16* const* srcs, int n, int64_t len, bool first, int ctas, cudaStream_t s);

}  // namespace zp
