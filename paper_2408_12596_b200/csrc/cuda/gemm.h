// Dense bf16 GEMM on sm_100a tensor cores (tcgen05 + TMEM + TMA), host-side interface.
//
//   C[z][m, n] = epilogue( alpha * sum_k A[z][m, k] * B[z][n, k] )
//
// A is logically [M, K], B is logically [N, K] (i.e. the product is A * B^T).
// Each operand is stored either K-major (element (r, k) at ptr[r*ld + k]) or
// MN-major (element (r, k) at ptr[k*ld + r]); this covers the forward
// (X W^T), data-gradient (dY W) and weight-gradient (dY^T X) products of a
// linear layer without any transpose pass. A batch index z = z1 + nb1*z2 maps
// to element offsets z1*bs1 + z2*bs2, so per-(sample, head) attention GEMMs
// read head slices of the fused QKV activation in place.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace zp {

enum GemmMajor : int { kKMajor = 0, kMNMajor = 1 };

enum GemmEpilogue : int {
  kEpiStoreBf16 = 0,      // C(bf16) = alpha*acc
  kEpiStoreF32 = 1,       // C(f32)  = alpha*acc
  kEpiAccumF32 = 2,       // C(f32) += alpha*acc
  kEpiBiasBf16 = 3,       // C(bf16) = acc + bias[n]
  kEpiBiasResidBf16 = 4,  // C(bf16) = acc + bias[n] + R[m, n]   (R may alias C)
  kEpiBiasGeluBf16 = 5,   // u = acc + bias[n]; C(bf16) = gelu(u), aux_out(bf16) = gelu'(u)
  kEpiGeluBwdBf16 = 6,    // C(bf16) = acc * aux[m, n]   (aux = gelu'(u) from the forward)
  kEpiAtomicF32 = 7,      // C(f32) += alpha*acc with fp32 vector atomics (split-K partials)
  kEpiSwiGluBf16 = 8,     // C(bf16) = acc (gate/up interleaved in 32-column blocks);
                          // aux_out[m, j] (bf16, ld = ldc / 2) = silu(gate_j) * up_j
  kEpiRopeBf16 = 9,       // C(bf16) = acc, columns [0, rope_cols) rotated (rotate-half pairs
                          // (j, j + dh/2) of every head of rope_dh) by position m % rope_seq
  kEpiSwiGluBwdBf16 = 10, // acc = dh [M, N] (never stored): with aux = u [M, 2N] (gate/up
                          // interleaved in 32-column blocks, as kEpiSwiGluBf16 wrote it), C [M, 2N]
                          // (same layout, row stride ldc) = (dgate, dup) of h = silu(gate) * up
  kEpiDvecBf16 = 11,      // C(bf16) = acc (dO of attention); with aux = O (same layout, heads of
                          // 128 columns): dvec[(m / dvec_seq * heads + head) * dvec_seq + m % dvec_seq]
                          // = sum over the head of bf16(C) * O; zero32 (fp32, [M, N], ld ldc) zeroed
};

enum GemmCausal : int {
  kCausalNone = 0,
  kCausalSkipUpper = 1,  // skip tiles whose first column is past the tile's last row
  kCausalKUpper = 2,     // reduce only over k <= last row of the tile (A is lower-triangular)
  kCausalKLower = 3,     // reduce only over k >= first row of the tile (A is upper-triangular)
};

struct GemmOperand {
  const void* ptr = nullptr;  // bf16
  int major = kKMajor;
  int64_t ld = 0;             // elements between stored rows
  int64_t bs1 = 0, bs2 = 0;   // batch strides in elements
};

struct GemmArgs {
  int M = 0, N = 0, K = 0;
  int nb1 = 1, nb2 = 1;
  GemmOperand a, b;
  void* c = nullptr;
  int64_t ldc = 0, cs1 = 0, cs2 = 0;  // C row stride / batch strides (elements)
  float alpha = 1.0f;
  int epilogue = kEpiStoreBf16;
  int causal = kCausalNone;
  const void* bias = nullptr;  // bf16 [N]; may be null (no bias)
  const void* aux = nullptr;   // bf16, same layout as C (residual R or pre-activation U)
  void* aux_out = nullptr;     // bf16, same layout as C (gelu'(u) written by kEpiBiasGeluBf16)
  int max_ctas = 0;            // SM budget cap (0 = all SMs)
  int split_k = 1;             // >1: K range split across CTAs; -1: auto; requires kEpiAtomicF32
  float* colsum = nullptr;     // bf16 epilogues: += column sums of the output (fp32 [N]; bias grad)
  // kEpiRopeBf16: (cos, sin) table float2 [rope_seq][rope_dh / 2] (kernels.h rope_table)
  const void* rope_tab = nullptr;
  int rope_seq = 0, rope_dh = 0, rope_cols = 0;
  // kEpiDvecBf16: the attention backward's D vector and its fp32 dQ workspace to clear
  float* dvec = nullptr;
  float* zero32 = nullptr;
  int dvec_seq = 0;
};

// Returns cudaSuccess or the launch/encode error.
cudaError_t gemm(const GemmArgs& args, cudaStream_t stream);

}  // namespace zp
