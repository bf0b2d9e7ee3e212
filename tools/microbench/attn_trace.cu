// Pipeline timeline of the head_dim-128 attention backward: CTA 0 stamps clock64 at every
// barrier hand-off of its first key tile (ZP_ATTN_TRACE hooks in attention.cu), and this driver
// prints per-query-tile event times relative to the first dP^T issue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -DZP_ATTN_TRACE -lineinfo \
//     tools/microbench/attn_trace.cu paper_2408_12596_b200/csrc/cuda/kernels.cu -lcuda -o /tmp/attn_trace
// Usage: attn_trace [batch 2] [seq 4096] [heads 32] [dbg 0] [fwd]   (dbg: ZP_ATTN_DBG bits; "fwd":
// time and trace the forward instead)
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../paper_2408_12596_b200/csrc/cuda/attention.cu"

namespace {
__global__ void fill_k(zp::bf16* p, int64_t n, uint32_t seed, float amp) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x = uint32_t(i) * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = __float2bfloat16(amp * (float(x & 0xffff) / 32768.f - 1.f));
  }
}
}  // namespace

int main(int argc, char** argv) {
  const int64_t batch = argc > 1 ? atoi(argv[1]) : 2;
  const int seq = argc > 2 ? atoi(argv[2]) : 4096;
  const int heads = argc > 3 ? atoi(argv[3]) : 32;
  if (argc > 4) setenv("ZP_ATTN_DBG", argv[4], 1);
  const int h = heads * 128;
  const int64_t T = batch * seq;
  zp::bf16 *qkv, *out, *dout, *dqkv;
  float *lse, *dvec, *dq32;
  cudaMalloc(&qkv, T * 3 * h * 2);
  cudaMalloc(&out, T * h * 2);
  cudaMalloc(&dout, T * h * 2);
  cudaMalloc(&dqkv, T * 3 * h * 2);
  cudaMalloc(&lse, batch * heads * seq * 4);
  cudaMalloc(&dvec, batch * heads * seq * 4);
  cudaMalloc(&dq32, T * h * 4);
  fill_k<<<1184, 256>>>(qkv, T * 3 * h, 1, 1.f);
  fill_k<<<1184, 256>>>(dout, T * h, 2, 0.1f);
  if (zp::attention_fwd(qkv, out, lse, batch, seq, heads, 0, nullptr, 128) != cudaSuccess) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  if (argc > 5 && std::string(argv[5]) == "fwd") {
    float bestf = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      if (zp::attention_fwd(qkv, out, lse, batch, seq, heads, 0, nullptr, 128) != cudaSuccess) return 2;
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < bestf) bestf = ms;
    }
    const double ff = 4.0 * batch * heads * double(seq) * seq * 128 / 2;
    printf("attention fwd d128 b%lld s%d h%d: %.3f ms, %.0f TFLOP/s causal\n", (long long)batch, seq, heads, bestf,
           ff / (bestf * 1e-3) / 1e12);
    unsigned long long tf[16][64];
    cudaMemcpyFromSymbol(tf, zp::g_attn_trace_f, sizeof(tf));
    const char* fn[12] = {"PV0_iss", "S0_iss", "PV1_iss", "S1_iss", "g0_sfull", "g0_max", "g0_exp", "g0_pfull",
                          "g1_sfull", "g1_max", "g1_exp", "g1_pfull"};
    const unsigned long long f0 = tf[1][0];
    printf("tile");
    for (int e = 0; e < 12; ++e) printf(" %9s", fn[e]);
    printf("   period\n");
    for (int i = 0; i < seq / 128 && i < 64; ++i) {
      printf("%4d", i);
      for (int e = 0; e < 12; ++e) printf(" %9lld", (long long)(tf[e][i] - f0));
      printf("   %6lld\n", i ? (long long)(tf[1][i] - tf[1][i - 1]) : 0LL);
    }
    return 0;
  }
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0);
    if (zp::attention_bwd(qkv, out, dout, lse, dvec, dq32, dqkv, batch, seq, heads, 0, nullptr, 128) != cudaSuccess)
      return 2;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  const cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return 3;
  }
  const double flops = 2.5 * 4.0 * batch * heads * double(seq) * seq * 128 / 2;
  printf("attention bwd d128 b%lld s%d h%d: %.3f ms (incl. dvec, memset, cast), %.0f TFLOP/s causal\n",
         (long long)batch, seq, heads, best, flops / (best * 1e-3) / 1e12);
  unsigned long long tr[16][64];
  cudaMemcpyFromSymbol(tr, zp::g_attn_trace, sizeof(tr));
  const char* names[14] = {"dP_iss", "dV_iss", "S_iss", "dK_iss", "dQ_iss", "P_beg", "P_end",
                           "dS_beg", "dS_end", "unused", "dSsm_end", "dQ_rd", "dQ_free", "red_end"};
  const unsigned long long t0 = tr[0][0];
  printf("tile");
  for (int e = 0; e < 14; ++e) printf(" %9s", names[e]);
  printf("   period\n");
  const int ntiles = seq / 128;
  for (int i = 0; i < ntiles && i < 64; ++i) {
    printf("%4d", i);
    for (int e = 0; e < 14; ++e) printf(" %9lld", (long long)(tr[e][i] - t0));
    printf("   %6lld\n", i ? (long long)(tr[0][i] - tr[0][i - 1]) : 0LL);
  }
  return 0;
}
