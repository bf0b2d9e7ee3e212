// Timeline of the attention backward kernel (CTA 0): build with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr -I include \
//        -DZP_ATTN_TRACE tools/debug/attn_trace.cu -o /tmp/attn_trace -lcuda
#include "../../paper_2408_12596_b200/csrc/cuda/attention.cu"

#include <cstdio>
#include <vector>

namespace zp {
void note_launch(int64_t) {}
}

int main() {
  using namespace zp;
  const int b = 16, s = 1024, H = 12, h = H * 64;
  const int64_t T = int64_t(b) * s;
  std::vector<uint16_t> hq(T * 3 * h), hd(T * h);
  uint32_t x = 12345;
  auto rnd = [&]() { x = x * 1664525u + 1013904223u; return uint16_t(0x3f00 | ((x >> 16) & 0x7f)) ^ ((x >> 8) & 0x8000); };
  for (auto& v : hq) v = rnd();
  for (auto& v : hd) v = rnd();
  bf16 *qkv, *out, *dout, *dqkv;
  float *lse, *dvec, *dq32;
  cudaMalloc(&qkv, T * 3 * h * 2); cudaMalloc(&out, T * h * 2); cudaMalloc(&dout, T * h * 2); cudaMalloc(&dqkv, T * 3 * h * 2);
  cudaMalloc(&lse, T * H * 4); cudaMalloc(&dvec, T * H * 4); cudaMalloc(&dq32, T * h * 4);
  cudaMemcpy(qkv, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dout, hd.data(), hd.size() * 2, cudaMemcpyHostToDevice);
  attention_fwd(qkv, out, lse, b, s, H, 132, 0);
#ifdef ZP_TRACE_FWD
  {
    unsigned int zero[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_trace_n, zero, sizeof(zero));
    for (int rep = 0; rep < 3; ++rep) attention_fwd(qkv, out, lse, b, s, H, 132, 0);
  }
#else
  for (int rep = 0; rep < 3; ++rep) {
#ifdef ZP_ATTN_TRACE
    unsigned int zero[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_trace_n, zero, sizeof(zero));
#endif
    cudaError_t eb = attention_bwd(qkv, out, dout, lse, dvec, dq32, dqkv, b, s, H, 132, 0);
    if (eb != cudaSuccess) printf("attention_bwd: %s\n", cudaGetErrorString(eb));
  }
#endif
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
#ifdef ZP_TRACE_FWD
  for (int rep = 0; rep < 0; ++rep) {
#else
  for (int rep = 0; rep < 10; ++rep) {
#endif
    cudaError_t eb = attention_bwd(qkv, out, dout, lse, dvec, dq32, dqkv, b, s, H, 132, 0);
    if (eb != cudaSuccess && rep == 0) printf("attention_bwd (timed): %s\n", cudaGetErrorString(eb));
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("bwd %.4f ms per call\n", ms / 10);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
#ifndef ZP_ATTN_TRACE
  return 0;
#else
  static unsigned long long tr[4][8192];
  unsigned int n[4];
  cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
  cudaMemcpyFromSymbol(n, g_trace_n, sizeof(n));
  unsigned long long t0 = ~0ull;
  for (int r = 0; r < 4; ++r)
    for (unsigned i = 0; i < n[r] && i < 8192; ++i) t0 = std::min(t0, tr[r][i] & ((1ull << 56) - 1));
  const char* names[4] = {"mma", "bld", "dq", "prod"};
  for (int r = 0; r < 4; ++r) {
    printf("== %s (%u events)\n", names[r], n[r]);
    for (unsigned i = 0; i < n[r] && i < 400; ++i)
      printf("%s %d %llu\n", names[r], int(tr[r][i] >> 56), (tr[r][i] & ((1ull << 56) - 1)) - t0);
  }
  return 0;
#endif
}
