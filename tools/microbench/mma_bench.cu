// tcgen05.mma throughput microbenchmark (one CTA per SM, one issuing thread, descriptors
// precomputed, 8 MMAs per unrolled iteration): cycles per MMA instruction per operand shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I include tools/microbench/mma_bench.cu -o /tmp/mma_bench
#include <cstdio>
#include "../../paper_2408_12596_b200/csrc/cuda/ptx.cuh"

using namespace zp;
constexpr int kTile = 128 * 64 * 2;

__device__ __forceinline__ uint64_t kdesc(uint32_t base, int k16) { return ptx::smem_desc_sw128(base + k16 * 32, 16, 1024); }
__device__ __forceinline__ uint64_t kdesc2(uint32_t base, int k16) {
  return ptx::smem_desc_sw128(base + (k16 >> 2) * kTile + (k16 & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int k16) { return ptx::smem_desc_sw128(base + k16 * 2048, kTile, 1024); }

template <int MODE, int M, int N>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(sm), b = ptx::smem_u32(sm + 4 * kTile);
    constexpr uint32_t id = ptx::idesc_bf16_f32(M, N, MODE == 1 ? 1 : 0, (MODE == 1 || MODE == 2 || MODE == 3) ? 1 : 0);
    uint64_t da[8], db[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      da[k] = MODE == 1 ? mndesc(a, k) : (MODE == 0 ? kdesc(a, k & 3) : kdesc2(a, k));
      db[k] = (MODE == 1 || MODE == 2 || MODE == 3) ? mndesc(b, k) : kdesc(b, k & 3);
    }
    const long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 3)
          ptx::umma_bf16_ts(tmem + 256, tmem + 128 + 8 * k, db[k], id, 1);
        else
          ptx::umma_bf16(tmem, da[k], db[k], id, 1);
      }
    }
    ptx::umma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

unsigned long long* d;
template <int MODE, int M, int N>
void run(const char* name) {
  auto k = bench<MODE, M, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kTile + 1024);
  const int iters = 8192;
  for (int rep = 0; rep < 2; ++rep) k<<<148, 128, 8 * kTile + 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %7.1f clk/MMA  %6.0f MAC/clk/SM  (%s)\n", name, double(c) / iters, double(M) * N * 16 * iters / c,
         cudaGetErrorString(e));
}

int main() {
  cudaMalloc(&d, 64);
  run<0, 128, 256>("128x256x16 K/K");
  run<0, 128, 128>("128x128x16 K/K");
  run<0, 128, 64>("128x64x16 K/K");
  run<0, 128, 32>("128x32x16 K/K");
  run<1, 128, 64>("128x64x16 MN/MN");
  run<2, 128, 64>("128x64x16 K(2blk)/MN");
  run<3, 128, 64>("128x64x16 TMEM/MN");
  run<2, 128, 128>("128x128x16 K(2blk)/MN");
  run<0, 64, 128>("64x128x16 K/K");
  run<0, 64, 256>("64x256x16 K/K");
  return 0;
}
