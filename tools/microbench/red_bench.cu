// fp32 reduction throughput into global memory (the attention backward's dQ accumulation):
// every CTA adds `tiles` [128 x 128] fp32 tiles into dQ rows with row stride `h`, 4 warps.
//   mode 0: red.global.add.f32, a warp instruction = 32 consecutive floats of one row (128 B)
//   mode 1: red.global.add.v4.f32, a warp instruction = one row's 128 floats (512 B)
//   mode 2: cp.reduce.async.bulk (1-D bulk reduce-add from shared memory, 512 B per row)
// `share`: CTAs per distinct target tile (1 = every CTA its own rows; 9 = nine CTAs hit the same
// rows at the same time, as concurrent key tiles of one head do).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 tools/microbench/red_bench.cu -o /tmp/red_bench
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__global__ void __launch_bounds__(128, 1) red_k(float* dq, int h, int tiles, int share, int mode) {
  __shared__ __align__(128) float stage[4][512];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int slot = blockIdx.x / share;
  for (int i = 0; i < 512; i += 32) stage[warp][i + lane] = 1.f;
  __syncwarp();
  for (int t = 0; t < tiles; ++t) {
    // tile rows: (slot * tiles + t) * 128 .. +127 ; 128 columns starting at 0
    float* base = dq + int64_t(slot * tiles + t) * 128 * h;
    if (mode == 0) {
      // warp w owns columns 32w..32w+31, lane = column, 128 rows
#pragma unroll 8
      for (int r = 0; r < 128; ++r)
        asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(base + int64_t(r) * h + warp * 32 + lane),
                     "f"(1.f) : "memory");
    } else if (mode == 1) {
      // warp w owns rows 32w..32w+31; one row (32 x float4) per instruction
#pragma unroll 4
      for (int r = 0; r < 32; r += 1) {
        float* p = base + int64_t(warp * 32 + r) * h + lane * 4;
        asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f),
                     "f"(1.f), "f"(1.f) : "memory");
      }
    } else {
      if (lane == 0) {
        for (int r = 0; r < 32; ++r) {
          float* p = base + int64_t(warp * 32 + r) * h;
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;" ::"l"(p),
                       "r"(uint32_t(__cvta_generic_to_shared(stage[warp]))) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
    }
  }
  if (mode == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int tiles = argc > 1 ? atoi(argv[1]) : 64;
  const int h = 4096;
  const int grid = 148;
  float* dq;
  const size_t rows = size_t(grid) * tiles * 128;
  cudaMalloc(&dq, rows * h * 4);
  cudaMemset(dq, 0, rows * h * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (int mode = 0; mode < 3; ++mode)
    for (int share : {1, 4, 9}) {
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        red_k<<<grid, 128>>>(dq, h, tiles, share, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
      }
      const double bytes = double(grid) * tiles * 128 * 128 * 4;
      printf("mode %d share %d: %.3f ms  %.0f GB/s reduced  (%.1f B/clk/SM at %d MHz nominal) %s\n", mode, share, best,
             bytes / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / (clk_khz * 1e3) / grid, clk_khz / 1000,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
