// NVLink peer-memory collectives (see peer.h): pull reduce-scatter, fused
// reduce-scatter + AdamW + push all-gather, and pull all-gather.
#include "peer.h"

#include <cuda_bf16.h>

namespace zp {
namespace {

constexpr int kThreads = 256;
constexpr unsigned long long kTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s, then trap

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin until flags[j] has reached `epoch` for every rank j (serial-number comparison).
__device__ void wait_all(const uint32_t* flags, int n, uint32_t epoch) {
  const uint64_t t0 = global_ns();
  for (int j = 0; j < n; ++j) {
    while (int32_t(ld_acquire_sys(flags + j) - epoch) < 0) {
      __nanosleep(100);
      if (global_ns() - t0 > kTimeoutNs) __trap();  // a peer never arrived: fail, do not hang
    }
  }
}

// Entry: CTA 0 announces "my inputs are final" to every rank; every CTA waits for all ranks.
__device__ void entry_barrier(const PeerView& pv, uint32_t epoch, int blk) {
  if (threadIdx.x == 0) {
    if (blk == 0)
      for (int j = 0; j < pv.n; ++j) st_release_sys(&pv.flags[j]->ready[pv.rank], epoch);
    wait_all(pv.flags[pv.rank]->ready, pv.n, epoch);
  }
  __syncthreads();
}

// Exit: the last CTA of this rank to finish tells every rank "done with your buffers" and waits
// until every rank said the same, so the kernel completes only when all peers finished.
__device__ void exit_barrier(const PeerView& pv, uint32_t epoch, int nblk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t old = atomicInc(&pv.flags[pv.rank]->ctr, nblk - 1);
    if (old == nblk - 1) {
      __threadfence_system();
      for (int j = 0; j < pv.n; ++j) st_release_sys(&pv.flags[j]->done[pv.rank], epoch);
      wait_all(pv.flags[pv.rank]->done, pv.n, epoch);
    }
  }
}

// This block's rank instance: (block index, block count) within the rank's grid; in an emulated
// launch also the rank itself and its pointer / shard offsets.
struct Blk {
  int blk, nblk, rank;
};
__device__ __forceinline__ Blk resolve(const PeerEmu& emu, int rank) {
  if (emu.g == 0) return {int(blockIdx.x), int(gridDim.x), rank};
  return {int(blockIdx.x) % emu.g, emu.g, int(blockIdx.x) / emu.g};
}
template <class T>
__device__ __forceinline__ T* rank_ptr(T* p, const PeerEmu& emu, int rank) {
  return (emu.g == 0 || p == nullptr) ? p : reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(p) + emu.stride * rank);
}

__device__ __forceinline__ void add_bf16x8(float (&a)[8], const uint4& u) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    a[2 * k] += f.x;
    a[2 * k + 1] += f.y;
  }
}

// Sum over ranks (fixed order 0..n-1, identical on every rank) of 8 gradient elements.
template <bool F32>
__device__ __forceinline__ void pull_sum8(const PeerView& pv, int64_t src_off, int64_t e, float (&g)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) g[k] = 0.f;
  for (int j = 0; j < pv.n; ++j) {
    if constexpr (F32) {
      const float4* p = reinterpret_cast<const float4*>(pv.base[j] + src_off) + e / 4;
      const float4 a = p[0], b = p[1];
      g[0] += a.x; g[1] += a.y; g[2] += a.z; g[3] += a.w;
      g[4] += b.x; g[5] += b.y; g[6] += b.z; g[7] += b.w;
    } else {
      const uint4 u = *(reinterpret_cast<const uint4*>(pv.base[j] + src_off) + e / 8);
      add_bf16x8(g, u);
    }
  }
}

__global__ void __launch_bounds__(kThreads) peer_rs_acc_k(PeerView pv, int64_t src_off, int64_t shard_off,
                                                          float* __restrict__ acc, int64_t len, int overwrite,
                                                          uint32_t epoch, PeerEmu emu) {
  const Blk B = resolve(emu, pv.rank);
  pv.rank = B.rank;
  acc = rank_ptr(acc, emu, B.rank);
  shard_off += emu.shard * B.rank;
  entry_barrier(pv, epoch, B.blk);
  const int64_t n8 = len / 8;
  const int64_t step = int64_t(B.nblk) * kThreads;
  int64_t i0 = B.blk * int64_t(kThreads) + threadIdx.x;
  // two items per thread: 2n remote loads in flight before the sums (same per-element order)
  for (; i0 + step < n8; i0 += 2 * step) {
    float g[2][8];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int k = 0; k < 8; ++k) g[t][k] = 0.f;
#pragma unroll 8
    for (int j = 0; j < pv.n; ++j) {
      const uint4* p = reinterpret_cast<const uint4*>(pv.base[j] + src_off) + shard_off / 8;
      const uint4 u0 = p[i0], u1 = p[i0 + step];
      add_bf16x8(g[0], u0);
      add_bf16x8(g[1], u1);
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      float4* a = reinterpret_cast<float4*>(acc) + 2 * (i0 + t * step);
      if (!overwrite) {
        const float4 x = a[0], y = a[1];
        g[t][0] += x.x; g[t][1] += x.y; g[t][2] += x.z; g[t][3] += x.w;
        g[t][4] += y.x; g[t][5] += y.y; g[t][6] += y.z; g[t][7] += y.w;
      }
      a[0] = make_float4(g[t][0], g[t][1], g[t][2], g[t][3]);
      a[1] = make_float4(g[t][4], g[t][5], g[t][6], g[t][7]);
    }
  }
  for (int64_t i = i0; i < n8; i += step) {
    float g[8];
    pull_sum8<false>(pv, src_off, shard_off + i * 8, g);
    float4* a = reinterpret_cast<float4*>(acc) + 2 * i;
    if (!overwrite) {
      const float4 x = a[0], y = a[1];
      g[0] += x.x; g[1] += x.y; g[2] += x.z; g[3] += x.w;
      g[4] += y.x; g[5] += y.y; g[6] += y.z; g[7] += y.w;
    }
    a[0] = make_float4(g[0], g[1], g[2], g[3]);
    a[1] = make_float4(g[4], g[5], g[6], g[7]);
  }
  exit_barrier(pv, epoch, B.nblk);
}

template <bool F32>
__global__ void __launch_bounds__(kThreads) peer_rs_adam_ag_k(PeerView pv, int64_t src_off, int64_t shard_off,
                                                              const float* __restrict__ acc,
                                                              float* __restrict__ p32, float* __restrict__ m,
                                                              float* __restrict__ v, int64_t p16_off,
                                                              float* __restrict__ gout, int64_t len,
                                                              AdamParams ap, uint32_t epoch, PeerEmu emu) {
  const Blk B = resolve(emu, pv.rank);
  pv.rank = B.rank;
  acc = rank_ptr(acc, emu, B.rank);
  p32 = rank_ptr(p32, emu, B.rank);
  m = rank_ptr(m, emu, B.rank);
  v = rank_ptr(v, emu, B.rank);
  gout = rank_ptr(gout, emu, B.rank);
  shard_off += emu.shard * B.rank;
  entry_barrier(pv, epoch, B.blk);
  const float inv_bc1 = 1.0f / ap.bc1;
  const float inv_sqrt_bc2 = rsqrtf(ap.bc2);
  const int64_t n8 = len / 8;
  for (int64_t i = B.blk * int64_t(kThreads) + threadIdx.x; i < n8; i += int64_t(B.nblk) * kThreads) {
    float g[8];
    pull_sum8<F32>(pv, src_off, shard_off + i * 8, g);
    if (acc) {
      const float4 x = reinterpret_cast<const float4*>(acc)[2 * i], y = reinterpret_cast<const float4*>(acc)[2 * i + 1];
      g[0] += x.x; g[1] += x.y; g[2] += x.z; g[3] += x.w;
      g[4] += y.x; g[5] += y.y; g[6] += y.z; g[7] += y.w;
    }
    if (gout) {
      reinterpret_cast<float4*>(gout)[2 * i] = make_float4(g[0], g[1], g[2], g[3]);
      reinterpret_cast<float4*>(gout)[2 * i + 1] = make_float4(g[4], g[5], g[6], g[7]);
    }
    float P[8], M[8], V[8];
    *reinterpret_cast<float4*>(P) = reinterpret_cast<const float4*>(p32)[2 * i];
    *reinterpret_cast<float4*>(P + 4) = reinterpret_cast<const float4*>(p32)[2 * i + 1];
    *reinterpret_cast<float4*>(M) = reinterpret_cast<const float4*>(m)[2 * i];
    *reinterpret_cast<float4*>(M + 4) = reinterpret_cast<const float4*>(m)[2 * i + 1];
    *reinterpret_cast<float4*>(V) = reinterpret_cast<const float4*>(v)[2 * i];
    *reinterpret_cast<float4*>(V + 4) = reinterpret_cast<const float4*>(v)[2 * i + 1];
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // same arithmetic as adam_k (kernels.cu)
      M[k] = ap.beta1 * M[k] + (1.f - ap.beta1) * g[k];
      V[k] = ap.beta2 * V[k] + (1.f - ap.beta2) * g[k] * g[k];
      const float denom = sqrtf(V[k]) * inv_sqrt_bc2 + ap.eps;
      P[k] -= ap.lr * ((M[k] * inv_bc1) / denom + ap.weight_decay * P[k]);
    }
    reinterpret_cast<float4*>(p32)[2 * i] = *reinterpret_cast<float4*>(P);
    reinterpret_cast<float4*>(p32)[2 * i + 1] = *reinterpret_cast<float4*>(P + 4);
    reinterpret_cast<float4*>(m)[2 * i] = *reinterpret_cast<float4*>(M);
    reinterpret_cast<float4*>(m)[2 * i + 1] = *reinterpret_cast<float4*>(M + 4);
    reinterpret_cast<float4*>(v)[2 * i] = *reinterpret_cast<float4*>(V);
    reinterpret_cast<float4*>(v)[2 * i + 1] = *reinterpret_cast<float4*>(V + 4);
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) oh[k] = __floats2bfloat162_rn(P[2 * k], P[2 * k + 1]);
    for (int j = 0; j < pv.n; ++j)  // push the new parameters to every rank (the all-gather)
      *(reinterpret_cast<uint4*>(pv.base[j] + p16_off) + (shard_off / 8 + i)) = o;
  }
  exit_barrier(pv, epoch, B.nblk);
}

__global__ void __launch_bounds__(kThreads) peer_ag_k(PeerView pv, int64_t src_off, bf16* __restrict__ dst,
                                                      int64_t len, uint32_t epoch, PeerEmu emu) {
  const Blk B = resolve(emu, pv.rank);
  pv.rank = B.rank;
  dst = rank_ptr(dst, emu, B.rank);
  entry_barrier(pv, epoch, B.blk);
  const int64_t n8 = len / 8, total8 = n8 * pv.n;
  const int64_t step = int64_t(B.nblk) * kThreads;
  int64_t i = B.blk * int64_t(kThreads) + threadIdx.x;
  // Item i is element e of the c-th shard in this rank's visiting order, which starts at the next
  // rank: at any moment every GPU is read by one peer instead of all ranks reading rank 0 first.
  // Four remote 16-byte loads in flight per thread before their stores (NVLink latency).
  for (; i + 3 * step < total8; i += 4 * step) {
    uint4 u[4];
    int64_t d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t ii = i + k * step;
      const int c = int(ii / n8);
      const int64_t e = ii - int64_t(c) * n8;
      const int j = (c + pv.rank + 1) % pv.n;
      u[k] = *(reinterpret_cast<const uint4*>(pv.base[j] + src_off) + e);
      d[k] = int64_t(j) * n8 + e;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) reinterpret_cast<uint4*>(dst)[d[k]] = u[k];
  }
  for (; i < total8; i += step) {
    const int c = int(i / n8);
    const int64_t e = i - int64_t(c) * n8;
    const int j = (c + pv.rank + 1) % pv.n;
    reinterpret_cast<uint4*>(dst)[int64_t(j) * n8 + e] = *(reinterpret_cast<const uint4*>(pv.base[j] + src_off) + e);
  }
  exit_barrier(pv, epoch, B.nblk);
}

int grid(int64_t items, int ctas) {
  const int64_t want = (items + kThreads - 1) / kThreads;
  const int64_t cap = int64_t(ctas) * 4;
  return int(want < 1 ? 1 : (want < cap ? want : cap));
}

// One launch per rank, or (emu.g > 0) one cooperative launch of every rank's instance.
template <class K, class... Args>
cudaError_t launch(K kernel, int g, const PeerView& pv, const PeerEmu& emu, cudaStream_t s, Args... args) {
  if (emu.g == 0) {
    kernel<<<g, kThreads, 0, s>>>(args..., emu);
    note_launch();
    return cudaGetLastError();
  }
  PeerEmu e = emu;
  e.g = g;
  void* params[] = {&args..., &e};
  const cudaError_t r = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(g * pv.n),
                                                    dim3(kThreads), params, 0, s);
  note_launch();
  return r;
}

}  // namespace

cudaError_t peer_rs_accumulate(const PeerView& pv, int64_t src_off, int64_t shard_off, float* acc,
                               int64_t len, bool overwrite, uint32_t epoch, int ctas, cudaStream_t s,
                               const PeerEmu& emu) {
  if (len % 8 || shard_off % 8 || emu.shard % 8) return cudaErrorInvalidValue;
  return launch(peer_rs_acc_k, grid(len / 8, ctas), pv, emu, s, pv, src_off, shard_off, acc, len,
                overwrite ? 1 : 0, epoch);
}

cudaError_t peer_rs_adam_ag(const PeerView& pv, int64_t src_off, bool src_f32, int64_t shard_off,
                            const float* acc, float* p32, float* m, float* v, int64_t p16_off,
                            float* gout, int64_t len, const AdamParams& ap, uint32_t epoch, int ctas,
                            cudaStream_t s, const PeerEmu& emu) {
  if (len % 8 || shard_off % 8 || emu.shard % 8) return cudaErrorInvalidValue;
  if (src_f32)
    return launch(peer_rs_adam_ag_k<true>, grid(len / 8, ctas), pv, emu, s, pv, src_off, shard_off, acc, p32, m,
                  v, p16_off, gout, len, ap, epoch);
  return launch(peer_rs_adam_ag_k<false>, grid(len / 8, ctas), pv, emu, s, pv, src_off, shard_off, acc, p32, m, v,
                p16_off, gout, len, ap, epoch);
}

cudaError_t peer_all_gather(const PeerView& pv, int64_t shard_src_off, bf16* dst, int64_t len,
                            uint32_t epoch, int ctas, cudaStream_t s, const PeerEmu& emu) {
  if (len % 8) return cudaErrorInvalidValue;
  return launch(peer_ag_k, grid(len / 8 * pv.n, ctas), pv, emu, s, pv, shard_src_off, dst, len, epoch);
}

}  // namespace zp
