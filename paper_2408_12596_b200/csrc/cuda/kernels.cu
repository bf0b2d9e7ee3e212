// HBM-bound kernels: embedding, LayerNorm, cross-entropy, reductions,
// and the ZeRO accumulate / AdamW update. 16-byte vector accesses, warp-shuffle
// reductions, grid-stride loops capped at the rank's CTA budget.
#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "kernels.h"

#include <mutex>
#include "ptx.cuh"

namespace zp {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void unpack2(uint32_t w, float& lo, float& hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xffff0000u);
}
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  unpack2(u.x, f[0], f[1]);
  unpack2(u.y, f[2], f[3]);
  unpack2(u.z, f[4], f[5]);
  unpack2(u.w, f[6], f[7]);
}
// (lo, hi) -> bf16x2 in one cvt, kept in registers (no address-taken temporaries)
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
}

int grid_for(int64_t work_items, int per_block, int ctas, int per_sm = 4) {
  int64_t g = (work_items + per_block - 1) / per_block;
  const int64_t cap = static_cast<int64_t>(ctas) * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// ------------------------------------------------------------------ init / data

__global__ void init_normal_k(float* p32, bf16* p16, int64_t n, float stdv, uint64_t seed,
                              uint64_t offset) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t h1 = mix64(seed ^ mix64(offset + uint64_t(i)));
    const uint64_t h2 = mix64(h1 ^ 0x5851f42d4c957f2dull);
    const float u1 = (float((h1 >> 40) + 1) * (1.0f / 16777217.0f));
    const float u2 = float(h2 >> 40) * (1.0f / 16777216.0f);
    const float z = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
    const float v = __bfloat162float(__float2bfloat16_rn(stdv * z));  // bf16-representable master
    if (p32) p32[i] = v;
    if (p16) p16[i] = __float2bfloat16_rn(v);
  }
}

__global__ void init_const_k(float* p32, bf16* p16, int64_t n, float value) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (p32) p32[i] = value;
    if (p16) p16[i] = __float2bfloat16_rn(value);
  }
}

__global__ void synth_tokens_k(int32_t* tok, int64_t first, int64_t count, int sp1, int vocab,
                               uint64_t seed, uint64_t it) {
  const int64_t total = count * sp1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = first + i / sp1;
    const int64_t t = i % sp1;
    const uint64_t h = mix64(mix64(mix64(seed ^ 0x7f4a7c15ull) ^ it) ^ (uint64_t(j) << 20 | uint64_t(t)));
    tok[i] = int32_t(h % uint64_t(vocab));
  }
}

// ------------------------------------------------------------------ embedding

// x[r] = wte[tok[r]] + wpe[r % seq]; tokens are [samples, seq+1] (inputs are columns 0..seq-1).
__global__ void embed_fwd_k(const int32_t* tok, int seq, const bf16* wte, const bf16* wpe, bf16* x,
                            int64_t rows, int h) {
  const int vec = h / 8;
  const int64_t total = rows * vec;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / vec;
    const int c = int(i % vec) * 8;
    const int64_t smp = r / seq;
    const int pos = int(r % seq);
    const int32_t t = tok[smp * (seq + 1) + pos];
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(wte + int64_t(t) * h + c), a);
    if (wpe) {
      unpack8(*reinterpret_cast<const uint4*>(wpe + int64_t(pos) * h + c), b);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += b[k];
    }
    *reinterpret_cast<uint4*>(x + r * h + c) = pack8(a);
  }
}

__global__ void embed_bwd_k(const int32_t* tok, int seq, const bf16* dx, float* dwte, float* dwpe,
                            int64_t rows, int h) {
  const int vec = h / 8;
  const int64_t total = rows * vec;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / vec;
    const int c = int(i % vec) * 8;
    const int64_t smp = r / seq;
    const int pos = int(r % seq);
    const int32_t t = tok[smp * (seq + 1) + pos];
    float d[8];
    unpack8(*reinterpret_cast<const uint4*>(dx + r * h + c), d);
    float4* wt = reinterpret_cast<float4*>(dwte + int64_t(t) * h + c);
    atomicAdd(wt, make_float4(d[0], d[1], d[2], d[3]));
    atomicAdd(wt + 1, make_float4(d[4], d[5], d[6], d[7]));
    if (dwpe) {
      float4* wp = reinterpret_cast<float4*>(dwpe + int64_t(pos) * h + c);
      atomicAdd(wp, make_float4(d[0], d[1], d[2], d[3]));
      atomicAdd(wp + 1, make_float4(d[4], d[5], d[6], d[7]));
    }
  }
}

// ------------------------------------------------------------------ LayerNorm (one warp per row)

// RMS = true: RMSNorm (no centring, no beta).
template <int NC, bool RMS>  // h = NC * 256
__global__ void __launch_bounds__(kThreads) ln_fwd_k(const bf16* __restrict__ x,
                                                     const bf16* __restrict__ g,
                                                     const bf16* __restrict__ b, bf16* y,
                                                     float* mean, float* rstd, int64_t rows) {
  constexpr int h = NC * 256;
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (kThreads / 32);
  for (int64_t r = blockIdx.x * int64_t(kThreads / 32) + threadIdx.x / 32; r < rows; r += warps) {
    if (r + warps < rows) {  // this warp's next row, toward L2
#pragma unroll
      for (int c = 0; c < NC; ++c)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + (r + warps) * h + (c * 32 + lane) * 8));
    }
    float v[NC][8];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      unpack8(*reinterpret_cast<const uint4*>(x + r * h + (c * 32 + lane) * 8), v[c]);
#pragma unroll
      for (int k = 0; k < 8; ++k) s += v[c][k];
    }
    const float mu = RMS ? 0.f : warp_sum(s) * (1.0f / h);
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float d = v[c][k] - mu;
        q += d * d;
      }
    const float rs = rsqrtf(warp_sum(q) * (1.0f / h) + 1e-5f);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int col = (c * 32 + lane) * 8;
      float gg[8], bb[8], o[8];
      unpack8(*reinterpret_cast<const uint4*>(g + col), gg);
      if (RMS) {
#pragma unroll
        for (int k = 0; k < 8; ++k) bb[k] = 0.f;
      } else {
        unpack8(*reinterpret_cast<const uint4*>(b + col), bb);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = (v[c][k] - mu) * rs * gg[k] + bb[k];
      *reinterpret_cast<uint4*>(y + r * h + col) = pack8(o);
    }
    if (lane == 0) {
      mean[r] = mu;
      rstd[r] = rs;
    }
  }
}

// LayerNorm / RMSNorm backward, rows: dx = dres + rstd * (g*dy - mean(g*dy) - xhat*mean(g*dy*xhat)).
// One warp per row, two streaming passes (sums, then dx) so no row is held in registers.
template <bool RMS>
__global__ void __launch_bounds__(kThreads) ln_bwd_rows_k(const bf16* __restrict__ dy,
                                                          const bf16* __restrict__ x,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ rstd,
                                                          const bf16* __restrict__ g, const bf16* dres,
                                                          bf16* dx, int64_t rows, int h) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (kThreads / 32);
  const float inv_h = 1.0f / h;
  for (int64_t r = blockIdx.x * int64_t(kThreads / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float mu = mean[r], rs = rstd[r];
    const bf16* xr = x + r * h;
    const bf16* dyr = dy + r * h;
    float s1 = 0.f, s2 = 0.f;
    for (int col = lane * 8; col < h; col += 256) {
      float xv[8], dv[8], gg[8];
      unpack8(*reinterpret_cast<const uint4*>(xr + col), xv);
      unpack8(*reinterpret_cast<const uint4*>(dyr + col), dv);
      unpack8(*reinterpret_cast<const uint4*>(g + col), gg);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float gd = gg[k] * dv[k];
        s1 += gd;
        s2 += gd * (xv[k] - mu) * rs;
      }
    }
    const float m1 = RMS ? 0.f : warp_sum(s1) * inv_h;
    const float m2 = warp_sum(s2) * inv_h;
    for (int col = lane * 8; col < h; col += 256) {
      float xv[8], dv[8], gg[8], rr[8], o[8];
      unpack8(*reinterpret_cast<const uint4*>(xr + col), xv);
      unpack8(*reinterpret_cast<const uint4*>(dyr + col), dv);
      unpack8(*reinterpret_cast<const uint4*>(g + col), gg);
      if (dres) {
        unpack8(*reinterpret_cast<const uint4*>(dres + r * h + col), rr);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) rr[k] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = rr[k] + rs * (gg[k] * dv[k] - m1 - (xv[k] - mu) * rs * m2);
      *reinterpret_cast<uint4*>(dx + r * h + col) = pack8(o);
    }
  }
}

// LayerNorm / RMSNorm backward in one pass over the rows: dx (+ residual) as above, plus per-CTA
// column partials of dgamma, dbeta and, with CS, of dx itself (the bias gradient of the linear
// layer whose output this norm read). Replaces the rows kernel + the column kernel (which re-read
// dy and x from HBM) + the separate bias colsum (which re-read dx). Each warp takes two rows at
// a time (their loads in flight together; a lane owns 8 consecutive columns per 256), adds the
// two rows' column contributions in registers and folds them into its own shared-memory slice,
// laid out [q][vector][k][lane] so each access is one conflict-free wavefront; the CTA folds its
// 8 slices at the end.
template <bool RMS, bool CS, int NV>  // NV = h / 256 when known at compile time, else 0
__global__ void __launch_bounds__(kThreads, 2) ln_bwd_fused_k(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                           const float* __restrict__ mean,
                                                           const float* __restrict__ rstd,
                                                           const bf16* __restrict__ g, const bf16* dres, bf16* dx,
                                                           int64_t rows, int h, int64_t chunk,
                                                           float* __restrict__ part, float* __restrict__ cs) {
  constexpr int Q = (RMS ? 1 : 2) + (CS ? 1 : 0);
  extern __shared__ float4 ln_acc4[];
  float* acc = reinterpret_cast<float*>(ln_acc4);  // [8 warps][Q][h]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nv = NV > 0 ? NV : h / 256;
  float* my = acc + size_t(w) * Q * h;
  for (int i = lane; i < Q * h; i += 32) my[i] = 0.f;
  __syncwarp();
  const float inv_h = 1.0f / h;
  const int64_t r0 = blockIdx.x * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  for (int64_t ra = r0 + 2 * w; ra < r1; ra += 2 * (kThreads / 32)) {
    const bool two = ra + 1 < r1;
    const int64_t rb = two ? ra + 1 : ra;
    const float mua = mean[ra], rsa = rstd[ra], mub = mean[rb], rsb = rstd[rb];
    const bf16* xa = x + ra * h + lane * 8;
    const bf16* xb = x + rb * h + lane * 8;
    const bf16* da = dy + ra * h + lane * 8;
    const bf16* db = dy + rb * h + lane * 8;
    float s1a = 0.f, s2a = 0.f, s1b = 0.f, s2b = 0.f;
    // four column chunks per step: 16 loads in flight per lane (one 8-warp CTA per SM at wide h is
    // otherwise latency-bound at ~0.45 of HBM)
#pragma unroll 4
    for (int j = 0; j < nv; ++j) {
      const uint4 qxa = *reinterpret_cast<const uint4*>(xa + 256 * j);
      const uint4 qda = *reinterpret_cast<const uint4*>(da + 256 * j);
      const uint4 qxb = *reinterpret_cast<const uint4*>(xb + 256 * j);
      const uint4 qdb = *reinterpret_cast<const uint4*>(db + 256 * j);
      if (dres) {  // the residual gradient is read in the second pass: start its HBM fetch now
        asm volatile("prefetch.global.L2 [%0];" ::"l"(dres + ra * h + lane * 8 + 256 * j));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(dres + rb * h + lane * 8 + 256 * j));
      }
      if (ra + 2 * (kThreads / 32) + 1 < r1) {  // the warp's next two rows, toward L2
        const int64_t rn = ra + 2 * (kThreads / 32);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + rn * h + lane * 8 + 256 * j));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(dy + rn * h + lane * 8 + 256 * j));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + (rn + 1) * h + lane * 8 + 256 * j));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(dy + (rn + 1) * h + lane * 8 + 256 * j));
      }
      float gg[8], xv[8], dv[8];
      unpack8(*reinterpret_cast<const uint4*>(g + lane * 8 + 256 * j), gg);
      unpack8(qxa, xv);
      unpack8(qda, dv);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float gd = gg[k] * dv[k];
        s1a += gd;
        s2a += gd * (xv[k] - mua) * rsa;
      }
      unpack8(qxb, xv);
      unpack8(qdb, dv);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float gd = gg[k] * dv[k];
        s1b += gd;
        s2b += gd * (xv[k] - mub) * rsb;
      }
    }
    const float m1a = RMS ? 0.f : warp_sum(s1a) * inv_h;
    const float m2a = warp_sum(s2a) * inv_h;
    const float m1b = RMS ? 0.f : warp_sum(s1b) * inv_h;
    const float m2b = warp_sum(s2b) * inv_h;
#pragma unroll 2
    for (int j = 0; j < nv; ++j) {  // second pass re-reads the two rows (L1 / L2 hits)
      const int col = lane * 8 + 256 * j;
      const uint4 qxa = *reinterpret_cast<const uint4*>(xa + 256 * j);
      const uint4 qda = *reinterpret_cast<const uint4*>(da + 256 * j);
      const uint4 qxb = *reinterpret_cast<const uint4*>(xb + 256 * j);
      const uint4 qdb = *reinterpret_cast<const uint4*>(db + 256 * j);
      uint4 qra = make_uint4(0, 0, 0, 0), qrb = make_uint4(0, 0, 0, 0);
      if (dres) {
        qra = *reinterpret_cast<const uint4*>(dres + ra * h + col);
        qrb = *reinterpret_cast<const uint4*>(dres + rb * h + col);
      }
      float gg[8], xv[8], dv[8], o[8], sg[8], sb[8], sc[8];
      unpack8(*reinterpret_cast<const uint4*>(g + col), gg);
      unpack8(qxa, xv);
      unpack8(qda, dv);
      unpack8(qra, o);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float xh = (xv[k] - mua) * rsa;
        o[k] += rsa * (gg[k] * dv[k] - m1a - xh * m2a);
        sg[k] = xh * dv[k];
        sb[k] = dv[k];
        sc[k] = o[k];
      }
      *reinterpret_cast<uint4*>(dx + ra * h + col) = pack8(o);
      unpack8(qxb, xv);
      unpack8(qdb, dv);
      unpack8(qrb, o);
      const float keep = two ? 1.f : 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float xh = (xv[k] - mub) * rsb;
        o[k] += rsb * (gg[k] * dv[k] - m1b - xh * m2b);
        sg[k] += keep * (xh * dv[k]);
        sb[k] += keep * dv[k];
        sc[k] += keep * o[k];
      }
      if (two) *reinterpret_cast<uint4*>(dx + rb * h + col) = pack8(o);
      float* p0 = my + (size_t(j) * 8) * 32 + lane;  // [q][j][k][lane]
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        p0[k * 32] += sg[k];
        if (!RMS) p0[h + k * 32] += sb[k];
        if (CS) p0[(Q - 1) * h + k * 32] += sc[k];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Q * h; i += kThreads) {
    const int q = i / h, c = i - q * h;
    const int sl = q * h + ((c >> 8) * 8 + (c & 7)) * 32 + ((c & 255) >> 3);
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < kThreads / 32; ++k) t += acc[size_t(k) * Q * h + sl];
    if (q == 0)
      part[int64_t(blockIdx.x) * h + c] = t;
    else if (!RMS && q == 1)
      part[int64_t(gridDim.x + blockIdx.x) * h + c] = t;
    else
      cs[int64_t(blockIdx.x) * h + c] = t;
  }
}

// The same backward for wide rows (h = 2048 V): the whole CTA takes one row at a time, thread t
// owning columns 8t + 2048v (v < V), so the row sits in registers for both passes (the warp-per-row
// kernel above re-reads each row from L2 and, at one 128 KB-smem CTA per SM, stays latency-bound
// at ~0.5 of HBM for h = 4096). The row statistics are one block reduction per row through a
// double-buffered shared array (one barrier per row); the next row's loads are issued before it.
// dgamma / dbeta / dx column partials accumulate in registers: no shared-memory slices. Output
// layout as ln_bwd_fused_k: part[blk][h] (dgamma), part[grid + blk][h] (dbeta), cs[blk][h].
template <bool RMS, bool CS, int V>
__global__ void __launch_bounds__(kThreads, 2) ln_bwd_rows_k(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ rstd,
                                                          const bf16* __restrict__ g, const bf16* dres, bf16* dx,
                                                          int64_t rows, int64_t chunk, float* __restrict__ part,
                                                          float* __restrict__ cs) {
  constexpr int h = 2048 * V;
  __shared__ float2 red[2][kThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int col0 = threadIdx.x * 8;
  float gg[V][8], ag[V][8], ab[V][8], ac[V][8];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    unpack8(*reinterpret_cast<const uint4*>(g + col0 + 2048 * v), gg[v]);
#pragma unroll
    for (int k = 0; k < 8; ++k) ag[v][k] = ab[v][k] = ac[v][k] = 0.f;
  }
  const int64_t r0 = blockIdx.x * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  uint4 qx[V], qd[V], qr[V];
  auto load = [&](int64_t r, uint4 (&ox)[V], uint4 (&od)[V], uint4 (&orr)[V]) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int64_t o = r * h + col0 + 2048 * v;
      ox[v] = *reinterpret_cast<const uint4*>(x + o);
      od[v] = *reinterpret_cast<const uint4*>(dy + o);
      orr[v] = dres ? *reinterpret_cast<const uint4*>(dres + o) : make_uint4(0, 0, 0, 0);
    }
  };
  if (r0 < r1) load(r0, qx, qd, qr);
  for (int64_t r = r0; r < r1; ++r) {
    uint4 nx[V], nd[V], nr[V];
    if (r + 1 < r1) load(r + 1, nx, nd, nr);  // in flight during this row's reduction
    if (r + 2 < r1) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int64_t o = (r + 2) * h + col0 + 2048 * v;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(dy + o));
      }
    }
    const float mu = RMS ? 0.f : mean[r], rs = rstd[r];
    float xv[V][8], dv[V][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      unpack8(qx[v], xv[v]);
      unpack8(qd[v], dv[v]);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        xv[v][k] = (xv[v][k] - mu) * rs;  // x-hat
        const float gd = gg[v][k] * dv[v][k];
        s1 += gd;
        s2 += gd * xv[v][k];
      }
    }
    s2 = warp_sum(s2);
    if (!RMS) s1 = warp_sum(s1);
    if (lane == 0) red[r & 1][w] = make_float2(s1, s2);
    __syncthreads();
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) {
      const float2 p = red[r & 1][i];
      t1 += p.x;
      t2 += p.y;
    }
    const float m1 = RMS ? 0.f : t1 * (1.0f / h), m2 = t2 * (1.0f / h);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float o[8];
      unpack8(qr[v], o);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        o[k] += rs * (gg[v][k] * dv[v][k] - m1 - xv[v][k] * m2);
        ag[v][k] += xv[v][k] * dv[v][k];
        if (!RMS) ab[v][k] += dv[v][k];
        if (CS) ac[v][k] += o[k];
      }
      *reinterpret_cast<uint4*>(dx + r * h + col0 + 2048 * v) = pack8(o);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      qx[v] = nx[v];
      qd[v] = nd[v];
      qr[v] = nr[v];
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    float* pg = part + int64_t(blockIdx.x) * h + col0 + 2048 * v;
    *reinterpret_cast<float4*>(pg) = make_float4(ag[v][0], ag[v][1], ag[v][2], ag[v][3]);
    *reinterpret_cast<float4*>(pg + 4) = make_float4(ag[v][4], ag[v][5], ag[v][6], ag[v][7]);
    if (!RMS) {
      float* pb = part + int64_t(gridDim.x + blockIdx.x) * h + col0 + 2048 * v;
      *reinterpret_cast<float4*>(pb) = make_float4(ab[v][0], ab[v][1], ab[v][2], ab[v][3]);
      *reinterpret_cast<float4*>(pb + 4) = make_float4(ab[v][4], ab[v][5], ab[v][6], ab[v][7]);
    }
    if (CS) {
      float* pc = cs + int64_t(blockIdx.x) * h + col0 + 2048 * v;
      *reinterpret_cast<float4*>(pc) = make_float4(ac[v][0], ac[v][1], ac[v][2], ac[v][3]);
      *reinterpret_cast<float4*>(pc + 4) = make_float4(ac[v][4], ac[v][5], ac[v][6], ac[v][7]);
    }
  }
}

// dgamma / dbeta partial column sums over a chunk of rows: block (32, 8) covers 256 columns.
// part[chunk][h] holds dgamma partials, part[nchunks + chunk][h] dbeta partials.
template <bool RMS>
__global__ void ln_bwd_cols_k(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                              const float* __restrict__ mean, const float* __restrict__ rstd, int64_t rows,
                              int h, int64_t chunk, float* part) {
  __shared__ float sg[8][256], sb[8][256];
  const int c = blockIdx.x * 256 + threadIdx.x * 8;
  const int64_t r0 = blockIdx.y * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  float ag[8], ab[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) ag[k] = ab[k] = 0.f;
  if (c < h) {
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      const float mu = mean[r], rs = rstd[r];
      float xv[8], dv[8];
      unpack8(*reinterpret_cast<const uint4*>(x + r * h + c), xv);
      unpack8(*reinterpret_cast<const uint4*>(dy + r * h + c), dv);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ag[k] += dv[k] * (xv[k] - mu) * rs;
        ab[k] += dv[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    sg[threadIdx.y][threadIdx.x * 8 + k] = ag[k];
    sb[threadIdx.y][threadIdx.x * 8 + k] = ab[k];
  }
  __syncthreads();
  const int t = threadIdx.y * 32 + threadIdx.x;
  const int col = blockIdx.x * 256 + t;
  if (col < h) {
    float a = 0.f, bsum = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a += sg[k][t];
      bsum += sb[k][t];
    }
    part[int64_t(blockIdx.y) * h + col] = a;
    if (!RMS) part[int64_t(gridDim.y + blockIdx.y) * h + col] = bsum;
  }
}

// ------------------------------------------------------------------ cross-entropy

__device__ __forceinline__ float block_reduce(float v, float* sh, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float t = (threadIdx.x < kThreads / 32) ? sh[threadIdx.x] : (is_max ? -INFINITY : 0.f);
  if (w == 0) t = is_max ? warp_max(t) : warp_sum(t);
  if (threadIdx.x == 0) sh[0] = t;
  __syncthreads();
  return sh[0];
}

// Combines two (max, sum-of-exp2) pairs of an online softmax in the log2 domain.
__device__ __forceinline__ float ex2_fast(float x) {  // MUFU.EX2 (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  const float mx = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * exp2f(m - mx)) + (m2 == -INFINITY ? 0.f : s2 * exp2f(m2 - mx));
  m = mx;
}

// One CTA per row. Pass 1: per-thread online max / sum of exp2 in the log2 domain (one read of
// the logits, one exp2 per element, a rescale only when the running max grows). Pass 2:
// overwrite the logits with (softmax - onehot) * gscale (one exp2 per element).
__global__ void __launch_bounds__(kThreads) ce_k(bf16* logits, const int32_t* tok, int seq, int64_t rows,
                                                 int vocab, int ldv, float gscale, float* row_loss) {
  constexpr float kL2e = 1.4426950408889634f;
  __shared__ float shm[kThreads / 32], shs[kThreads / 32];
  const int nvec = ldv / 8;
  const int nfull = vocab / 8;  // chunks entirely inside the vocabulary
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    bf16* lg = logits + r * ldv;
    const int64_t smp = r / seq;
    const int pos = int(r % seq);
    const int target = tok[smp * (seq + 1) + pos + 1];
    float m = -INFINITY, sum = 0.f;
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(lg + i * 8), f);
      float cm = -INFINITY;
      if (i < nfull) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          f[k] *= kL2e;
          cm = fmaxf(cm, f[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          f[k] = (i * 8 + k < vocab) ? f[k] * kL2e : -INFINITY;
          cm = fmaxf(cm, f[k]);
        }
      }
      if (cm == -INFINITY) continue;
      if (cm > m) {
        sum = (m == -INFINITY) ? 0.f : sum * exp2f(m - cm);
        m = cm;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += exp2f(f[k] - m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      lse_merge(m, sum, m2, s2);
    }
    __syncthreads();
    if (lane == 0) {
      shm[w] = m;
      shs[w] = sum;
    }
    __syncthreads();
    m = shm[0];
    sum = shs[0];
    for (int k = 1; k < kThreads / 32; ++k) lse_merge(m, sum, shm[k], shs[k]);
    const float lse = (m + log2f(sum)) / kL2e;  // natural log-sum-exp
    const float tl = __bfloat162float(lg[target]);
    __syncthreads();  // everyone has read lg[target] before it is overwritten
    const float coef = gscale / sum;
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(lg + i * 8), f);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int col = i * 8 + k;
        float gv = (i < nfull || col < vocab) ? exp2f(f[k] * kL2e - m) * coef : 0.f;
        if (col == target) gv -= gscale;
        f[k] = gv;
      }
      *reinterpret_cast<uint4*>(lg + i * 8) = pack8(f);
    }
    if (threadIdx.x == 0) row_loss[r] = lse - tl;
  }
}

// Rows that fit twice in shared memory (vocab up to ~56K): one persistent CTA per SM streams
// rows through two smem buffers with bulk copies (the next row loads while this one is
// processed), so the logits are read from HBM once and the gradient written once. Pass 1 (online
// max / sum of exp2) and pass 2 (gradient) both read the row from shared memory.
constexpr int kCeThreads = 512;
__global__ void __launch_bounds__(kCeThreads, 1) ce_smem_k(bf16* logits, const int32_t* tok, int seq, int64_t rows,
                                                           int vocab, int ldv, float gscale, float* row_loss) {
  constexpr float kL2e = 1.4426950408889634f;
  extern __shared__ __align__(128) uint8_t ce_smem[];
  __shared__ uint64_t bar[2];
  __shared__ float shm[kCeThreads / 32], shs[kCeThreads / 32];
  const uint32_t row_bytes = uint32_t(ldv) * 2;
  const uint32_t stride = (row_bytes + 127) & ~127u;
  const int nvec = ldv / 8, nfull = vocab / 8;
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int64_t r, int buf) {
    ptx::mbar_arrive_expect_tx(&bar[buf], row_bytes);
    ptx::bulk_load(ce_smem + buf * stride, logits + r * ldv, row_bytes, &bar[buf]);
  };
  if (threadIdx.x == 0 && blockIdx.x < rows) issue(blockIdx.x, 0);
  uint32_t it = 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++it) {
    const int buf = it & 1;
    if (threadIdx.x == 0 && r + gridDim.x < rows) issue(r + gridDim.x, buf ^ 1);
    ptx::mbar_wait(&bar[buf], (it >> 1) & 1);
    const uint4* row = reinterpret_cast<const uint4*>(ce_smem + buf * stride);
    const int64_t smp = r / seq;
    const int pos = int(r % seq);
    const int target = tok[smp * (seq + 1) + pos + 1];
    // One MUFU exp2 per element: pass 1 takes the row max (packed bf16x2 max, order-preserving
    // under the positive log2(e) scale); pass 2 computes e = exp2(x*log2e - max), sums it and
    // stores it in place as bf16; pass 3 writes (e / sum - onehot) * gscale.
    float tl = 0.f;
    if (threadIdx.x == 0) tl = __bfloat162float(reinterpret_cast<const bf16*>(row)[target]);
    __nv_bfloat162 mx2 = __float2bfloat162_rn(-INFINITY);
    for (int i = threadIdx.x; i < nfull; i += kCeThreads) {
      const uint4 u = row[i];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
      mx2 = __hmax2(mx2, __hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3])));
    }
    float m = fmaxf(__low2float(mx2), __high2float(mx2));
    if (nfull < nvec && threadIdx.x == (nfull % kCeThreads)) {  // ragged tail chunk (vocab % 8)
      const bf16* t = reinterpret_cast<const bf16*>(row) + nfull * 8;
      for (int k = 0; k < vocab - nfull * 8; ++k) m = fmaxf(m, __bfloat162float(t[k]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) shm[w] = m;
    __syncthreads();
    m = shm[0];
#pragma unroll
    for (int k = 1; k < kCeThreads / 32; ++k) m = fmaxf(m, shm[k]);
    m *= kL2e;
    uint4* rw = reinterpret_cast<uint4*>(ce_smem + buf * stride);
    float s0 = 0.f, s1 = 0.f;
    for (int i = threadIdx.x; i < nvec; i += kCeThreads) {
      const uint4 u = rw[i];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
      float f[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 t = __bfloat1622float2(h[k]);
        f[2 * k] = ex2_fast(fmaf(t.x, kL2e, -m));
        f[2 * k + 1] = ex2_fast(fmaf(t.y, kL2e, -m));
      }
      if (i >= nfull) {
        const int valid = vocab - i * 8;  // < 8 on the ragged tail chunk
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = k < valid ? f[k] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        s0 += f[k];
        s1 += f[k + 1];
      }
      rw[i] = pack8(f);
    }
    float sum = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) shs[w] = sum;
    __syncthreads();
    sum = shs[0];
#pragma unroll
    for (int k = 1; k < kCeThreads / 32; ++k) sum += shs[k];
    const float coef = gscale / sum;
    uint4* out = reinterpret_cast<uint4*>(logits + r * ldv);
    for (int i = threadIdx.x; i < nvec; i += kCeThreads) {
      float f[8];
      unpack8(rw[i], f);
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] *= coef;
      out[i] = pack8(f);
    }
    // one-hot term: the thread that wrote the target's chunk rewrites that element (program
    // order on the same address)
    if (threadIdx.x == (target / 8) % kCeThreads) {
      const float e = __bfloat162float(reinterpret_cast<const bf16*>(rw)[target]);
      logits[r * ldv + target] = __float2bfloat16_rn(e * coef - gscale);
    }
    if (threadIdx.x == 0) row_loss[r] = (m + __log2f(sum)) / kL2e - tl;
    __syncthreads();  // buffer `buf` is refilled by the next iteration's prefetch
  }
}

// The same cross-entropy with each thread's share of the row held in registers (MAXC 16-byte
// chunks): one shared-memory read pass instead of three, and the row's buffer is handed back to
// the bulk-copy engine as soon as the block has read it (two rows in flight while one computes).
template <int MAXC>
__global__ void __launch_bounds__(kCeThreads, 1) ce_reg_k(bf16* logits, const int32_t* tok, int seq, int64_t rows,
                                                          int vocab, int ldv, float gscale, float* row_loss) {
  constexpr float kL2e = 1.4426950408889634f;
  extern __shared__ __align__(128) uint8_t ce_smem[];
  __shared__ uint64_t bar[2];
  __shared__ float shm[kCeThreads / 32], shs[kCeThreads / 32];
  const uint32_t row_bytes = uint32_t(ldv) * 2;
  const uint32_t stride = (row_bytes + 127) & ~127u;
  const int nvec = ldv / 8, nfull = vocab / 8;
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int64_t r, int buf) {
    ptx::mbar_arrive_expect_tx(&bar[buf], row_bytes);
    ptx::bulk_load(ce_smem + buf * stride, logits + r * ldv, row_bytes, &bar[buf]);
  };
  if (threadIdx.x == 0) {
    if (blockIdx.x < rows) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < rows) issue(blockIdx.x + gridDim.x, 1);
  }
  uint32_t it = 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++it) {
    const int buf = it & 1;
    ptx::mbar_wait(&bar[buf], (it >> 1) & 1);
    const uint4* row = reinterpret_cast<const uint4*>(ce_smem + buf * stride);
    const int64_t smp = r / seq;
    const int pos = int(r % seq);
    const int target = tok[smp * (seq + 1) + pos + 1];
    float tl = 0.f;
    if (threadIdx.x == 0) tl = __bfloat162float(reinterpret_cast<const bf16*>(row)[target]);
    uint4 q[MAXC];
    __nv_bfloat162 mx2 = __float2bfloat162_rn(-INFINITY);
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = threadIdx.x + c * kCeThreads;
      q[c] = i < nvec ? row[i] : make_uint4(0, 0, 0, 0);
      if (i < nfull) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[c]);
        mx2 = __hmax2(mx2, __hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3])));
      }
    }
    float m = fmaxf(__low2float(mx2), __high2float(mx2));
    if (nfull < nvec && threadIdx.x == (nfull % kCeThreads)) {  // ragged tail chunk (vocab % 8)
      const bf16* t = reinterpret_cast<const bf16*>(row) + nfull * 8;
      for (int k = 0; k < vocab - nfull * 8; ++k) m = fmaxf(m, __bfloat162float(t[k]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) shm[w] = m;
    __syncthreads();  // every thread has read the row: the buffer takes the row after next
    if (threadIdx.x == 0 && r + 2 * int64_t(gridDim.x) < rows) {
      ptx::fence_proxy_async_smem();
      issue(r + 2 * int64_t(gridDim.x), buf);
    }
    m = shm[0];
#pragma unroll
    for (int k = 1; k < kCeThreads / 32; ++k) m = fmaxf(m, shm[k]);
    m *= kL2e;
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = threadIdx.x + c * kCeThreads;
      if (i < nvec) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[c]);
        float f[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 t = __bfloat1622float2(h[k]);
          f[2 * k] = ex2_fast(fmaf(t.x, kL2e, -m));
          f[2 * k + 1] = ex2_fast(fmaf(t.y, kL2e, -m));
        }
        if (i >= nfull) {
          const int valid = vocab - i * 8;
#pragma unroll
          for (int k = 0; k < 8; ++k) f[k] = k < valid ? f[k] : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          s0 += f[k];
          s1 += f[k + 1];
        }
        q[c] = pack8(f);  // e rounded to bf16, as the shared-memory kernel stores it
      }
    }
    float sum = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) shs[w] = sum;
    __syncthreads();
    sum = shs[0];
#pragma unroll
    for (int k = 1; k < kCeThreads / 32; ++k) sum += shs[k];
    const float coef = gscale / sum;
    uint4* out = reinterpret_cast<uint4*>(logits + r * ldv);
    const int tchunk = target / 8, tk = target - tchunk * 8;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = threadIdx.x + c * kCeThreads;
      if (i < nvec) {
        float f[8];
        unpack8(q[c], f);
        const float sub = i == tchunk ? gscale : 0.f;  // one-hot term, branch-free
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = f[k] * coef - (k == tk ? sub : 0.f);
        out[i] = pack8(f);
      }
    }
    if (threadIdx.x == 0) row_loss[r] = (m + __log2f(sum)) / kL2e - tl;
    __syncthreads();  // shm / shs reused by the next row
  }
}

// ------------------------------------------------------------------ reductions

// Partial column sums: block (32, 8) covers 256 columns (8 per thread, 16-byte loads) x one
// row chunk; warp rows read 512 contiguous bytes.
__global__ void colsum_part_k(const bf16* X, int64_t rows, int N, int ld, int64_t chunk, float* work) {
  __shared__ float sh[8][256];
  const int c = blockIdx.x * 256 + threadIdx.x * 8;
  const int64_t r0 = blockIdx.y * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 0.f;
  if (c < N) {
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      if (r + 32 < r1) asm volatile("prefetch.global.L2 [%0];" ::"l"(X + (r + 32) * ld + c));  // 4 rows ahead
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(X + r * ld + c), f);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += f[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) sh[threadIdx.y][threadIdx.x * 8 + k] = a[k];
  __syncthreads();
  const int t = threadIdx.y * 32 + threadIdx.x;  // 256 threads, one column each
  const int col = blockIdx.x * 256 + t;
  if (col < N) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += sh[k][t];
    work[int64_t(blockIdx.y) * N + col] = s;
  }
}

// out[c] = sum over k of part[k, c]: block (32 columns x 8 row stripes), coalesced 128-byte rows.
// 32 columns per CTA, 32 row groups: a few independent loads per thread (latency-bound size)
// Column sums of nparts partial rows: out[c] (bf16) = sum, or, with out32, out32[c] = (acc32 ?
// out32[c] : 0) + sum (a gradient written straight into the fp32 accumulator).
__global__ void __launch_bounds__(1024) sum_partials_k(const float* part, int nparts, int N, bf16* out,
                                                       float* out32, int acc32) {
  __shared__ float sh[32][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  float s0 = 0.f, s1 = 0.f;
  if (c < N) {
    int k = threadIdx.y;
    for (; k + 32 < nparts; k += 64) {
      s0 += part[int64_t(k) * N + c];
      s1 += part[int64_t(k + 32) * N + c];
    }
    if (k < nparts) s0 += part[int64_t(k) * N + c];
  }
  sh[threadIdx.y][threadIdx.x] = s0 + s1;
  __syncthreads();
  if (threadIdx.y == 0 && c < N) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) s += sh[k][threadIdx.x];
    if (out32)
      out32[c] = acc32 ? out32[c] + s : s;
    else
      out[c] = __float2bfloat16_rn(s);
  }
}

__global__ void cast_k(const float* in, bf16* out, int64_t n) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(in)[i];
    uint2 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
    o2[0] = __floats2bfloat162_rn(v.x, v.y);
    o2[1] = __floats2bfloat162_rn(v.z, v.w);
    reinterpret_cast<uint2*>(out)[i] = o;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

__global__ void reduce_sum_k(const float* x, int64_t n, float* out) {
  __shared__ float sh[32];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) s += x[i];
  s = block_reduce(s, sh, false);
  if (threadIdx.x == 0) *out = s;
}

// ------------------------------------------------------------------ ZeRO: accumulate / AdamW

__global__ void add_f32_k(float* dst, const float* src, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

// acc[i] = (first ? 0 : acc[i]) + sum over j = 0..n-1, in rank order, of bf16 src_j[i]: the local
// half of the copy-engine ZeRO-3 reduce-scatter (the same fixed-order fp32 sum as peer_rs_acc_k).
struct SliceSrcs {
  const bf16* p[8];
};
__global__ void reduce_slices_k(float* __restrict__ acc, SliceSrcs src, int n, int64_t len, bool first) {
  const int64_t n8 = len / 8;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    float a[8];
    if (first) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = 0.f;
    } else {
      const float4 x = reinterpret_cast<const float4*>(acc)[2 * i], y = reinterpret_cast<const float4*>(acc)[2 * i + 1];
      a[0] = x.x; a[1] = x.y; a[2] = x.z; a[3] = x.w; a[4] = y.x; a[5] = y.y; a[6] = y.z; a[7] = y.w;
    }
    for (int j = 0; j < n; ++j) {
      float v[8];
      unpack8(reinterpret_cast<const uint4*>(src.p[j])[i], v);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += v[k];
    }
    reinterpret_cast<float4*>(acc)[2 * i] = make_float4(a[0], a[1], a[2], a[3]);
    reinterpret_cast<float4*>(acc)[2 * i + 1] = make_float4(a[4], a[5], a[6], a[7]);
  }
}

__global__ void accumulate_k(float* acc, const bf16* src, int64_t n, bool overwrite) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint2 raw = reinterpret_cast<const uint2*>(src)[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
    const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
    float4 o = make_float4(a.x, a.y, b.x, b.y);
    if (!overwrite) {
      const float4 p = reinterpret_cast<const float4*>(acc)[i];
      o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
    }
    reinterpret_cast<float4*>(acc)[i] = o;
  }
}

// 4 elements per thread-iteration: 16 B of p32, m, v (+acc) and 8 B of bf16 grad / params.
__global__ void __launch_bounds__(kThreads) adam_k(float* __restrict__ p32, float* __restrict__ m,
                                                   float* __restrict__ v, bf16* __restrict__ p16,
                                                   const float* __restrict__ acc,
                                                   const bf16* __restrict__ g16,
                                                   const float* __restrict__ g32, int64_t n,
                                                   AdamParams ap) {
  const int64_t n4 = n / 4;
  const float inv_bc1 = 1.0f / ap.bc1;
  const float inv_sqrt_bc2 = rsqrtf(ap.bc2);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    if (acc) {
      const float4 a = reinterpret_cast<const float4*>(acc)[i];
      g[0] = a.x; g[1] = a.y; g[2] = a.z; g[3] = a.w;
    }
    if (g16) {
      const uint2 raw = reinterpret_cast<const uint2*>(g16)[i];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
      g[0] += a.x; g[1] += a.y; g[2] += b.x; g[3] += b.y;
    }
    if (g32) {
      const float4 a = reinterpret_cast<const float4*>(g32)[i];
      g[0] += a.x; g[1] += a.y; g[2] += a.z; g[3] += a.w;
    }
    float4 pp = reinterpret_cast<float4*>(p32)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float* P = &pp.x;
    float* M = &mm.x;
    float* V = &vv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      M[k] = ap.beta1 * M[k] + (1.f - ap.beta1) * g[k];
      V[k] = ap.beta2 * V[k] + (1.f - ap.beta2) * g[k] * g[k];
      const float denom = sqrtf(V[k]) * inv_sqrt_bc2 + ap.eps;
      P[k] -= ap.lr * ((M[k] * inv_bc1) / denom + ap.weight_decay * P[k]);
    }
    reinterpret_cast<float4*>(p32)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    uint2 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
    oh[0] = __floats2bfloat162_rn(pp.x, pp.y);
    oh[1] = __floats2bfloat162_rn(pp.z, pp.w);
    reinterpret_cast<uint2*>(p16)[i] = o;
  }
}

}  // namespace

// ------------------------------------------------------------------ RoPE (rotate-half, any head_dim)

// cos / sin of pos * theta^(-2j/64) for pos < seq, j < 32 (computed once per (seq, theta) in
// double precision, kept in a small per-process table).
// cos/sin of position pos and rotation pair j (frequency theta^(-2j/dh)), [seq][dh/2].
__global__ void rope_table_k(float2* tab, int seq, int half, double log_theta) {
  const int n = seq * half;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int pos = i / half, j = i % half;
    const double ang = double(pos) * exp(-double(2 * j) / double(2 * half) * log_theta);
    tab[i] = make_float2(float(cos(ang)), float(sin(ang)));
  }
}

// In place on the Q and K column blocks of qkv [T, 3h]; inverse = rotation by -theta (backward).
// Rotate-half pairing (i, i + dh/2) inside every head of dh columns. One thread per
// (token, Q|K, head, group of 8 rotation pairs): two 16-byte loads / stores.
__global__ void rope_k(bf16* qkv, const float2* __restrict__ tab, int64_t tokens, int seq, int h, int dh,
                       float sign) {
  const int heads = h / dh, half = dh / 2, groups = half / 8;
  const int per_tok = 2 * heads * groups;
  const int64_t total = tokens * per_tok;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / per_tok;
    const int r = int(i - t * per_tok);
    const int blk = r / (heads * groups), rem = r - blk * (heads * groups);
    const int head = rem / groups, j0 = (rem % groups) * 8;
    const int pos = int(t % seq);
    bf16* v = qkv + t * 3 * h + blk * h + head * dh + j0;
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(v), a);
    unpack8(*reinterpret_cast<const uint4*>(v + half), b);
    const float4* cs4 = reinterpret_cast<const float4*>(tab + pos * half + j0);
    float o0[8], o1[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 w = cs4[k];  // (cos, sin) of pairs 2k and 2k+1
      const float c0 = w.x, s0 = sign * w.y, c1 = w.z, s1 = sign * w.w;
      o0[2 * k] = a[2 * k] * c0 - b[2 * k] * s0;
      o1[2 * k] = b[2 * k] * c0 + a[2 * k] * s0;
      o0[2 * k + 1] = a[2 * k + 1] * c1 - b[2 * k + 1] * s1;
      o1[2 * k + 1] = b[2 * k + 1] * c1 + a[2 * k + 1] * s1;
    }
    *reinterpret_cast<uint4*>(v) = pack8(o0);
    *reinterpret_cast<uint4*>(v + half) = pack8(o1);
  }
}

// ------------------------------------------------------------------ SwiGLU (gate/up interleaved
// in 32-column blocks: feature j has gate at 64*(j/32) + j%32 and up 32 columns later)

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }

__global__ void swiglu_fwd_k(const bf16* __restrict__ gu, bf16* __restrict__ out, int64_t tokens, int f) {
  const int64_t total = tokens * (f / 8);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / (f / 8);
    const int j0 = int(i % (f / 8)) * 8;  // 8 features, same 32-block
    const int64_t gbase = t * 2 * f + (j0 / 32) * 64 + (j0 % 32);
    float a[8], b[8], o[8];
    unpack8(*reinterpret_cast<const uint4*>(gu + gbase), a);
    unpack8(*reinterpret_cast<const uint4*>(gu + gbase + 32), b);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = a[k] * sigmoidf_(a[k]) * b[k];
    *reinterpret_cast<uint4*>(out + t * f + j0) = pack8(o);
  }
}

__global__ void swiglu_bwd_k(const bf16* __restrict__ gu, const bf16* __restrict__ dh, bf16* __restrict__ dgu,
                             int64_t tokens, int f) {
  const int64_t total = tokens * (f / 8);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / (f / 8);
    const int j0 = int(i % (f / 8)) * 8;
    const int64_t gbase = t * 2 * f + (j0 / 32) * 64 + (j0 % 32);
    float a[8], b[8], d[8], da[8], db[8];
    unpack8(*reinterpret_cast<const uint4*>(gu + gbase), a);
    unpack8(*reinterpret_cast<const uint4*>(gu + gbase + 32), b);
    unpack8(*reinterpret_cast<const uint4*>(dh + t * f + j0), d);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float sg = sigmoidf_(a[k]);
      const float silu = a[k] * sg;
      db[k] = d[k] * silu;
      da[k] = d[k] * b[k] * sg * (1.0f + a[k] * (1.0f - sg));
    }
    *reinterpret_cast<uint4*>(dgu + gbase) = pack8(da);
    *reinterpret_cast<uint4*>(dgu + gbase + 32) = pack8(db);
  }
}

// ------------------------------------------------------------------ launchers

std::atomic<int64_t> g_launches{0};
void note_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }


void init_normal(float* p32, bf16* p16, int64_t n, float stdv, uint64_t seed, uint64_t offset,
                 int ctas, cudaStream_t s) {
  init_normal_k<<<grid_for(n, kThreads, ctas), kThreads, 0, s>>>(p32, p16, n, stdv, seed, offset); note_launch();
}
void init_const(float* p32, bf16* p16, int64_t n, float value, int ctas, cudaStream_t s) {
  init_const_k<<<grid_for(n, kThreads, ctas), kThreads, 0, s>>>(p32, p16, n, value); note_launch();
}
void synth_tokens(int32_t* tokens, int64_t first, int64_t count, int sp1, int vocab, uint64_t seed,
                  uint64_t it, int ctas, cudaStream_t s) {
  if (count <= 0) return;
  synth_tokens_k<<<grid_for(count * sp1, kThreads, ctas), kThreads, 0, s>>>(tokens, first, count,
                                                                          sp1, vocab, seed, it); note_launch();
}
void embed_fwd(const int32_t* tokens, int seq, const bf16* wte, const bf16* wpe, bf16* x,
               int64_t rows, int h, int ctas, cudaStream_t s) {
  embed_fwd_k<<<grid_for(rows * h / 8, kThreads, ctas), kThreads, 0, s>>>(tokens, seq, wte, wpe, x,
                                                                          rows, h); note_launch();
}
const float2* rope_table(int seq, int dh, float theta, cudaStream_t s) {
  // per-device cos/sin table for the largest sequence seen on that device (a process may drive
  // several GPUs, one host thread each)
  struct Table {
    float2* tab = nullptr;
    int seq = 0, half = 0;
    float theta = 0.f;
  };
  static Table tables[64];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  Table& t = tables[dev & 63];
  if (seq > t.seq || theta != t.theta || dh / 2 != t.half) {
    if (t.tab) cudaFree(t.tab);
    t.tab = nullptr;
    t.seq = 0;
    if (cudaMalloc(&t.tab, size_t(seq) * (dh / 2) * sizeof(float2)) != cudaSuccess) return nullptr;
    rope_table_k<<<(seq * (dh / 2) + kThreads - 1) / kThreads, kThreads, 0, s>>>(t.tab, seq, dh / 2,
                                                                               std::log(double(theta)));
    note_launch();
    t.seq = seq;
    t.half = dh / 2;
    t.theta = theta;
  }
  return t.tab;
}

void rope(bf16* qkv, int64_t tokens, int seq, int h, float theta, bool inverse, int ctas, cudaStream_t s, int dh) {
  const float2* tab = rope_table(seq, dh, theta, s);
  if (!tab) return;
  rope_k<<<grid_for(tokens * 2 * (h / dh) * (dh / 16), kThreads, ctas), kThreads, 0, s>>>(qkv, tab, tokens, seq, h,
                                                                                        dh, inverse ? -1.f : 1.f);
  note_launch();
}
void swiglu_fwd(const bf16* gu, bf16* out, int64_t tokens, int f, int ctas, cudaStream_t s) {
  swiglu_fwd_k<<<grid_for(tokens * f / 8, kThreads, ctas), kThreads, 0, s>>>(gu, out, tokens, f); note_launch();
}
void swiglu_bwd(const bf16* gu, const bf16* dh, bf16* dgu, int64_t tokens, int f, int ctas, cudaStream_t s) {
  swiglu_bwd_k<<<grid_for(tokens * f / 8, kThreads, ctas), kThreads, 0, s>>>(gu, dh, dgu, tokens, f); note_launch();
}
void embed_bwd(const int32_t* tokens, int seq, const bf16* dx, float* dwte32, float* dwpe32,
               int64_t rows, int h, int ctas, cudaStream_t s) {
  embed_bwd_k<<<grid_for(rows * h / 8, kThreads, ctas), kThreads, 0, s>>>(tokens, seq, dx, dwte32,
                                                                          dwpe32, rows, h); note_launch();
}

#define ZP_LN_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(8) X(12) X(16)

cudaError_t layernorm_fwd(const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mean,
                          float* rstd, int64_t rows, int h, int ctas, cudaStream_t s) {
  const int grid = grid_for(rows, kThreads / 32, ctas, 8);
  switch (h / 256) {
#define X(NC)                                                                     \
  case NC:                                                                        \
    if (h % 256) return cudaErrorInvalidValue;                                    \
    if (b)                                                                        \
      ln_fwd_k<NC, false><<<grid, kThreads, 0, s>>>(x, g, b, y, mean, rstd, rows); \
    else                                                                          \
      ln_fwd_k<NC, true><<<grid, kThreads, 0, s>>>(x, g, b, y, mean, rstd, rows); note_launch();         \
    return cudaGetLastError();
    ZP_LN_CASES(X)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t layernorm_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd,
                          const bf16* g, const bf16* dres, bf16* dx, float* part, int* nblk,
                          int64_t rows, int h, int ctas, cudaStream_t s, bool rms, float* cs) {
  if (h % 256) return cudaErrorInvalidValue;
  static const bool rows_kernel = !std::getenv("ZP_LN_ROWS") || std::atoi(std::getenv("ZP_LN_ROWS")) != 0;
  if (rows_kernel && (h == 2048 || (h == 4096 && rms && !cs))) {  // wide rows: one row per CTA step
    int grid = int(std::min<int64_t>(int64_t(ctas) * 2, rows));
    if (grid < 1) grid = 1;
    const int64_t chunk = (rows + grid - 1) / grid;
    grid = int((rows + chunk - 1) / chunk);
    *nblk = grid;
    // (h = 4096 only for RMSNorm without the dx column sums: more accumulators would spill)
    const auto kern = h == 4096 ? ln_bwd_rows_k<true, false, 2>
                      : rms     ? (cs ? ln_bwd_rows_k<true, true, 1> : ln_bwd_rows_k<true, false, 1>)
                                : (cs ? ln_bwd_rows_k<false, true, 1> : ln_bwd_rows_k<false, false, 1>);
    kern<<<grid, kThreads, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, chunk, part, cs);
    note_launch();
    return cudaGetLastError();
  }
  const int Q = (rms ? 1 : 2) + (cs ? 1 : 0);
  const size_t smem = size_t(kThreads / 32) * Q * h * sizeof(float);
  if (smem <= 200 * 1024) {
    // one pass; as many CTAs per SM slot of the budget as shared memory allows
    const int per_sm = int(std::max<size_t>(1, std::min<size_t>(2, 227 * 1024 / (smem + 1024))));  // 2: registers
    int grid = int(std::min<int64_t>(int64_t(ctas) * per_sm, (rows + 31) / 32));
    if (grid < 1) grid = 1;
    const int64_t chunk = (rows + grid - 1) / grid;
    grid = int((rows + chunk - 1) / chunk);
    *nblk = grid;
#define ZP_LNB(R, C, NV)                                                                               \
  {                                                                                                    \
    static std::atomic<uint64_t> attr{0};                                                                          \
    if (first_on_device(attr)) {                                                                                       \
      cudaFuncSetAttribute(ln_bwd_fused_k<R, C, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
    }                                                                                                  \
    ln_bwd_fused_k<R, C, NV><<<grid, kThreads, smem, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h, chunk, part, cs); \
  }
    if (rms) {
      if (cs) ZP_LNB(true, true, 0) else ZP_LNB(true, false, 0)
    } else if (h == 768) {
      if (cs) ZP_LNB(false, true, 3) else ZP_LNB(false, false, 3)
    } else if (h == 1024) {
      if (cs) ZP_LNB(false, true, 4) else ZP_LNB(false, false, 4)
    } else {
      if (cs) ZP_LNB(false, true, 0) else ZP_LNB(false, false, 0)
    }
#undef ZP_LNB
    note_launch();
    return cudaGetLastError();
  }
  if (cs) return cudaErrorInvalidValue;
  const int grid = grid_for(rows, kThreads / 32, ctas, 8);
  if (rms)
    ln_bwd_rows_k<true><<<grid, kThreads, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h);
  else
    ln_bwd_rows_k<false><<<grid, kThreads, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h);
  note_launch();
  const int col_blocks = h / 256;
  int chunks = (ctas * 4 + col_blocks - 1) / col_blocks;
  if (chunks > 4 * 148) chunks = 4 * 148;
  const int64_t chunk = (rows + chunks - 1) / chunks;
  chunks = int((rows + chunk - 1) / chunk);
  *nblk = chunks;
  if (rms)
    ln_bwd_cols_k<true><<<dim3(col_blocks, chunks), dim3(32, 8), 0, s>>>(dy, x, mean, rstd, rows, h, chunk, part);
  else
    ln_bwd_cols_k<false><<<dim3(col_blocks, chunks), dim3(32, 8), 0, s>>>(dy, x, mean, rstd, rows, h, chunk, part);
  note_launch();
  return cudaGetLastError();
}

void cross_entropy_fwd_bwd(bf16* logits, const int32_t* tokens, int seq, int64_t rows, int vocab,
                           int ldv, float grad_scale, float* row_loss, int ctas, cudaStream_t s) {
  const size_t stride = (size_t(ldv) * 2 + 127) & ~size_t(127);
  const int nvec = ldv / 8;
  if (2 * stride <= 200 * 1024 && nvec <= 16 * kCeThreads) {
    const int grid = int(rows < ctas ? rows : ctas);
#define ZP_CE(C)                                                                                        \
  {                                                                                                     \
    static std::atomic<uint64_t> attr{0};                                                                           \
    if (first_on_device(attr)) {                                                                                        \
      cudaFuncSetAttribute(ce_reg_k<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);       \
    }                                                                                                   \
    ce_reg_k<C><<<grid, kCeThreads, 2 * stride, s>>>(logits, tokens, seq, rows, vocab, ldv, grad_scale, row_loss); \
  }
    if (nvec <= 8 * kCeThreads)
      ZP_CE(8)
    else if (nvec <= 13 * kCeThreads)
      ZP_CE(13)
    else
      ZP_CE(16)
#undef ZP_CE
    note_launch();
    return;
  }
  if (2 * stride <= 200 * 1024) {
    static std::atomic<uint64_t> attr{0};
    if (first_on_device(attr)) {
      cudaFuncSetAttribute(ce_smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    const int grid = int(rows < ctas ? rows : ctas);
    ce_smem_k<<<grid, kCeThreads, 2 * stride, s>>>(logits, tokens, seq, rows, vocab, ldv, grad_scale, row_loss);
    note_launch();
    return;
  }
  ce_k<<<grid_for(rows, 1, ctas, 8), kThreads, 0, s>>>(logits, tokens, seq, rows, vocab, ldv,
                                                      grad_scale, row_loss); note_launch();
}

void colsum_bf16(const bf16* X, int64_t rows, int N, int ld, float* work, bf16* out, int ctas,
                 cudaStream_t s, float* out32, bool acc32) {
  const int col_blocks = (N + 255) / 256;
  int chunks = (ctas * 4 + col_blocks - 1) / col_blocks;
  if (chunks < 1) chunks = 1;
  if (chunks > 256) chunks = 256;
  const int64_t chunk = (rows + chunks - 1) / chunks;
  chunks = int((rows + chunk - 1) / chunk);
  colsum_part_k<<<dim3(col_blocks, chunks), dim3(32, 8), 0, s>>>(X, rows, N, ld, chunk, work); note_launch();
  sum_partials_k<<<(N + 31) / 32, dim3(32, 32), 0, s>>>(work, chunks, N, out, out32, acc32 ? 1 : 0); note_launch();
}
void sum_partials(const float* part, int nparts, int N, bf16* out, cudaStream_t s, float* out32, bool acc32) {
  sum_partials_k<<<(N + 31) / 32, dim3(32, 32), 0, s>>>(part, nparts, N, out, out32, acc32 ? 1 : 0); note_launch();
}
void cast_f32_bf16(const float* in, bf16* out, int64_t n, int ctas, cudaStream_t s) {
  cast_k<<<grid_for(n / 4 + 1, kThreads, ctas), kThreads, 0, s>>>(in, out, n); note_launch();
}
void reduce_sum_f32(const float* x, int64_t n, float* out, cudaStream_t s) {
  reduce_sum_k<<<1, kThreads, 0, s>>>(x, n, out); note_launch();
}
void reduce_slices(float* acc, const bf16* const* srcs, int n, int64_t len, bool first, int ctas, cudaStream_t s) {
  SliceSrcs ss{};
  for (int j = 0; j < n && j < 8; ++j) ss.p[j] = srcs[j];
  reduce_slices_k<<<grid_for(len / 8, kThreads, ctas), kThreads, 0, s>>>(acc, ss, n, len, first); note_launch();
}
void add_f32(float* dst, const float* src, int64_t n, int ctas, cudaStream_t s) {
  add_f32_k<<<grid_for(n, kThreads, ctas), kThreads, 0, s>>>(dst, src, n); note_launch();
}
void accumulate_bf16(float* acc, const bf16* src, int64_t n, bool overwrite, int ctas,
                     cudaStream_t s) {
  accumulate_k<<<grid_for(n / 4, kThreads, ctas), kThreads, 0, s>>>(acc, src, n, overwrite); note_launch();
}
void adam_update(float* p32, float* m, float* v, bf16* p16, const float* acc, const bf16* g16,
                 const float* g32, int64_t n, const AdamParams& ap, int ctas, cudaStream_t s) {
  adam_k<<<grid_for(n / 4, kThreads, ctas), kThreads, 0, s>>>(p32, m, v, p16, acc, g16, g32, n, ap); note_launch();
}

}  // namespace zp
