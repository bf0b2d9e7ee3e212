// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
// One CTA per SM (grid capped by the rank's SM budget). Warp roles:
//   warp 0      : TMA producer (one elected thread), SWIZZLE_128B tiles into an S-stage ring
//   warp 1      : MMA issuer (one thread), tcgen05.mma 128xBNx16 into a double-buffered TMEM
//                 accumulator (2*BN columns)
//   warp 2      : TMEM allocator
//   warps 4..7  : epilogue, tcgen05.ld 32x32b -> registers -> fused epilogue -> global
// Pipelines: smem full/empty mbarriers (TMA <-> MMA) and TMEM full/empty mbarriers
// (MMA <-> epilogue), so the epilogue of tile i overlaps the mainloop of tile i+1.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "gemm.h"
#include "kernels.h"
#include "ptx.cuh"

namespace zp {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle span of bf16
constexpr int kThreads = 384;   // 4 control warps + 8 epilogue warps
constexpr int kEpiWarps = 8;
constexpr int kStageBufBytes = 32 * 64 * 2;  // one warp's [32 rows x 64 cols] bf16 TMA-store box

// CG = 1: one CTA per 128 x BN tile. CG = 2: a cluster pair computes a 256 x BN tile with
// tcgen05.mma.cta_group::2; each CTA stages its 128 rows of A and BN/2 rows of B.
template <int BN, int CG = 1>
struct Cfg {
  static constexpr int kATileBytes = kBM * kBK * 2;
  static constexpr int kBTileBytes = (BN / CG) * kBK * 2;
  static constexpr int kStageBytes = kATileBytes + kBTileBytes;
  static constexpr int kEpiBytes = kEpiWarps * 2 * kStageBufBytes;  // double-buffered per warp
  static constexpr int kStages = (232448 - kEpiBytes - 1024 - 512) / kStageBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024 /*align*/ + 512 /*barriers*/;
};

constexpr int kGroupM = 8;

struct TileInfo {
  int z1, z2, m0, n0, kb0, kb1;
  bool skip;
};

struct Sched {
  int m_tiles, n_tiles, nb1, total, split_k;
  int M, N, K, BN, causal, tile_m;  // tile_m = 128 * CTA-group size
  __device__ TileInfo tile(int unit) const {
    TileInfo ti;
    const int split = unit % split_k;
    const int t = unit / split_k;
    const int per_batch = m_tiles * n_tiles;
    const int z = t / per_batch;
    const int r = t - z * per_batch;
    // grouped raster: runs of kGroupM m-tiles sweep the n-tiles together, so the tiles in flight
    // at any time share a few A row-blocks and B column-blocks (L2 reuse for large N, e.g. the
    // LM head)
    const int first_m = (r / (kGroupM * n_tiles)) * kGroupM;
    const int gsize = min(kGroupM, m_tiles - first_m);
    const int rr = r - first_m * n_tiles;
    const int mb = first_m + rr % gsize;
    const int nb = rr / gsize;
    ti.z1 = z % nb1;
    ti.z2 = z / nb1;
    ti.m0 = mb * tile_m;
    ti.n0 = nb * BN;
    int kb0 = 0, kb1 = (K + kBK - 1) / kBK;
    ti.skip = false;
    if (causal == kCausalSkipUpper) {
      ti.skip = ti.n0 > ti.m0 + tile_m - 1;
    } else if (causal == kCausalKUpper) {
      const int kend = min(K, ti.m0 + tile_m);
      kb1 = (kend + kBK - 1) / kBK;
    } else if (causal == kCausalKLower) {
      kb0 = ti.m0 / kBK;
    }
    if (split_k > 1) {
      const int nk = kb1 - kb0;
      const int per = (nk + split_k - 1) / split_k;
      kb0 = kb0 + split * per;
      kb1 = min(kb1, kb0 + per);
    }
    ti.kb0 = kb0;
    ti.kb1 = kb1;
    if (kb1 <= kb0) ti.skip = true;
    return ti;
  }
};

struct EpiParams {
  void* c;
  int64_t ldc, cs1, cs2;
  float alpha;
  int epilogue;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* aux;
  __nv_bfloat16* aux_out;
  int tma_store;  // bf16 output written through swizzled smem boxes + TMA stores
  int aux_tma;      // residual / GELU-input rows loaded by TMA into the staging boxes
  int aux_out_tma;  // GELU pre-activation written by TMA stores
  float* colsum;    // += column sums of the bf16-path output over the rows (fp32 [N]); may be null
  const float2* rope_tab;  // kEpiRopeBf16: (cos, sin) [rope_seq][rope_dh / 2]
  int rope_seq, rope_dh, rope_cols;
  float* dvec;             // kEpiDvecBf16
  float* zero32;
  int dvec_seq;
};

// Column sums of one warp's 32 rows x 64 columns (v[g][i]: row = lane, column = 32g + i) added
// into colsum with one fp32 atomic per column: a butterfly transpose-reduce leaves column L's sum
// in lane L (31 shuffles per 32 columns). Destroys v.
__device__ __forceinline__ void warp_colsum_add(float (&v)[2][32], bool valid, float* colsum, int n0, int N) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    if (!valid) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[g][i] = 0.f;
    }
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool up = lane & s;
#pragma unroll
      for (int i = 0; i < s; ++i) {
        const float send = up ? v[g][i] : v[g][i + s];
        const float keep = up ? v[g][i + s] : v[g][i];
        v[g][i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    const int n = n0 + 32 * g + lane;
    if (n < N) atomicAdd(colsum + n, v[g][0]);
  }
}

// GELU (tanh form) with the MUFU tanh approximation (rel. error ~2^-11, below bf16 output
// rounding).
__device__ __forceinline__ float gelu_tanh(float x) {
#ifdef ZP_GEMM_CHEAP_GELU  // timing experiment only (wrong values)
  return 0.5f * x;
#endif
  // 0.5 x (1 + tanh(k0 (x + k1 x^3))): 3 FMUL + 2 FFMA + 1 MUFU
  constexpr float k0 = 0.7978845608028654f, k0k1 = 0.7978845608028654f * 0.044715f;
  const float t = ptx::tanh_approx(x * fmaf(k0k1, x * x, k0));
  const float hx = 0.5f * x;
  return fmaf(hx, t, hx);
}

// GELU and its derivative from one tanh: the forward epilogue stores gelu'(u) for the backward,
// whose epilogue then only multiplies (no tanh, no pre-activation reload).
__device__ __forceinline__ void gelu_tanh_and_grad(float x, float& y, float& dy) {
  constexpr float k0 = 0.7978845608028654f, k0k1 = 0.7978845608028654f * 0.044715f;
  const float x2 = x * x;
  const float t = ptx::tanh_approx(x * fmaf(k0k1, x2, k0));
  const float hx = 0.5f * x;
  y = fmaf(hx, t, hx);
  const float hd = x * fmaf(1.5f * k0k1, x2, 0.5f * k0);
  dy = fmaf(hd, fmaf(-t, t, 1.0f), fmaf(0.5f, t, 0.5f));
}

__device__ __forceinline__ float gelu_tanh_grad(float x) {
  // 0.5 (1 + t) + 0.5 x (1 - t^2) k0 (1 + 3 k1 x^2), t = tanh(k0 (x + k1 x^3))
  constexpr float k0 = 0.7978845608028654f, k0k1 = 0.7978845608028654f * 0.044715f;
  const float x2 = x * x;
  const float t = ptx::tanh_approx(x * fmaf(k0k1, x2, k0));
  const float hd = x * fmaf(1.5f * k0k1, x2, 0.5f * k0);  // 0.5 x d(inner)/dx
  return fmaf(hd, fmaf(-t, t, 1.0f), fmaf(0.5f, t, 0.5f));
}

// bf16-output epilogue math on 32 consecutive columns [n, n+32) of one row; leaves the final
// values in v. `valid` = row < M; columns >= N are computed from zeros and clipped by the store.
__device__ __forceinline__ void epi_bf16_math(const EpiParams& ep, float (&v)[32], int64_t off, int n,
                                              int N, bool valid) {
  const int e = ep.epilogue;
  const bool full = valid && (n + 32 <= N);
  if (e == kEpiStoreBf16) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= ep.alpha;
    return;
  }
  if (e == kEpiBiasBf16 || e == kEpiBiasResidBf16 || e == kEpiBiasGeluBf16) {
    if (!ep.bias) {
      // bias-free layers (Llama): residual / activation only
    } else if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        const uint4 braw = *reinterpret_cast<const uint4*>(ep.bias + n + i);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&braw);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 bf = __bfloat1622float2(b2[j]);
          v[i + 2 * j] += bf.x;
          v[i + 2 * j + 1] += bf.y;
        }
      }
    } else if (valid) {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) if (n + i < N) v[i] += __bfloat162float(ep.bias[n + i]);
    }
    if (e == kEpiBiasResidBf16) {
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const uint4 rraw = *reinterpret_cast<const uint4*>(ep.aux + off + i);
          const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rraw);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 rf = __bfloat1622float2(r2[j]);
            v[i + 2 * j] += rf.x;
            v[i + 2 * j + 1] += rf.y;
          }
        }
      } else if (valid) {
        _Pragma("unroll") for (int i = 0; i < 32; ++i) if (n + i < N) v[i] += __bfloat162float(ep.aux[off + i]);
      }
    } else if (e == kEpiBiasGeluBf16) {
      // C = gelu(u), aux_out = gelu'(u)
      float d[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) gelu_tanh_and_grad(v[i], v[i], d[i]);
      __nv_bfloat16* u = ep.aux_out + off;
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 o;
          __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
          for (int j = 0; j < 4; ++j) o2[j] = __floats2bfloat162_rn(d[i + 2 * j], d[i + 2 * j + 1]);
          *reinterpret_cast<uint4*>(u + i) = o;
        }
      } else if (valid) {
        _Pragma("unroll") for (int i = 0; i < 32; ++i) if (n + i < N) u[i] = __float2bfloat16_rn(d[i]);
      }
    }
  } else if (e == kEpiGeluBwdBf16) {
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        const uint4 uraw = *reinterpret_cast<const uint4*>(ep.aux + off + i);
        const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uraw);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 uf = __bfloat1622float2(u2[j]);
          v[i + 2 * j] *= uf.x;  // aux = gelu'(u) stored by the forward epilogue
          v[i + 2 * j + 1] *= uf.y;
        }
      }
    } else if (valid) {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) if (n + i < N) v[i] *= __bfloat162float(ep.aux[off + i]);
    }
  }
}

__device__ __forceinline__ void epi_bias(const EpiParams& ep, float (&v)[32], int n, int N, bool valid) {
  if (valid && n + 32 <= N) {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      const uint4 braw = *reinterpret_cast<const uint4*>(ep.bias + n + i);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&braw);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 bf = __bfloat1622float2(b2[j]);
        v[i + 2 * j] += bf.x;
        v[i + 2 * j + 1] += bf.y;
      }
    }
  } else if (valid) {
    _Pragma("unroll") for (int i = 0; i < 32; ++i) if (n + i < N) v[i] += __bfloat162float(ep.bias[n + i]);
  }
}

// One lane's row of a warp's [32 rows x 64 cols] bf16 staging box (SWIZZLE_128B).
__device__ __forceinline__ void stage_row_bf16(uint8_t* sb, int lane, const float (&v)[2][32]) {
  const uint32_t srow = ptx::smem_u32(sb) + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float* w = &v[j >> 2][(j & 3) * 8];
    uint32_t p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p[k]) : "f"(w[2 * k + 1]), "f"(w[2 * k]));
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(srow + ((j ^ (lane & 7)) << 4)), "r"(p[0]),
                 "r"(p[1]), "r"(p[2]), "r"(p[3])
                 : "memory");
  }
}

// Writes 32 consecutive columns [n, n+32) of one row.
__device__ __forceinline__ void epilogue_row32(const EpiParams& ep, const uint32_t (&acc)[32],
                                               int64_t off, int n, int N) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(acc[i]);
  const bool full = (n + 32 <= N);
  const int e = ep.epilogue;
  if (e == kEpiAtomicF32) {
    float* c = static_cast<float*>(ep.c) + off;
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        atomicAdd(reinterpret_cast<float4*>(c + i),
                  make_float4(ep.alpha * v[i], ep.alpha * v[i + 1], ep.alpha * v[i + 2], ep.alpha * v[i + 3]));
    } else {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) if (n + i < N) atomicAdd(c + i, ep.alpha * v[i]);
    }
    return;
  }
  if (e == kEpiStoreF32 || e == kEpiAccumF32) {
    float* c = static_cast<float*>(ep.c) + off;
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 o = make_float4(ep.alpha * v[i], ep.alpha * v[i + 1], ep.alpha * v[i + 2],
                               ep.alpha * v[i + 3]);
        if (e == kEpiAccumF32) {
          const float4 p = *reinterpret_cast<const float4*>(c + i);
          o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
        }
        *reinterpret_cast<float4*>(c + i) = o;
      }
    } else {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) if (n + i < N) {
        const float o = ep.alpha * v[i];
        c[i] = (e == kEpiAccumF32) ? c[i] + o : o;
      }
    }
    return;
  }
  // bf16 outputs, direct row stores (batched GEMMs / unaligned outputs)
  epi_bf16_math(ep, v, off, n, N, true);
  __nv_bfloat16* c = static_cast<__nv_bfloat16*>(ep.c) + off;
  if (full) {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) o2[j] = __floats2bfloat162_rn(v[i + 2 * j], v[i + 2 * j + 1]);
      *reinterpret_cast<uint4*>(c + i) = o;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (n + i < N) c[i] = __float2bfloat16_rn(v[i]);
  }
}

// kEpiSwiGluBwdBf16, one 64-column chunk of dh = features [n0, n0 + 64) of this warp's 32 rows:
// u columns [2 n0, 2 n0 + 128) arrive by TMA as two [32 x 64] boxes (box j: gate | up of features
// n0 + 32j .. +31), (dgate, dup) overwrite them in place and leave by TMA store into C. Same math as
// kernels.cu swiglu_bwd_k, from the fp32 dh instead of its bf16 copy.
__device__ __forceinline__ void swiglu_bwd_chunk(uint32_t tcol, int n0, int r0, int lane, uint8_t* stage_buf,
                                                 uint64_t* ab, uint32_t (&ph)[2], const CUtensorMap* map_u,
                                                 const CUtensorMap* map_c) {
  if (lane == 0) {
    ptx::bulk_wait_read<0>();  // the previous chunk's stores have read the boxes
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      ptx::mbar_arrive_expect_tx(&ab[j], kStageBufBytes);
      ptx::tma_load_2d(stage_buf + j * kStageBufBytes, map_u, &ab[j], 2 * n0 + 64 * j, r0);
    }
  }
  float d[2][32];
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(tcol + 32 * g, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) d[g][i] = __uint_as_float(r[i]);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    ptx::mbar_wait(&ab[j], ph[j]);
    ph[j] ^= 1;
    const uint32_t srow = ptx::smem_u32(stage_buf + j * kStageBufBytes) + lane * 128;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // 16-byte chunk k: gate features 8k..8k+7, chunk k + 4: their up
      const uint32_t ag = srow + ((k ^ (lane & 7)) << 4), au = srow + (((k + 4) ^ (lane & 7)) << 4);
      uint32_t gq[4], uq[4];
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(gq[0]), "=r"(gq[1]), "=r"(gq[2]), "=r"(gq[3]) : "r"(ag));
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(uq[0]), "=r"(uq[1]), "=r"(uq[2]), "=r"(uq[3]) : "r"(au));
      uint32_t dg[4], du[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float a2[2] = {__uint_as_float(gq[e] << 16), __uint_as_float(gq[e] & 0xffff0000u)};
        float b2[2] = {__uint_as_float(uq[e] << 16), __uint_as_float(uq[e] & 0xffff0000u)};
        float oa[2], ob[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const float dv = d[j][8 * k + 2 * e + t];
          const float sg = 1.0f / (1.0f + __expf(-a2[t]));
          ob[t] = dv * (a2[t] * sg);
          oa[t] = dv * b2[t] * sg * (1.0f + a2[t] * (1.0f - sg));
        }
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(dg[e]) : "f"(oa[1]), "f"(oa[0]));
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(du[e]) : "f"(ob[1]), "f"(ob[0]));
      }
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ag), "r"(dg[0]), "r"(dg[1]), "r"(dg[2]), "r"(dg[3]) : "memory");
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(au), "r"(du[0]), "r"(du[1]), "r"(du[2]), "r"(du[3]) : "memory");
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_2d(map_c, stage_buf + j * kStageBufBytes, 2 * n0 + 64 * j, r0);
      ptx::bulk_commit();
    }
  }
}

template <int BN, int A_MN, int B_MN, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c,
                   const __grid_constant__ CUtensorMap map_x, Sched sched, EpiParams ep) {
  using C = Cfg<BN, CG>;
  constexpr int BNL = BN / CG;  // B rows staged by this CTA
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::kStages * C::kATileBytes;
  uint8_t* smem_epi = smem + C::kStages * C::kStageBytes;  // [8 warps][2][32 x 64] bf16, SW128
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_epi + C::kEpiBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::kStages;
  uint64_t* tfull = bars + 2 * C::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* auxbar = tempty + 2;  // [8 epilogue warps][2 staging buffers]: aux tile TMA loads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(auxbar + 2 * kEpiWarps);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cr = CG == 2 ? ptx::cluster_ctarank() : 0;  // rank in the CTA pair
  const int unit0 = blockIdx.x / CG, units = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&map_a);
    ptx::tma_prefetch_desc(&map_b);
    if (ep.tma_store) ptx::tma_prefetch_desc(&map_c);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 32 * kEpiWarps * CG);
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i) ptx::mbar_init(&auxbar[i], 1);
    ptx::fence_barrier_init();
  }
  if (CG == 2) ptx::cluster_sync();  // both CTAs' barriers exist before any remote arrive / TMA
  if (warp == 2) {
    if (CG == 2)
      ptx::tmem_alloc2(tmem_slot, C::kTmemCols);
    else
      ptx::tmem_alloc(tmem_slot, C::kTmemCols);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      auto load = [&](void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
        if (CG == 2)
          ptx::tma_load_4d_2sm(dst, map, bar, c0, c1, c2, c3);
        else
          ptx::tma_load_4d(dst, map, bar, c0, c1, c2, c3);
      };
      for (int t = unit0; t < sched.total; t += units) {
        const TileInfo ti = sched.tile(t);
        if (ti.skip) continue;
        const int am = ti.m0 + int(cr) * kBM;   // this CTA's A rows
        const int bn = ti.n0 + int(cr) * BNL;   // this CTA's B rows
        for (int kb = ti.kb0; kb < ti.kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          // the leader's full barrier counts both CTAs' bytes
          if (cr == 0) ptx::mbar_arrive_expect_tx(&full[stage], CG * C::kStageBytes);
          uint8_t* sa = smem_a + stage * C::kATileBytes;
          uint8_t* sb = smem_b + stage * C::kBTileBytes;
          const int k0 = kb * kBK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < kBM / 64; ++j)
              load(sa + j * 64 * kBK * 2, &map_a, &full[stage], am + 64 * j, k0, ti.z1, ti.z2);
          } else {
            load(sa, &map_a, &full[stage], k0, am, ti.z1, ti.z2);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BNL / 64; ++j)
              load(sb + j * 64 * kBK * 2, &map_b, &full[stage], bn + 64 * j, k0, ti.z1, ti.z2);
          } else {
            load(sb, &map_b, &full[stage], k0, bn, ti.z1, ti.z2);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && cr == 0) {
      // ------------------------------------------------------------ MMA issuer (leader CTA)
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kBM * CG, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = unit0; t < sched.total; t += units) {
        const TileInfo ti = sched.tile(t);
        if (ti.skip) continue;
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = ti.kb0; kb < ti.kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem_a + stage * C::kATileBytes);
          const uint32_t sb = ptx::smem_u32(smem_b + stage * C::kBTileBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            // K-major: advance 16 elements (32 B) inside the 128 B swizzle row.
            // MN-major: advance 16 K-rows (2 x 1024 B swizzle atoms); LBO = 64-wide MN chunk.
            const uint64_t da = A_MN ? ptx::smem_desc_sw128(sa + kk * 2048, 64 * kBK * 2, 1024)
                                     : ptx::smem_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? ptx::smem_desc_sw128(sb + kk * 2048, 64 * kBK * 2, 1024)
                                     : ptx::smem_desc_sw128(sb + kk * 32, 16, 1024);
            if (CG == 2)
              ptx::umma_bf16_2sm(d_tmem, da, db, idesc, (kb > ti.kb0 || kk > 0) ? 1u : 0u);
            else
              ptx::umma_bf16(d_tmem, da, db, idesc, (kb > ti.kb0 || kk > 0) ? 1u : 0u);
          }
          if (CG == 2)
            ptx::umma_commit_pair(&empty[stage]);
          else
            ptx::umma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2)
          ptx::umma_commit_pair(&tfull[acc]);
        else
          ptx::umma_commit(&tfull[acc]);
        ++local;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (8 warps)
    // warp w reads TMEM lane quarter w % 4 (rows 32q..32q+31) and column half (w - 4) / 4.
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int cols = BN >= 128 ? BN / 2 : (half == 0 ? BN : 0);
    const int c_begin = BN >= 128 ? half * (BN / 2) : 0;
    uint8_t* stage_buf = smem_epi + (warp - 4) * 2 * kStageBufBytes;
    int buf = 0;
    uint32_t aux_ph[2] = {0, 0};  // phases of this warp's two aux-load barriers
    float dacc = 0.f;             // kEpiDvecBf16: this row's dO . O over the current head
    int local = 0;
    const uint32_t tempty_leader = CG == 2 ? ptx::mapa(ptx::smem_u32(&tempty[0]), 0) : 0;
    for (int t = unit0; t < sched.total; t += units) {
      const TileInfo ti = sched.tile(t);
      if (ti.skip) continue;
      const int acc = local & 1;
      const int mrow0 = ti.m0 + int(cr) * kBM;  // this CTA's 128 accumulator rows
      if (ep.tma_store && ep.aux_tma) {
        // prefetch this tile's aux boxes (one per 64-column chunk, box j in staging buffer j)
        // before the accumulator is ready; the previous tile's stores must have read the boxes
        if (lane == 0) {
          ptx::bulk_wait_read<0>();
          for (int j = 0; j < 2 && c_begin + 64 * j < c_begin + cols && ti.n0 + c_begin + 64 * j < sched.N; ++j) {
            uint64_t* ab = &auxbar[(warp - 4) * 2 + j];
            ptx::mbar_arrive_expect_tx(ab, kStageBufBytes);
            ptx::tma_load_2d(stage_buf + j * kStageBufBytes, &map_x, ab, ti.n0 + c_begin + 64 * j, mrow0 + q * 32);
          }
        }
      }
      ptx::mbar_wait(&tfull[acc], (local >> 1) & 1);
      ptx::tc_fence_after();
      const int row = mrow0 + q * 32 + lane;
      const bool valid = row < sched.M;
      const int64_t row_off = ti.z1 * ep.cs1 + ti.z2 * ep.cs2 + int64_t(row) * ep.ldc;
      const uint32_t tbase = tmem_base + acc * BN + (uint32_t(q * 32) << 16);
#pragma unroll 1
      for (int c = c_begin; c < c_begin + cols && ti.n0 + c < sched.N; c += 64) {
        if (ep.epilogue == kEpiSwiGluBwdBf16) {
          swiglu_bwd_chunk(tbase + c, ti.n0 + c, mrow0 + q * 32, lane, stage_buf, &auxbar[(warp - 4) * 2], aux_ph,
                           &map_x, &map_c);
          continue;
        }
        if (ep.tma_store) {
          float v[2][32];
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(tbase + c + 32 * g, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[g][i] = __uint_as_float(r[i]);
          }
          const int n0 = ti.n0 + c, r0 = mrow0 + q * 32;
          if (ep.aux_tma) {
            // aux rows (residual / GELU input) arrive by TMA into this warp's staging box
            // instead of 32 uncoalesced per-row loads; bias and GELU' applied in registers
            const int j = (c - c_begin) >> 6;  // chunk index == staging box of its prefetched aux
            buf = j;
            uint8_t* sb = stage_buf + j * kStageBufBytes;
            uint64_t* ab = &auxbar[(warp - 4) * 2 + j];
            ptx::mbar_wait(ab, aux_ph[j]);
            aux_ph[j] ^= 1;
            const uint32_t srow = ptx::smem_u32(sb) + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint32_t p[4];
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3])
                           : "r"(srow + ((j ^ (lane & 7)) << 4)));
              float* w = &v[j >> 2][(j & 3) * 8];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float a0 = __uint_as_float(p[k] << 16), a1 = __uint_as_float(p[k] & 0xffff0000u);
                if (ep.epilogue == kEpiGeluBwdBf16) {  // aux = gelu'(u)
                  w[2 * k] *= a0;
                  w[2 * k + 1] *= a1;
                } else if (ep.epilogue == kEpiDvecBf16) {  // aux = O: D += bf16(dO) * O
                  uint32_t pk;
                  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk) : "f"(w[2 * k + 1]), "f"(w[2 * k]));
                  dacc = fmaf(__uint_as_float(pk << 16), a0, dacc);
                  dacc = fmaf(__uint_as_float(pk & 0xffff0000u), a1, dacc);
                } else {  // residual
                  w[2 * k] += a0;
                  w[2 * k + 1] += a1;
                }
              }
            }
            __syncwarp();  // every lane has read the aux box before it is overwritten
            if (ep.epilogue == kEpiDvecBf16) {
              // this warp's column half is one head (128 columns): D after its second chunk; the
              // chunk's fp32 dQ workspace is cleared for the attention backward's reductions
              if (valid) {
                float4* zr = reinterpret_cast<float4*>(ep.zero32 + int64_t(row) * ep.ldc + n0);
#pragma unroll
                for (int i = 0; i < 16; ++i) zr[i] = make_float4(0.f, 0.f, 0.f, 0.f);
              }
              if (c == c_begin + 64) {
                if (valid) {
                  const int heads = sched.N >> 7, head = n0 >> 7;
                  const int smp = row / ep.dvec_seq, qi = row - smp * ep.dvec_seq;
                  ep.dvec[(int64_t(smp) * heads + head) * ep.dvec_seq + qi] = dacc;
                }
                dacc = 0.f;
              }
            }
            if (ep.epilogue == kEpiBiasResidBf16 && ep.bias) {
#pragma unroll
              for (int g = 0; g < 2; ++g) epi_bias(ep, v[g], n0 + 32 * g, sched.N, valid);
            }
          } else if (ep.epilogue == kEpiBiasGeluBf16 && ep.aux_out_tma) {
            // C = gelu(u); gelu'(u) -> staging box -> TMA store into aux_out
            float d[2][32];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              epi_bias(ep, v[g], n0 + 32 * g, sched.N, valid);
#pragma unroll
              for (int i = 0; i < 32; ++i) gelu_tanh_and_grad(v[g][i], v[g][i], d[g][i]);
            }
            if (lane == 0) ptx::bulk_wait_read<1>();
            __syncwarp();
            uint8_t* sb = stage_buf + buf * kStageBufBytes;
            stage_row_bf16(sb, lane, d);
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_2d(&map_x, sb, n0, r0);
              ptx::bulk_commit();
            }
            buf ^= 1;
          } else if (ep.epilogue == kEpiSwiGluBf16) {
            // 64-column chunk = 32 gate + 32 up columns of 32 features: h = silu(gate) * up,
            // written straight from registers (64 contiguous bytes per row)
            if (valid && n0 < sched.N) {
              __nv_bfloat16* hrow = ep.aux_out + int64_t(row) * (ep.ldc / 2) + n0 / 2;
#pragma unroll
              for (int i = 0; i < 32; i += 8) {
                uint32_t p[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const float g0 = v[0][i + 2 * k], g1 = v[0][i + 2 * k + 1];
                  const float h0 = g0 / (1.f + __expf(-g0)) * v[1][i + 2 * k];
                  const float h1 = g1 / (1.f + __expf(-g1)) * v[1][i + 2 * k + 1];
                  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p[k]) : "f"(h1), "f"(h0));
                }
                *reinterpret_cast<uint4*>(hrow + i) = make_uint4(p[0], p[1], p[2], p[3]);
              }
            }
          } else if (ep.epilogue == kEpiRopeBf16) {
            // rotary embedding of the Q / K columns on the fp32 accumulators (one bf16 rounding):
            // the partner column j +- dh/2 of the same head is re-read from TMEM (the tile is
            // aligned to heads). Warp-uniform branches only: tcgen05.ld is warp-collective.
            const int halfd = ep.rope_dh >> 1;
            const int pos = row % ep.rope_seq;
#pragma unroll 1
            for (int g = 0; g < 2; ++g) {
              const int n = n0 + 32 * g;
              if (n >= ep.rope_cols) continue;
              const int j = n % ep.rope_dh;
              const bool lo = j < halfd;
              uint32_t pr[32];
              ptx::tmem_ld_32x32b_x32(tbase + c + 32 * g + (lo ? halfd : -halfd), pr);
              ptx::tmem_ld_wait();
              const float4* cs = reinterpret_cast<const float4*>(ep.rope_tab + int64_t(pos) * halfd + (j % halfd));
              const float sg = lo ? -1.f : 1.f;  // lo: a cos - b sin ; hi: b cos + a sin
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float4 w = cs[i >> 1];  // (cos, sin) of frequencies f + i, f + i + 1
                v[g][i] = fmaf(sg * w.y, __uint_as_float(pr[i]), v[g][i] * w.x);
                v[g][i + 1] = fmaf(sg * w.w, __uint_as_float(pr[i + 1]), v[g][i + 1] * w.z);
              }
            }
          } else {
#pragma unroll
            for (int g = 0; g < 2; ++g) epi_bf16_math(ep, v[g], row_off + n0 + 32 * g, n0 + 32 * g, sched.N, valid);
          }
          // this warp's staging box was last handed to TMA two bulk groups ago: wait until read
          if (lane == 0) ptx::bulk_wait_read<1>();
          __syncwarp();
          uint8_t* sb = stage_buf + buf * kStageBufBytes;
          stage_row_bf16(sb, lane, v);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(&map_c, sb, n0, r0);
            ptx::bulk_commit();
          }
          buf ^= 1;
          if (ep.colsum) warp_colsum_add(v, valid, ep.colsum, n0, sched.N);
        } else {
#pragma unroll 1
          for (int g = 0; g < 2; ++g) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(tbase + c + 32 * g, r);
            ptx::tmem_ld_wait();
            const int n = ti.n0 + c + 32 * g;
            if (valid && n < sched.N) epilogue_row32(ep, r, row_off + n, n, sched.N);
          }
        }
      }
      ptx::tc_fence_before();
      if (CG == 2)
        ptx::mbar_arrive_cluster(tempty_leader + acc * 8);  // the leader's MMA reuses this TMEM
      else
        ptx::mbar_arrive(&tempty[acc]);
      ++local;
    }
    if (ep.tma_store && lane == 0) ptx::bulk_wait<0>();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (CG == 2) ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    if (CG == 2)
      ptx::tmem_dealloc2(tmem_base, C::kTmemCols);
    else
      ptx::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ------------------------------------------------------------------ host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// rows x inner matrix (inner contiguous), plus two batch dims; box = {64, box_rows}.
bool make_map(CUtensorMap* map, const GemmOperand& op, int64_t inner, int64_t rows, int nb1,
              int nb2, int box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(nb1), cuuint64_t(nb2)};
  // Strides for dims 1..3 in bytes; batch strides of size-1 dims must still be valid.
  const int64_t row_bytes = op.ld * 2;
  const int64_t s1 = (nb1 > 1 ? op.bs1 : rows * op.ld) * 2;
  const int64_t s2 = (nb2 > 1 ? op.bs2 : s1 * nb1 / 2) * 2;
  cuuint64_t strides[3] = {cuuint64_t(row_bytes), cuuint64_t(s1), cuuint64_t(s2)};
  cuuint32_t box[4] = {64, cuuint32_t(box_rows), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(op.ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Output map: [M rows, N cols] bf16 with row stride ldc; box = 64 cols x 32 rows, SWIZZLE_128B
// (matches the epilogue warps' staging layout).
bool make_store_map(CUtensorMap* map, void* c, int64_t M, int64_t N, int64_t ldc) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc || (ldc * 2) % 16) return false;
  cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(M)};
  cuuint64_t strides[1] = {cuuint64_t(ldc * 2)};
  cuuint32_t box[2] = {64, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN, int A_MN, int B_MN, int CG>
cudaError_t launch(const GemmArgs& a, cudaStream_t stream) {
  using C = Cfg<BN, CG>;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, CG>;
  static std::atomic<uint64_t> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    if (CG == 2) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
      (void)e;
    }
  }
  CUtensorMap ma, mb, mc;
  const bool ok_a = A_MN ? make_map(&ma, a.a, a.M, a.K, a.nb1, a.nb2, 64)
                         : make_map(&ma, a.a, a.K, a.M, a.nb1, a.nb2, kBM);
  const bool ok_b = B_MN ? make_map(&mb, a.b, a.N, a.K, a.nb1, a.nb2, 64)
                         : make_map(&mb, a.b, a.K, a.N, a.nb1, a.nb2, BN / CG);
  if (!ok_a || !ok_b) return cudaErrorInvalidValue;
  // bf16 outputs of plain (unbatched) GEMMs go through TMA stores.
  const bool bf16_out = a.epilogue == kEpiStoreBf16 || a.epilogue == kEpiBiasBf16 ||
                        a.epilogue == kEpiBiasResidBf16 || a.epilogue == kEpiBiasGeluBf16 ||
                        a.epilogue == kEpiGeluBwdBf16 || a.epilogue == kEpiSwiGluBf16 || a.epilogue == kEpiRopeBf16 ||
                        a.epilogue == kEpiDvecBf16;
  if (a.epilogue == kEpiSwiGluBf16 && (a.N % 64 || !a.aux_out || a.nb1 != 1 || a.nb2 != 1))
    return cudaErrorInvalidValue;
  bool tma_store = bf16_out && a.nb1 == 1 && a.nb2 == 1 && (reinterpret_cast<uintptr_t>(a.c) % 16) == 0;
  if (tma_store) tma_store = make_store_map(&mc, a.c, a.M, a.N, a.ldc);
  if (a.epilogue == kEpiSwiGluBf16 && !tma_store) return cudaErrorInvalidValue;
  if (a.epilogue == kEpiSwiGluBwdBf16) {
    // C and aux are [M, 2N] (row stride ldc); the accumulator (dh) itself is never stored
    if (a.N % 64 || !a.aux || a.nb1 != 1 || a.nb2 != 1 || a.alpha != 1.0f || a.colsum ||
        (reinterpret_cast<uintptr_t>(a.c) % 16) || (reinterpret_cast<uintptr_t>(a.aux) % 16) ||
        !make_store_map(&mc, a.c, a.M, 2 * int64_t(a.N), a.ldc))
      return cudaErrorInvalidValue;
    tma_store = true;
  }
  if (a.epilogue == kEpiRopeBf16 &&
      (!tma_store || !a.rope_tab || a.rope_seq < 1 || (a.rope_dh != 64 && a.rope_dh != 128) || BN % a.rope_dh ||
       a.rope_cols % a.rope_dh || a.alpha != 1.0f || (reinterpret_cast<uintptr_t>(a.rope_tab) % 16)))
    return cudaErrorInvalidValue;
  if (a.colsum && !tma_store) return cudaErrorInvalidValue;
  if (!tma_store) mc = ma;  // unused placeholder
  // aux tiles share C's layout (ldc): residual / GELU input loaded, pre-activation stored by TMA
  CUtensorMap mx = mc;
  bool aux_tma = false, aux_out_tma = false;
  if (a.epilogue == kEpiSwiGluBwdBf16 && !make_store_map(&mx, const_cast<void*>(a.aux), a.M, 2 * int64_t(a.N), a.ldc))
    return cudaErrorInvalidValue;  // u: loaded box by box inside the epilogue (no prefetch)
  if (tma_store && (a.epilogue == kEpiBiasResidBf16 || a.epilogue == kEpiGeluBwdBf16 || a.epilogue == kEpiDvecBf16) &&
      a.aux && (reinterpret_cast<uintptr_t>(a.aux) % 16) == 0)
    aux_tma = make_store_map(&mx, const_cast<void*>(a.aux), a.M, a.N, a.ldc);
  if (a.epilogue == kEpiDvecBf16 &&
      (!aux_tma || BN != 256 || a.N % 256 || !a.dvec || !a.zero32 || a.dvec_seq < 1 || a.alpha != 1.0f ||
       a.colsum || (reinterpret_cast<uintptr_t>(a.zero32) % 16)))
    return cudaErrorInvalidValue;
  if (tma_store && a.epilogue == kEpiBiasGeluBf16 && a.aux_out && (reinterpret_cast<uintptr_t>(a.aux_out) % 16) == 0)
    aux_out_tma = make_store_map(&mx, a.aux_out, a.M, a.N, a.ldc);
  Sched s;
  s.tile_m = kBM * CG;
  s.m_tiles = (a.M + s.tile_m - 1) / s.tile_m;
  s.n_tiles = (a.N + BN - 1) / BN;
  s.nb1 = a.nb1;
  int ctas = num_sms();
  if (a.max_ctas > 0 && a.max_ctas < ctas) ctas = a.max_ctas;
  const int workers = ctas / CG;  // persistent CTAs (pairs)
  const int tiles = s.m_tiles * s.n_tiles * a.nb1 * a.nb2;
  s.split_k = a.split_k > 1 ? a.split_k : 1;
  if (a.split_k < 0) {
    // auto split-K: the split count whose work units fill the persistent CTAs in the fewest,
    // fullest waves (ties to the smaller split), keeping >= 8 k-blocks per unit
    const int kblocks = (a.K + kBK - 1) / kBK;
    const int max_split = kblocks / 8 < 64 ? kblocks / 8 : 64;
    double best = -1.0;
    for (int sp = 1; sp <= max_split; ++sp) {
      const int u = tiles * sp;
      const int waves = (u + workers - 1) / workers;
      // efficiency of the last wave, discounted by a small per-split atomic overhead
      const double eff = double(u) / double(waves * workers) - 0.004 * sp;
      if (eff > best + 1e-9) {
        best = eff;
        s.split_k = sp;
      }
    }
  }
  if (s.split_k > 1 && a.epilogue != kEpiAtomicF32) return cudaErrorInvalidValue;
  s.total = tiles * s.split_k;
  s.M = a.M;
  s.N = a.N;
  s.K = a.K;
  s.BN = BN;
  s.causal = a.causal;
  EpiParams ep;
  ep.c = a.c;
  ep.ldc = a.ldc;
  ep.cs1 = a.cs1;
  ep.cs2 = a.cs2;
  ep.alpha = a.alpha;
  ep.epilogue = a.epilogue;
  ep.bias = static_cast<const __nv_bfloat16*>(a.bias);
  ep.aux = static_cast<const __nv_bfloat16*>(a.aux);
  ep.aux_out = static_cast<__nv_bfloat16*>(a.aux_out);
  ep.tma_store = tma_store ? 1 : 0;
  ep.aux_tma = aux_tma ? 1 : 0;
  ep.aux_out_tma = aux_out_tma ? 1 : 0;
  ep.colsum = a.colsum;
  ep.rope_tab = static_cast<const float2*>(a.rope_tab);
  ep.rope_seq = a.rope_seq;
  ep.rope_dh = a.rope_dh;
  ep.rope_cols = a.rope_cols;
  ep.dvec = a.dvec;
  ep.zero32 = a.zero32;
  ep.dvec_seq = a.dvec_seq;
  int units = workers;
  if (s.total < units) units = s.total;
  if (units < 1) return cudaSuccess;
  if (CG == 1) {
    kern<<<units, kThreads, C::kSmemBytes, stream>>>(ma, mb, mc, mx, s, ep);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units * CG);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mx, s, ep);
    if (e != cudaSuccess) return e;
  }
  note_launch();
  return cudaGetLastError();
}

// CTA pairs (2-SM MMA, M = 256) for plain GEMMs with enough rows and N >= 128; single CTAs
// otherwise. ZP_GEMM_PAIRS=0 forces single-CTA tiles.
bool use_pairs(const GemmArgs& a, int BN) {
  static int env = -1;
  if (env < 0) {
    const char* v = getenv("ZP_GEMM_PAIRS");
    env = (v && v[0] == '0') ? 0 : 1;
  }
  return env == 1 && BN >= 128 && a.M >= 256 && a.nb1 == 1 && a.nb2 == 1 && a.causal == kCausalNone &&
         (a.max_ctas == 0 || a.max_ctas >= 2);
}

template <int BN>
cudaError_t dispatch_major(const GemmArgs& a, cudaStream_t s) {
  if (use_pairs(a, BN)) {
    if (a.a.major == kKMajor && a.b.major == kKMajor) return launch<BN, 0, 0, 2>(a, s);
    if (a.a.major == kKMajor && a.b.major == kMNMajor) return launch<BN, 0, 1, 2>(a, s);
    if (a.a.major == kMNMajor && a.b.major == kKMajor) return launch<BN, 1, 0, 2>(a, s);
    return launch<BN, 1, 1, 2>(a, s);
  }
  if (a.a.major == kKMajor && a.b.major == kKMajor) return launch<BN, 0, 0, 1>(a, s);
  if (a.a.major == kKMajor && a.b.major == kMNMajor) return launch<BN, 0, 1, 1>(a, s);
  if (a.a.major == kMNMajor && a.b.major == kKMajor) return launch<BN, 1, 0, 1>(a, s);
  return launch<BN, 1, 1, 1>(a, s);
}

}  // namespace

cudaError_t gemm(const GemmArgs& a, cudaStream_t stream) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.nb1 <= 0 || a.nb2 <= 0) return cudaErrorInvalidValue;
  if ((a.a.ld % 8) || (a.b.ld % 8) || (a.ldc % 8)) return cudaErrorInvalidValue;
  if (a.N <= 64) return dispatch_major<64>(a, stream);
  if (a.N <= 128) return dispatch_major<128>(a, stream);
  return dispatch_major<256>(a, stream);
}

}  // namespace zp
