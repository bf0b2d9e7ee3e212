// Fused causal attention on sm_100a tensor cores (tcgen05 + TMEM + TMA); the s x s scores never
// reach HBM. Four kernels:
//
// head_dim 64  forward  (attn_fwd_kernel): two independent pipelines per CTA (8 softmax warps, a
//              TMA warp and an MMA warp each, 256 TMEM columns each): S = Q K^T -> TMEM, the softmax
//              warps write P (bf16) back into TMEM, O += P V with P as the TMEM A operand, O resident
//              in TMEM with a lazy (> 2^8) rescale.
// head_dim 64  backward (attn_bwd_kernel): transposed, one CTA task per 128-key tile: S^T = K Q^T
//              and dP^T = V dO^T -> TMEM, 8 builder warps form P^T and dS'^T into TMEM (dV, dK take
//              them as TMEM A operands) and dS'^T into shared memory for dQ = dS' K, which four warps
//              add into an fp32 dQ with TMA bulk reduce-add; separate score / gradient MMA warps.
// head_dim 128 forward  (attn_fwd_d128_kernel): two query tiles per CTA share every K/V tile and
//              ping-pong their softmax warp groups with one MMA warp; P overwrites S in TMEM.
// head_dim 128 backward (attn_bwd_d128_kernel): the transposed scheme with every TMEM region
//              reused in place (S^T -> P^T, dP^T -> dS'^T -> dQ^T), dQ added with fp32 reductions
//              straight from registers, see the kernel's comment.
// Plus D = rowsum(dO * O) (attn_dvec_kernel) and the fp32 dQ -> bf16 cast (attn_dq_cast_kernel).
#include <cmath>
#include <cstdlib>

#include "attention.h"
#include "kernels.h"
#include "ptx.cuh"

namespace zp {
namespace {


constexpr int kT = 128;          // query / key tile
constexpr int kD = 64;           // head dim
constexpr int kTile = kT * kD * 2;  // one [128, 64] bf16 tile = 16 KiB
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// K-major SWIZZLE_128B operand: 128 rows x 64 elements, k16 step = +32 B.
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int k16) {
  return ptx::smem_desc_sw128(base + k16 * 32, 16, 1024);
}
// K-major operand made of two 64-wide K blocks (a [128, 128] tile): k16 steps 0..7.
__device__ __forceinline__ uint64_t kdesc2(uint32_t base, int k16) {
  return ptx::smem_desc_sw128(base + (k16 >> 2) * kTile + (k16 & 3) * 32, 16, 1024);
}
// MN-major operand whose K index runs over the 128 rows of a tile: k16 step = +2048 B; the
// MN extent is split into 64-wide chunks kTile apart.
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int k16) {
  return ptx::smem_desc_sw128(base + k16 * 2048, kTile, 1024);
}

// Byte offset of element (row r, col k) in a [128, 128] bf16 tile stored as two K-major
// SWIZZLE_128B [128, 64] blocks. Writes 8 consecutive columns (one 16-byte chunk) per call.
__device__ __forceinline__ uint32_t p_off(int r, int k) {
  const int blk = k >> 6, chunk = (k & 63) >> 3;
  return blk * kTile + r * 128 + ((chunk ^ (r & 7)) << 4);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {  // a -> low half, b -> high half
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

struct AttnTask {
  int tile, z;  // tile index (query tile in fwd, key tile in bwd) and z = sample * H + head
};

// Dynamic task scheduling. Forward tasks are numbered in groups of kGroupZ (sample, head) pairs;
// within a group the longest tiles come first (forward query tile qt needs qt+1 key tiles, backward key
// tile kt needs nt-kt query tiles). CTAs grab task numbers from a global counter, so the tiles
// of a few (sample, head) pairs are in flight together (their K/V, resp. Q/dO, tiles are read
// from HBM once and served from L2) and the longest-first order balances the CTAs.
constexpr int kGroupZ = 16;
__device__ unsigned int g_sched[4];  // [fwd counter, fwd done, bwd counter, bwd done]

__device__ __forceinline__ AttnTask group_task(int t, int nz, int nt, bool longest_is_last_tile,
                                              int group = kGroupZ) {
  const int per = group * nt;
  const int g = t / per;
  const int rem = t - g * per;
  const int gz = min(group, nz - g * group);
  const int rank = rem / gz;  // 0 = longest
  return {longest_is_last_tile ? nt - 1 - rank : rank, g * group + rem % gz};
}
__device__ __forceinline__ AttnTask fwd_task(int t, int nz, int nt) { return group_task(t, nz, nt, true); }
// Backward: static round-robin, tile-major (longest key tiles first) over all (sample, head)
// pairs: concurrent key tiles of the same (sample, head) would contend on the same dQ rows'
// atomics.
__device__ __forceinline__ AttnTask bwd_task_static(int t, int nz) { return {t / nz, t % nz}; }

__device__ __forceinline__ int lds_s32(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ float lds_f32(const float* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(ptx::smem_u32(p)) : "memory");
  return v;
}
// Four consecutive floats; one wavefront when the whole warp reads the same address (broadcast).
__device__ __forceinline__ float4 lds_v4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(ptx::smem_u32(p)));
  return v;
}
__device__ __forceinline__ void red_add_v2_f32(float* p, float a, float b) {  // p 8-byte aligned
  asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_f32(float* p, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(ptx::smem_u32(p)), "f"(v) : "memory");
}

// Four-slot ring carrying the grabbed task numbers from the producer to the other warp roles.
struct TaskRing {
  int* slot;        // [4]
  uint64_t* full;   // [4], count 1 (producer)
  uint64_t* empty;  // [4], count = number of consumer warps
  // producer: next task number (>= ntasks when the launch is exhausted; consumers see it too)
  __device__ int produce(uint32_t item, unsigned int* ctr) const {
    const int k = item & 3;
    ptx::mbar_wait(&empty[k], ((item >> 2) & 1) ^ 1);
    const int t = int(atomicAdd(ctr, 1u));
    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(ptx::smem_u32(&slot[k])), "r"(t) : "memory");
    ptx::mbar_arrive(&full[k]);
    return t;
  }
  // consumer warp (all lanes call): the item's task number; lane 0 releases the slot
  __device__ int consume(uint32_t item) const {
    const int k = item & 3;
    ptx::mbar_wait(&full[k], (item >> 2) & 1);
    const int t = lds_s32(&slot[k]);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&empty[k]);
    return t;
  }
  // single-thread consumer
  __device__ int consume1(uint32_t item) const {
    const int k = item & 3;
    ptx::mbar_wait(&full[k], (item >> 2) & 1);
    const int t = lds_s32(&slot[k]);
    ptx::mbar_arrive(&empty[k]);
    return t;
  }
};

// Called once per CTA by the producer after its last grab: the last CTA resets the counter for
// the next launch on the stream.
__device__ __forceinline__ void sched_finish(unsigned int* sched, unsigned int producers_per_cta) {
  __threadfence();
  if (atomicAdd(&sched[1], 1u) == gridDim.x * producers_per_cta - 1) {
    atomicExch(&sched[0], 0u);
    atomicExch(&sched[1], 0u);
  }
}

// ============================================================================ forward
// One CTA per SM running two independent pipelines (warps 10p .. 10p+9 for pipeline p), each
// with its own tasks, shared-memory stages, barriers and 256 TMEM columns: warps 0-7 softmax
// (TMEM lane quarter w % 4, key half w / 4), warp 8 TMA producer, warp 9 MMA issuer. TMEM per
// pipeline: S [0,128), P [128,192) as packed bf16 pairs, O [192,256). S = Q K^T lands in TMEM; the softmax warps read it, write P back into TMEM
// (tcgen05.st) and the MMA warp accumulates O += P V with P as a TMEM operand. O stays in TMEM
// for the whole query tile; the max used for the exponentials is only raised when the row max
// grows by more than 2^8 (lazy rescale of O and the row sum, in place). The two pipelines
// overlap one's softmax with the other's MMAs and barrier waits.
constexpr int kFwdPipes = 2;
constexpr int kFwdThreads = 320 * kFwdPipes;
constexpr int kFwdProducer = 8, kFwdMma = 9;
constexpr int kFwdKV = 2;              // K/V stages
constexpr float kRescaleLog2 = 8.0f;   // rescale O only when the max grows by more than 2^8
constexpr int kFwdTmemS = 0, kFwdTmemP = 128, kFwdTmemO = 192;

struct FwdSmem {
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;                // kFwdKV stages
  static constexpr int kV = kK + kFwdKV * kTile;       // kFwdKV stages
  static constexpr int kRed = kV + kFwdKV * kTile;     // [2 halves][128 rows] fp32 exchange
  static constexpr int kBar = kRed + 2 * 128 * 4;
  static constexpr int kPipe = (kBar + 256 + 1023) / 1024 * 1024;  // one pipeline (1 KiB multiple)
  static constexpr int kBytes = kFwdPipes * kPipe + 1024;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (the MUFU unit, 16 results/clk/SM, bounds the softmax): round-to-nearest
// split x = j + f with the 1.5*2^23 trick, cubic minimax for 2^f on [-0.5, 0.5] (max rel. error
// 7.5e-5, below bf16 resolution), 2^j added into the exponent bits. x is clamped to >= -126 so
// the exponent arithmetic cannot wrap (results there are ~1e-38, i.e. 0 for all uses here).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.055171647f, 0.24261112f);
  p = fmaf(p, f, 0.69326099f);
  p = fmaf(p, f, 0.99992807f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

static_assert(FwdSmem::kPipe % 1024 == 0, "pipeline regions keep the 1 KiB swizzle alignment");

__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap map_qkv, bf16* __restrict__ out,
                    float* __restrict__ lse, int seq, int heads, int nz, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  const int pipe = int(ptx::warp_id()) / 10;
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023)) +
                pipe * FwdSmem::kPipe;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + FwdSmem::kBar);
  uint64_t* q_full = bar + 0;
  uint64_t* q_empty = bar + 1;
  uint64_t* kv_full = bar + 2;            // [kFwdKV]
  uint64_t* kv_empty = bar + 2 + kFwdKV;  // [kFwdKV]
  uint64_t* s_full = bar + 2 + 2 * kFwdKV;  // S ready (MMA -> softmax)
  uint64_t* s_free = s_full + 1;   // S read out (softmax -> MMA)
  uint64_t* p_full = s_full + 2;   // P written to TMEM, O rescaled (softmax -> MMA)
  uint64_t* pv_done = s_full + 3;  // P.V complete: P free, O updated (MMA -> softmax)
  uint64_t* o_free = s_full + 4;   // O read out by the epilogue (softmax -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 5);
  const TaskRing ring{reinterpret_cast<int*>(s_full + 6), s_full + 8, s_full + 12};

  const int warp = int(ptx::warp_id()) % 10;  // role within the pipeline
  const int lane = threadIdx.x & 31;
  const int nt = seq / kT;
  const int ntasks = nt * nz;
  const int h = heads * kD;

  if (warp == kFwdProducer && lane == 0) {
    ptx::tma_prefetch_desc(&map_qkv);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int i = 0; i < kFwdKV; ++i) {
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_free, 256);
    ptx::mbar_init(p_full, 256);
    ptx::mbar_init(pv_done, 1);
    ptx::mbar_init(o_free, 256);
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&ring.full[i], 1);
      ptx::mbar_init(&ring.empty[i], 9);  // MMA thread + 8 softmax warps
    }
    ptx::fence_barrier_init();
  }
  uint32_t* tmem_slot0 = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(tmem_slot) - pipe * FwdSmem::kPipe);
  if (pipe == 0 && warp == kFwdProducer) ptx::tmem_alloc(tmem_slot0, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot0 + 256 * pipe;

  if (warp == kFwdProducer) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t item = 0;; ++item) {
        const int t = ring.produce(item, &g_sched[0]);
        if (t >= ntasks) break;
        const AttnTask tk = fwd_task(t, nz, nt);
        const int smp = tk.z / heads, head = tk.z % heads;
        const int row0 = smp * seq;
        ptx::mbar_wait(q_empty, (item & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(q_full, kTile);
        ptx::tma_load_4d(sm + FwdSmem::kQ, &map_qkv, q_full, head * kD, row0 + tk.tile * kT, 0, 0);
        for (int j = 0; j <= tk.tile; ++j) {
          ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&kv_full[stage], 2 * kTile);
          ptx::tma_load_4d(sm + FwdSmem::kK + stage * kTile, &map_qkv, &kv_full[stage], h + head * kD,
                           row0 + j * kT, 0, 0);
          ptx::tma_load_4d(sm + FwdSmem::kV + stage * kTile, &map_qkv, &kv_full[stage], 2 * h + head * kD,
                           row0 + j * kT, 0, 0);
          if (++stage == kFwdKV) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      sched_finish(&g_sched[0], kFwdPipes);
    }
  } else if (warp == kFwdMma) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      // Per task: S(0); then for each j: S(j+1) (after the softmax has read S(j)), P.V(j).
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t id_o = ptx::idesc_bf16_f32(128, 64, 0, 1);
      const uint32_t sq = ptx::smem_u32(sm + FwdSmem::kQ);
      int ks = 0, kp = 0;  // K/V stage of the next S issue and of the next P.V issue
      uint32_t ks_ph = 0;
      uint32_t gs = 0, gp = 0;  // S and P.V issues so far (barrier phases)
      auto issue_s = [&]() {
        ptx::mbar_wait(&kv_full[ks], ks_ph);
        ptx::mbar_wait(s_free, (gs & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t sk = ptx::smem_u32(sm + FwdSmem::kK + ks * kTile);
#pragma unroll
        for (int k = 0; k < 4; ++k) ptx::umma_bf16(tmem + kFwdTmemS, kdesc(sq, k), kdesc(sk, k), id_s, k > 0);
        ptx::umma_commit(s_full);
        if (++ks == kFwdKV) {
          ks = 0;
          ks_ph ^= 1;
        }
        ++gs;
      };
      for (uint32_t item = 0;; ++item) {
        const int t = ring.consume1(item);
        if (t >= ntasks) break;
        const AttnTask tk = fwd_task(t, nz, nt);
        const int nj = tk.tile + 1;
        ptx::mbar_wait(q_full, item & 1);
        issue_s();
        for (int j = 0; j < nj; ++j) {
          if (j + 1 < nj) {
            issue_s();
            if (j + 2 == nj) ptx::umma_commit(q_empty);  // the task's last S has been issued
          } else if (nj == 1) {
            ptx::umma_commit(q_empty);
          }
          if (j == 0) ptx::mbar_wait(o_free, (item & 1) ^ 1);  // previous task's epilogue read O
          ptx::mbar_wait(p_full, gp & 1);
          ptx::tc_fence_after();
          const uint32_t sv = ptx::smem_u32(sm + FwdSmem::kV + kp * kTile);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::umma_bf16_ts(tmem + kFwdTmemO, tmem + kFwdTmemP + 8 * k, mndesc(sv, k), id_o, (j > 0 || k > 0));
          ptx::umma_commit(pv_done);
          ptx::umma_commit(&kv_empty[kp]);
          if (++kp == kFwdKV) kp = 0;
          ++gp;
        }
      }
    }
  } else {  // -------------------------------------------------------------- softmax warps 0-7
    // Warp (q4, kh) owns query rows 32*q4..+31, keys 64*kh..+63 of every S tile (P columns
    // 32*kh..+31) and O columns 32*kh..+31. The two halves of a row exchange their maxima and
    // row sums through shared memory.
    // a warp may only touch the TMEM lane quarter (hardware warp index % 4)
    const int q4 = int(ptx::warp_id()) & 3, kh = warp >> 2;
    const int nb = 1 + 4 * pipe + q4;  // named barrier of the row quarter's two halves
    const int r = q4 * 32 + lane;  // query row within the tile == TMEM lane
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    float* red = reinterpret_cast<float*>(sm + FwdSmem::kRed);  // [2][128]
    const uint32_t t_s = tmem + kFwdTmemS + lane_off + kh * 64;
    const uint32_t t_p = tmem + kFwdTmemP + lane_off + kh * 32;
    const uint32_t t_o = tmem + kFwdTmemO + lane_off + kh * 32;
    uint32_t g = 0;  // tiles processed (S / P.V barrier phases)
    for (uint32_t item = 0;; ++item) {
      const int t = ring.consume(item);
      if (t >= ntasks) break;
      const AttnTask tk = fwd_task(t, nz, nt);
      const int smp = tk.z / heads, head = tk.z % heads;
      float m = -INFINITY, l = 0.f;  // m: max used for the exponentials (log2 domain)
      for (int j = 0; j <= tk.tile; ++j, ++g) {
        ptx::mbar_wait(s_full, g & 1);
        ptx::tc_fence_after();
        float sv[64];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(t_s + c * 32, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(v[i]);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(s_free);
        if (j == tk.tile) {  // diagonal tile: key > query is masked
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (kh * 64 + i > r) sv[i] = -INFINITY;
        }
        float pm[8];  // independent partial maxima (short dependency chains)
#pragma unroll
        for (int i = 0; i < 8; ++i) pm[i] = fmaxf(sv[i], sv[i + 8]);
#pragma unroll
        for (int i = 16; i < 64; i += 8) {
#pragma unroll
          for (int k = 0; k < 8; ++k) pm[k] = fmaxf(pm[k], sv[i + k]);
        }
        sts_f32(&red[kh * 128 + r], fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                          fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))));
        asm volatile("bar.sync %0, 64;" ::"r"(nb) : "memory");  // the row's two halves
        const float mx = fmaxf(lds_f32(&red[r]), lds_f32(&red[128 + r])) * scale_log2;
        asm volatile("bar.sync %0, 64;" ::"r"(nb) : "memory");  // red reusable next tile
        // lazy rescale: raise m only when the row max outgrows it by more than 2^8
        const bool raise = mx > m + kRescaleLog2;
        const float alpha = raise ? ex2(m - mx) : 1.f;  // 0 on the first tile (m = -inf)
        if (raise) m = mx;
        // exponentials and row sum (registers), packed bf16 pairs for the TMEM P tile
        uint32_t pk[32];
        float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          // (ex2_poly for a share of the pairs measured no faster here: the phase is not MUFU-bound)
          const bool poly = false;
          const float x0 = fmaf(sv[i], scale_log2, -m), x1 = fmaf(sv[i + 1], scale_log2, -m);
          const float p0 = poly ? ex2_poly(x0) : ex2(x0);
          const float p1 = poly ? ex2_poly(x1) : ex2(x1);
          ps[(i >> 1) & 7] += p0 + p1;
          pk[i >> 1] = pack_bf16(p0, p1);
        }
        // P.V(j-1) must have finished reading P and accumulating into O
        if (j > 0) {
          ptx::mbar_wait(pv_done, (g - 1) & 1);
          ptx::tc_fence_after();
          if (__any_sync(0xffffffffu, raise)) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(t_o, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            ptx::tmem_st_32x32b_x32(t_o, v);
          }
        }
        l = l * alpha + (((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7])));
        ptx::tmem_st_32x32b_x32(t_p, pk);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full);
      }
      // epilogue: wait for the last P.V, combine the halves' row sums, O / l -> bf16, LSE
      ptx::mbar_wait(pv_done, (g - 1) & 1);
      ptx::tc_fence_after();
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(t_o, v);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(o_free);
      sts_f32(&red[kh * 128 + r], l);
      asm volatile("bar.sync %0, 64;" ::"r"(nb) : "memory");
      const float lt = lds_f32(&red[r]) + lds_f32(&red[128 + r]);
      asm volatile("bar.sync %0, 64;" ::"r"(nb) : "memory");
      const float inv = 1.f / lt;
      const int64_t row = int64_t(smp) * seq + int64_t(tk.tile) * kT + r;
      bf16* dst = out + row * h + head * kD + kh * 32;
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        uint4 u;
        u.x = pack_bf16(__uint_as_float(v[c]) * inv, __uint_as_float(v[c + 1]) * inv);
        u.y = pack_bf16(__uint_as_float(v[c + 2]) * inv, __uint_as_float(v[c + 3]) * inv);
        u.z = pack_bf16(__uint_as_float(v[c + 4]) * inv, __uint_as_float(v[c + 5]) * inv);
        u.w = pack_bf16(__uint_as_float(v[c + 6]) * inv, __uint_as_float(v[c + 7]) * inv);
        *reinterpret_cast<uint4*>(dst + c) = u;
      }
      if (kh == 0) lse[int64_t(tk.z) * seq + int64_t(tk.tile) * kT + r] = (m + log2f(lt)) / kLog2e;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (pipe == 0 && warp == kFwdProducer) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(*tmem_slot0, 512);
  }
}

// ============================================================================ backward
// Transposed formulation: one CTA task = 128 keys of one (head, sample); for every query tile at
// or above the diagonal the MMA warp computes S^T = K Q^T and dP^T = V dO^T into TMEM (keys on
// the TMEM lanes). Eight builder warps turn them into P^T = exp2(S^T c - LSE) and
// dS'^T = P^T (dP^T - D) (per-query LSE and D come with the Q/dO stage) and write them back into
// TMEM as packed bf16 (P^T into its own columns, dS'^T in place over dP^T once both column halves
// of a row have read it), and dS'^T also into shared memory. S^T of the next tile is issued as
// soon as the builders have read this one, so it overlaps their work. Then dV += P^T dO and dK += dS'^T Q take P^T / dS'^T as
// TMEM A operands (no shared-memory round trip), and dQ_tile = dS' K reads the shared dS'^T tile
// as an MN-major operand. Four warps read dQ out of TMEM and add it into the fp32 dQ with TMA
// bulk reduce-add; after a task's last tile they write dK (scaled) and dV.
// Warp roles: 0-7 builders (TMEM lane quarter w % 4, query half w / 4), 8-11 dQ / dK dV out,
// 12 TMA producer, 13 score MMA issuer (S^T, dP^T), 14 gradient MMA issuer (dK, dV, dQ): the two
// issuers never block each other, so the next tile's scores are issued while this tile's
// gradient products wait for the builders. K/V are double-buffered so the next task's key tile loads
// while this one runs.
constexpr int kBwdThreads = 480;
constexpr int kBwdQD = 3;  // Q/dO (+LSE, D) stages
constexpr int kBwdKV = 2;  // K/V stages
// TMEM columns: S^T, dP^T, dS'^T packed (then dQ of the same tile, after dK has read dS'^T),
// P^T packed, dV, dK. S^T and dP^T of the next tile are issued as soon as the builders have read
// this one; the builders store P^T once dV of the previous tile is done and dS'^T (the last thing
// they write) once the previous dQ has been read out.
constexpr int kBwdTS = 0, kBwdTDP = 128, kBwdTDS = 256, kBwdTDQ = 256, kBwdTP = 320, kBwdTDV = 384,
              kBwdTDK = 448;

struct BwdSmem {
  static constexpr int kK = 0;                        // kBwdKV stages
  static constexpr int kV = kK + kBwdKV * kTile;      // kBwdKV stages
  static constexpr int kQ = kV + kBwdKV * kTile;      // kBwdQD stages
  static constexpr int kDO = kQ + kBwdQD * kTile;     // kBwdQD stages
  static constexpr int kDS = kDO + kBwdQD * kTile;    // dS'^T [128 keys, 128 queries]
  static constexpr int kDQ = kDS + 2 * kTile;         // dQ staging: 4 warps x [32 rows x 32] fp32
  static constexpr int kLD = kDQ + 4 * 32 * 32 * 4;   // kBwdQD stages x {LSE, D}[128] fp32
  static constexpr int kBar = kLD + kBwdQD * 2 * 128 * 4;
  static constexpr int kBytes = kBar + 256 + 1024;
};
static_assert(BwdSmem::kBytes <= 232448, "backward shared memory");

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_do,
                    const __grid_constant__ CUtensorMap map_dq,
                    const float* __restrict__ lse, const float* __restrict__ dvec,
                    bf16* __restrict__ dqkv, int seq, int heads, int nz, float scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BwdSmem::kBar);
  uint64_t* kv_full = bar + 0;                     // [kBwdKV]
  uint64_t* kv_empty = bar + kBwdKV;               // [kBwdKV]
  uint64_t* qd_full = bar + 2 * kBwdKV;            // [kBwdQD]
  uint64_t* qd_empty = qd_full + kBwdQD;           // [kBwdQD]
  uint64_t* s_full = qd_full + 2 * kBwdQD;         // S^T in TMEM
  uint64_t* s_free = s_full + 1;                   // S^T read by the builders
  uint64_t* dp_full = s_full + 2;                  // dP^T in TMEM
  uint64_t* pt_full = s_full + 3;                  // P^T, dS'^T in TMEM
  uint64_t* dp_free = s_full + 4;                  // dP^T read by the builders
  uint64_t* mm_done = s_full + 5;                  // dQ product done: dQ in TMEM (dS'^T columns), dS' smem free
  uint64_t* acc_free = s_full + 6;                 // dK/dV read out by the epilogue
  uint64_t* dq_free = s_full + 7;                  // dQ read out of TMEM
  uint64_t* dv_done = s_full + 8;                  // dV product done: P^T TMEM read
  uint64_t* dk_done = s_full + 10;                 // dK product done: dS'^T TMEM read
  uint64_t* ds_full = s_full + 9;                  // dS'^T in shared memory
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 11);

  const int warp = int(ptx::warp_id());
  const int lane = threadIdx.x & 31;
  const int nt = seq / kT;
  const int ntasks = nt * nz;
  const int h = heads * kD;

  if (warp == 12 && lane == 0) {
    ptx::tma_prefetch_desc(&map_qkv);
    ptx::tma_prefetch_desc(&map_do);
    ptx::tma_prefetch_desc(&map_dq);
    for (int i = 0; i < kBwdKV; ++i) {
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < kBwdQD; ++i) {
      ptx::mbar_init(&qd_full[i], 1);
      ptx::mbar_init(&qd_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_free, 256);
    ptx::mbar_init(dp_full, 1);
    ptx::mbar_init(pt_full, 256);
    ptx::mbar_init(ds_full, 256);
    ptx::mbar_init(dp_free, 256);
    ptx::mbar_init(dk_done, 1);
    ptx::mbar_init(dv_done, 1);
    ptx::mbar_init(mm_done, 1);
    ptx::mbar_init(acc_free, 128);
    ptx::mbar_init(dq_free, 128);
    ptx::fence_barrier_init();
  }
  if (warp == 12) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 12) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0, item = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++item) {
        const AttnTask tk = bwd_task_static(t, nz);
        const int smp = tk.z / heads, head = tk.z % heads;
        const int row0 = smp * seq;
        const int kvs = item % kBwdKV;
        ptx::mbar_wait(&kv_empty[kvs], ((item / kBwdKV) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[kvs], 2 * kTile);
        ptx::tma_load_4d(sm + BwdSmem::kK + kvs * kTile, &map_qkv, &kv_full[kvs], h + head * kD,
                         row0 + tk.tile * kT, 0, 0);
        ptx::tma_load_4d(sm + BwdSmem::kV + kvs * kTile, &map_qkv, &kv_full[kvs], 2 * h + head * kD,
                         row0 + tk.tile * kT, 0, 0);
        for (int i = tk.tile; i < nt; ++i) {
          ptx::mbar_wait(&qd_empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&qd_full[stage], 2 * kTile + 2 * 128 * 4);
          ptx::tma_load_4d(sm + BwdSmem::kQ + stage * kTile, &map_qkv, &qd_full[stage], head * kD,
                           row0 + i * kT, 0, 0);
          ptx::tma_load_4d(sm + BwdSmem::kDO + stage * kTile, &map_do, &qd_full[stage], head * kD,
                           row0 + i * kT, 0, 0);
          const int64_t q0 = int64_t(tk.z) * seq + int64_t(i) * kT;
          ptx::bulk_load(sm + BwdSmem::kLD + stage * 1024, lse + q0, 512, &qd_full[stage]);
          ptx::bulk_load(sm + BwdSmem::kLD + stage * 1024 + 512, dvec + q0, 512, &qd_full[stage]);
          if (++stage == kBwdQD) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 13) {
    if (lane == 0) {  // ------------------------------------------ score MMA issuer: S^T, dP^T
      constexpr uint32_t id_ss = ptx::idesc_bf16_f32(128, 128, 0, 0);
      int ss = 0;
      uint32_t ss_ph = 0, item = 0, it = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++item) {
        const AttnTask tk = bwd_task_static(t, nz);
        const int kvs = item % kBwdKV;
        ptx::mbar_wait(&kv_full[kvs], (item / kBwdKV) & 1);
        const uint32_t sk = ptx::smem_u32(sm + BwdSmem::kK + kvs * kTile);
        const uint32_t sv = ptx::smem_u32(sm + BwdSmem::kV + kvs * kTile);
        for (int i = tk.tile; i < nt; ++i, ++it) {
          ptx::mbar_wait(&qd_full[ss], ss_ph);
          const uint32_t sq = ptx::smem_u32(sm + BwdSmem::kQ + ss * kTile);
          const uint32_t sdo = ptx::smem_u32(sm + BwdSmem::kDO + ss * kTile);
          ptx::mbar_wait(s_free, (it & 1) ^ 1);  // builders read the previous S^T
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k) ptx::umma_bf16(tmem + kBwdTS, kdesc(sk, k), kdesc(sq, k), id_ss, k > 0);
          ptx::umma_commit(s_full);
          ptx::mbar_wait(dp_free, (it & 1) ^ 1);  // builders read the previous dP^T
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k) ptx::umma_bf16(tmem + kBwdTDP, kdesc(sv, k), kdesc(sdo, k), id_ss, k > 0);
          ptx::umma_commit(dp_full);
          if (++ss == kBwdQD) {
            ss = 0;
            ss_ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 14) {
    if (lane == 0) {  // --------------------------------------- gradient MMA issuer: dK, dV, dQ
      constexpr uint32_t id_t = ptx::idesc_bf16_f32(128, 64, 0, 1);  // dV, dK: A in TMEM, B MN-major
      constexpr uint32_t id_q = ptx::idesc_bf16_f32(128, 64, 1, 1);  // dQ: A = dS' (MN-major), B = K
      const uint32_t sds = ptx::smem_u32(sm + BwdSmem::kDS);
      int ss = 0;
      uint32_t item = 0, it = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++item) {
        const AttnTask tk = bwd_task_static(t, nz);
        const int kvs = item % kBwdKV;
        ptx::mbar_wait(&kv_full[kvs], (item / kBwdKV) & 1);
        const uint32_t sk = ptx::smem_u32(sm + BwdSmem::kK + kvs * kTile);
        for (int i = tk.tile; i < nt; ++i, ++it) {
          const uint32_t sq = ptx::smem_u32(sm + BwdSmem::kQ + ss * kTile);
          const uint32_t sdo = ptx::smem_u32(sm + BwdSmem::kDO + ss * kTile);
          const bool first = (i == tk.tile);
          if (first) ptx::mbar_wait(acc_free, (item & 1) ^ 1);  // previous task's dK/dV read out
          ptx::mbar_wait(pt_full, it & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::umma_bf16_ts(tmem + kBwdTDK, tmem + kBwdTDS + 8 * k, mndesc(sq, k), id_t, (!first || k > 0));
          ptx::umma_commit(dk_done);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::umma_bf16_ts(tmem + kBwdTDV, tmem + kBwdTP + 8 * k, mndesc(sdo, k), id_t, (!first || k > 0));
          ptx::umma_commit(dv_done);
          // dQ lands in the dS'^T columns: after dK has read dS'^T
          ptx::mbar_wait(dk_done, it & 1);
          ptx::mbar_wait(ds_full, it & 1);  // dS'^T in shared memory
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < 8; ++k) ptx::umma_bf16(tmem + kBwdTDQ, mndesc(sds, k), mndesc(sk, k), id_q, k > 0);
          ptx::umma_commit(mm_done);
          ptx::umma_commit(&qd_empty[ss]);  // the stage's S^T / dP^T products finished before pt_full
          if (i == nt - 1) ptx::umma_commit(&kv_empty[kvs]);
          if (++ss == kBwdQD) ss = 0;
        }
      }
    }
  } else if (warp < 8) {  // ------------------------------------------ P^T / dS'^T builders
    const int q4 = warp & 3, kh = warp >> 2;
    const int r = q4 * 32 + lane;  // key row of the tile == TMEM lane
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    const uint32_t sds = ptx::smem_u32(sm + BwdSmem::kDS);
    int ss = 0;
    uint32_t ss_ph = 0, it = 0;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
      const AttnTask tk = bwd_task_static(t, nz);
      for (int i = tk.tile; i < nt; ++i, ++it) {
        ptx::mbar_wait(&qd_full[ss], ss_ph);  // this stage's LSE / D (already complete: S^T needed Q)
        ptx::mbar_wait(s_full, it & 1);
        ptx::tc_fence_after();
        ptx::mbar_wait(dp_full, it & 1);
        ptx::tc_fence_after();
        // per-query LSE and D of this stage (broadcast shared reads), indexed from the __shared__
        // array itself so the compiler emits schedulable LDS
        const float4* ld4 = reinterpret_cast<const float4*>(smem_raw + (sm - smem_raw) + BwdSmem::kLD + ss * 1024);
        const float sl2 = scale * kLog2e;
        uint32_t dk[32];  // packed bf16 pairs of this thread's 64 dS'^T values
        // two passes of 32 query columns keep the live registers low
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t vs[32], vp[32], pk[16];
          ptx::tmem_ld_32x32b_x32(tmem + kBwdTS + lane_off + kh * 64 + c * 32, vs);
          ptx::tmem_ld_32x32b_x32(tmem + kBwdTDP + lane_off + kh * 64 + c * 32, vp);
          ptx::tmem_ld_wait();
          if (c == 1) {
            ptx::tc_fence_before();
            ptx::mbar_arrive(s_free);   // S^T and dP^T fully read: the MMA warp may issue the
            ptx::mbar_arrive(dp_free);  // next tile's products into these columns
          }
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const int q = kh * 64 + c * 32 + e;
            const float4 lq = ld4[q / 4], dq4 = ld4[32 + q / 4];
            const float l4[4] = {lq.x, lq.y, lq.z, lq.w}, d4[4] = {dq4.x, dq4.y, dq4.z, dq4.w};
            float pv[4], dv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              pv[u] = ex2(fmaf(__uint_as_float(vs[e + u]), sl2, -l4[u] * kLog2e));
              dv[u] = pv[u] * (__uint_as_float(vp[e + u]) - d4[u]);
            }
            pk[e / 2] = pack_bf16(pv[0], pv[1]);
            pk[e / 2 + 1] = pack_bf16(pv[2], pv[3]);
            dk[c * 16 + e / 2] = pack_bf16(dv[0], dv[1]);
            dk[c * 16 + e / 2 + 1] = pack_bf16(dv[2], dv[3]);
          }
          if (i == tk.tile) {  // diagonal tile: key (row r) > query (column) gives P = dS = 0
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int q0 = kh * 64 + c * 32 + 2 * e;
              const uint32_t keep = (r > q0 ? 0u : 0xffffu) | (r > q0 + 1 ? 0u : 0xffff0000u);
              pk[e] &= keep;
              dk[c * 16 + e] &= keep;
            }
          }
          if (c == 0) {
            ptx::mbar_wait(dv_done, (it & 1) ^ 1);  // dV of the previous tile has read P^T
            ptx::tc_fence_after();
          }
          ptx::tmem_st_32x32b_x16(tmem + kBwdTP + lane_off + kh * 32 + c * 16, pk);
        }
        // the dS'^T columns held dQ of the previous tile: read out by the dQ warps
        ptx::mbar_wait(dq_free, (it & 1) ^ 1);
        ptx::tc_fence_after();
        ptx::tmem_st_32x32b_x32(tmem + kBwdTDS + lane_off + kh * 32, dk);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(pt_full);  // dK / dV may start
        // dS'^T into shared memory for dQ = dS' K, once dQ of the previous tile has read it
        ptx::mbar_wait(mm_done, (it & 1) ^ 1);
#pragma unroll
        for (int g = 0; g < 8; ++g)
          st_shared_v4(sds + p_off(r, kh * 64 + g * 8), dk[4 * g], dk[4 * g + 1], dk[4 * g + 2], dk[4 * g + 3]);
        fence_proxy_async();
        ptx::mbar_arrive(ds_full);
        if (++ss == kBwdQD) {
          ss = 0;
          ss_ph ^= 1;
        }
      }
    }
  } else if (warp < 12) {  // ------------------------------------------ warps 8-11: dQ + dK/dV out
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    uint8_t* stg = sm + BwdSmem::kDQ + q4 * (32 * 32 * 4);
    uint32_t it = 0;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
      const AttnTask tk = bwd_task_static(t, nz);
      const int smp = tk.z / heads, head = tk.z % heads;
      for (int i = tk.tile; i < nt; ++i, ++it) {
        ptx::mbar_wait(mm_done, it & 1);  // on the critical path: dQ shares the P^T columns
        ptx::tc_fence_after();
        uint32_t v[2][32];
        ptx::tmem_ld_32x32b_x32(tmem + kBwdTDQ + lane_off, v[0]);
        ptx::tmem_ld_32x32b_x32(tmem + kBwdTDQ + lane_off + 32, v[1]);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(dq_free);
        // this warp's 32 dQ rows, 32 columns at a time -> swizzled fp32 box -> TMA reduce-add
        const int row = smp * seq + i * kT + q4 * 32;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (lane == 0) ptx::bulk_wait_read<0>();  // the previous reduce has read the box
          __syncwarp();
          const uint32_t rowa = ptx::smem_u32(stg) + lane * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowa + ((j ^ (lane & 7)) << 4)),
                         "r"(v[c][4 * j]), "r"(v[c][4 * j + 1]), "r"(v[c][4 * j + 2]), "r"(v[c][4 * j + 3])
                         : "memory");
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_reduce_add_2d(&map_dq, stg, head * kD + 32 * c, row);
            ptx::bulk_commit();
          }
        }
      }
      // epilogue: dK (scaled), dV rows of this key tile -> bf16 into dqkv
      const int64_t krow = int64_t(smp) * seq + int64_t(tk.tile) * kT + r;
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        bf16* dst = dqkv + krow * 3 * h + (which == 0 ? h : 2 * h) + head * kD;
        const uint32_t src = tmem + (which == 0 ? kBwdTDK : kBwdTDV) + lane_off;
        const float f = which == 0 ? scale : 1.f;  // dK = scale * dS'^T Q
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(src + c * 32, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(v[e]) * f, __uint_as_float(v[e + 1]) * f);
            u.y = pack_bf16(__uint_as_float(v[e + 2]) * f, __uint_as_float(v[e + 3]) * f);
            u.z = pack_bf16(__uint_as_float(v[e + 4]) * f, __uint_as_float(v[e + 5]) * f);
            u.w = pack_bf16(__uint_as_float(v[e + 6]) * f, __uint_as_float(v[e + 7]) * f);
            *reinterpret_cast<uint4*>(dst + c * 32 + e) = u;
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(acc_free);
    }
    if (lane == 0) ptx::bulk_wait<0>();  // dQ reductions complete before the kernel ends
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ============================================================================ forward, head_dim 128
// One CTA task = a block of two consecutive 128-query tiles (Q0, Q1) of one (head, sample); the two
// tiles share every K/V tile the TMA warp streams in, and their softmax warp groups ping-pong
// with the single MMA warp:
//   S0(0) S1(0) | PV0(0) S0(1) | PV1(0) S1(1) | PV0(1) S0(2) | ...
// so the tensor pipe computes one tile's products while the other tile's eight softmax warps turn
// scores into probabilities. TMEM: S0/P0 [0,128), S1/P1 [128,256), O0 [256,384), O1 [384,512).
// P (packed bf16 pairs) overwrites the S columns of the key half that produced it: a thread that
// owns keys 64*kh.. writes P columns 64*kh..64*kh+31, so the two halves of a row never touch each
// other's scores. S(j+1) is issued after P.V(j) in the same tensor pipe (in-order execution), so
// it only overwrites P(j) once P.V(j) has consumed it. Causal: Q0 = queries 256b..+127 needs key
// tiles 0..2b (2b diagonal), Q1 needs 0..2b+1 (2b+1 diagonal).
// Warp roles: 0-7 softmax of Q0, 8-15 softmax of Q1 (lane quarter w % 4, key half (w / 4) % 2),
// 16 TMA producer, 17 MMA issuer.
constexpr int kD2 = 128;
constexpr int kBlk = kT * 64 * 2;  // [128, 64] bf16 SWIZZLE_128B block = 16 KiB
constexpr int kTile2 = 2 * kBlk;   // [128, 128] tile (two blocks along the head dim)
constexpr int kF2Threads = 18 * 32;
constexpr int kFwdPolyDefault = 0;  // exponential pairs per 4 on the FMA pipe (ZP_ATTN_POLY overrides)
constexpr int kF2Producer = 16, kF2Mma = 17;

struct F2Smem {
  static constexpr int kQ = 0;                     // Q0, Q1
  static constexpr int kK = kQ + 2 * kTile2;       // 2 stages
  static constexpr int kV = kK + 2 * kTile2;       // 2 stages
  static constexpr int kRed = kV + 2 * kTile2;     // [2 groups][3 buffers][2 halves][128 rows] fp32
  static constexpr int kBar = kRed + 2 * 3 * 2 * 128 * 4;
  static constexpr int kBytes = kBar + 256 + 1024;
};
static_assert(F2Smem::kBytes <= 232448, "forward d128 shared memory");

__device__ unsigned int g_sched2[4];  // [fwd counter, fwd done, bwd counter, bwd done] (head_dim 128)

// Timeline diagnostics (tools/microbench/attn_trace.cu builds this file with ZP_ATTN_TRACE): CTA 0
// stamps clock64 at the pipeline events of its first tiles (ATR: backward, ATRF: forward).
#ifdef ZP_ATTN_TRACE
__device__ unsigned long long g_attn_trace[16][64];
__device__ unsigned long long g_attn_trace_f[16][64];
#define ATR(ev, i)                                                           \
  do {                                                                       \
    if (blockIdx.x == 0 && (i) < 64) g_attn_trace[ev][i] = clock64();       \
  } while (0)
#define ATRF(ev, i, first)                                                             \
  do {                                                                                 \
    if (blockIdx.x == 0 && (first) && (i) < 64) g_attn_trace_f[ev][i] = clock64();    \
  } while (0)
#else
#define ATR(ev, i) \
  do {             \
  } while (0)
#define ATRF(ev, i, first) \
  do {                     \
  } while (0)
#endif

// K-major [128, 128] tile stored as two 64-wide SWIZZLE_128B blocks, k16 step 0..7.
__device__ __forceinline__ uint64_t kdesc128(uint32_t base, int k16) {
  return ptx::smem_desc_sw128(base + (k16 >> 2) * kBlk + (k16 & 3) * 32, 16, 1024);
}

// POLY: how many of every 4 exponential pairs run on the FMA pipe (ex2_poly) instead of MUFU. At
// head_dim 128 a tile's 16384 exponentials take as long on MUFU (16/clk/SM) as its two 128-wide
// products take on the tensor pipe, so moving a share to the FMA pipe shortens the softmax phase.
template <int POLY>
__global__ void __launch_bounds__(kF2Threads, 1)
    attn_fwd_d128_kernel(const __grid_constant__ CUtensorMap map_qkv, bf16* __restrict__ out,
                         float* __restrict__ lse, int seq, int heads, int nz, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + F2Smem::kBar);
  uint64_t* q_full = bar + 0;
  uint64_t* q_empty = bar + 1;
  uint64_t* kv_full = bar + 2;   // [2]
  uint64_t* kv_empty = bar + 4;  // [2]
  uint64_t* s_full = bar + 6;    // [2 groups] S in TMEM (MMA -> softmax)
  uint64_t* p_full = bar + 8;    // [2] P in TMEM, O rescaled (softmax -> MMA)
  uint64_t* pv_done = bar + 10;  // [2] P.V complete (MMA -> softmax epilogue)
  uint64_t* o_free = bar + 12;   // [2] O read out (softmax -> MMA)
  const TaskRing ring{reinterpret_cast<int*>(bar + 14), bar + 16, bar + 20};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 24);

  const int warp = int(ptx::warp_id());
  const int lane = threadIdx.x & 31;
  const int nt = seq / kT;
  const int nb = (nt + 1) / 2;  // query blocks of two tiles
  const int ntasks = nb * nz;
  const int h = heads * kD2;

  if (warp == kF2Producer && lane == 0) {
    ptx::tma_prefetch_desc(&map_qkv);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 256);
      ptx::mbar_init(&pv_done[i], 1);
      ptx::mbar_init(&o_free[i], 256);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&ring.full[i], 1);
      ptx::mbar_init(&ring.empty[i], 17);  // MMA thread + 16 softmax warps
    }
    ptx::fence_barrier_init();
  }
  if (warp == kF2Producer) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kF2Producer) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t item = 0;; ++item) {
        const int t = ring.produce(item, &g_sched2[0]);
        if (t >= ntasks) break;
        const AttnTask tk = group_task(t, nz, nb, true);
        const int smp = tk.z / heads, head = tk.z % heads;
        const int row0 = smp * seq;
        const bool has1 = 2 * tk.tile + 1 < nt;
        const int q0 = row0 + 2 * tk.tile * kT;
        ptx::mbar_wait(q_empty, (item & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(q_full, (has1 ? 2 : 1) * kTile2);
        for (int q = 0; q < (has1 ? 2 : 1); ++q)
          for (int c = 0; c < 2; ++c)
            ptx::tma_load_4d(sm + F2Smem::kQ + q * kTile2 + c * kBlk, &map_qkv, q_full, head * kD2 + 64 * c,
                             q0 + q * kT, 0, 0);
        const int nj = 2 * tk.tile + (has1 ? 2 : 1);
        for (int j = 0; j < nj; ++j) {
          ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&kv_full[stage], 2 * kTile2);
          for (int c = 0; c < 2; ++c) {
            ptx::tma_load_4d(sm + F2Smem::kK + stage * kTile2 + c * kBlk, &map_qkv, &kv_full[stage],
                             h + head * kD2 + 64 * c, row0 + j * kT, 0, 0);
            ptx::tma_load_4d(sm + F2Smem::kV + stage * kTile2 + c * kBlk, &map_qkv, &kv_full[stage],
                             2 * h + head * kD2 + 64 * c, row0 + j * kT, 0, 0);
          }
          if (++stage == 2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      sched_finish(&g_sched2[0], 1);
    }
  } else if (warp == kF2Mma) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t id_o = ptx::idesc_bf16_f32(128, 128, 0, 1);
      int kw = 0;           // K/V tiles waited for (full barrier phases), as a running count
      int kd = 0;           // K/V tiles released
      uint32_t gp[2] = {0, 0};    // P.V issues per group (p_full phases)
      uint32_t ntask[2] = {0, 0}; // tasks per group (o_free phases)
      auto wait_kv = [&](int upto) {  // make sure K/V tile number `upto` (running count) has landed
        while (kw <= upto) {
          ptx::mbar_wait(&kv_full[kw & 1], (kw >> 1) & 1);
          ++kw;
        }
      };
      uint32_t titem = 0;  // trace: the first task only
      auto issue_s = [&](int g, int kvi) {
        ATRF(1 + 2 * g, kvi, titem == 0);
        const uint32_t sq = ptx::smem_u32(sm + F2Smem::kQ + g * kTile2);
        const uint32_t sk = ptx::smem_u32(sm + F2Smem::kK + (kvi & 1) * kTile2);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) ptx::umma_bf16(tmem + 128 * g, kdesc128(sq, k), kdesc128(sk, k), id_s, k > 0);
        ptx::umma_commit(&s_full[g]);
      };
      auto issue_pv = [&](int g, int kvi, bool acc) {
        ptx::mbar_wait(&p_full[g], gp[g] & 1);
        ++gp[g];
        ptx::tc_fence_after();
        ATRF(2 * g, kvi, titem == 0);
        const uint32_t sv = ptx::smem_u32(sm + F2Smem::kV + (kvi & 1) * kTile2);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t pcol = 128 * g + (k < 4 ? 8 * k : 64 + 8 * (k - 4));
          ptx::umma_bf16_ts(tmem + 256 + 128 * g, tmem + pcol, mndesc(sv, k), id_o, acc || k > 0);
        }
        ptx::umma_commit(&pv_done[g]);
      };
      for (uint32_t item = 0;; ++item) {
        const int t = ring.consume1(item);
        if (t >= ntasks) break;
        titem = item;
        const AttnTask tk = group_task(t, nz, nb, true);
        const bool has1 = 2 * tk.tile + 1 < nt;
        const int nj0 = 2 * tk.tile + 1, nj1 = has1 ? 2 * tk.tile + 2 : 0;
        const int nj = has1 ? nj1 : nj0;
        const int kv0 = kd;  // running index of this task's key tile 0
        ptx::mbar_wait(q_full, item & 1);
        wait_kv(kv0);
        issue_s(0, kv0);
        if (has1) issue_s(1, kv0);
        if (nj == 1) ptx::umma_commit(q_empty);
        for (int j = 0; j < nj; ++j) {
          const int kv = kv0 + j;
          if (j < nj0) {
            if (j == 0) ptx::mbar_wait(&o_free[0], (ntask[0] & 1) ^ 1);  // previous O0 read out
            issue_pv(0, kv, j > 0);
            if (j + 1 < nj0) {
              wait_kv(kv + 1);
              issue_s(0, kv + 1);
            }
          }
          if (j < nj1) {
            if (j == 0) ptx::mbar_wait(&o_free[1], (ntask[1] & 1) ^ 1);
            issue_pv(1, kv, j > 0);
            if (j + 1 < nj1) {
              wait_kv(kv + 1);
              issue_s(1, kv + 1);
            }
          }
          if (j + 2 == nj) ptx::umma_commit(q_empty);  // the task's last S has been issued
          ptx::umma_commit(&kv_empty[kv & 1]);
          ++kd;
        }
        ++ntask[0];
        if (has1) ++ntask[1];
      }
    }
  } else {  // -------------------------------------------------------------- softmax warps 0-15
    const int g = warp >> 3;                 // query tile of the block
    const int q4 = warp & 3, kh = (warp >> 2) & 1;
    const int nbar = 1 + g * 4 + q4;         // named barrier of the row quarter's two halves
    const int r = q4 * 32 + lane;            // query row within the tile == TMEM lane
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    // row-statistics exchange between the two halves of a row: [3 buffers][2 halves][128]; the
    // per-tile max alternates between buffers 0 and 1 (one barrier per tile: a half rewrites a
    // buffer only after the barrier of the next tile, which its partner passes after reading it),
    // buffer 2 carries the final row sum
    float* red0 = reinterpret_cast<float*>(sm + F2Smem::kRed) + g * 768;
    const uint32_t t_s = tmem + 128 * g + lane_off + kh * 64;
    const uint32_t t_p = tmem + 128 * g + lane_off + kh * 64;  // packed P over this half's S columns
    const uint32_t t_o = tmem + 256 + 128 * g + lane_off + kh * 64;
    uint32_t cnt = 0, ntk = 0;
    for (uint32_t item = 0;; ++item) {
      const int t = ring.consume(item);
      if (t >= ntasks) break;
      const AttnTask tk = group_task(t, nz, nb, true);
      const bool has1 = 2 * tk.tile + 1 < nt;
      if (g == 1 && !has1) continue;
      const int smp = tk.z / heads, head = tk.z % heads;
      const int qt = 2 * tk.tile + g;  // this group's query tile
      const int nj = qt + 1;           // key tiles 0..qt, qt diagonal
      float m = -INFINITY, l = 0.f;
      const bool tr = item == 0 && lane == 0 && (warp == 0 || warp == 8);
      for (int j = 0; j < nj; ++j, ++cnt) {
        ptx::mbar_wait(&s_full[g], cnt & 1);
        ptx::tc_fence_after();
        ATRF(4 + 4 * g, j, tr);
        float sv[64];
        {
          uint32_t v0[32], v1[32];
          ptx::tmem_ld_32x32b_x32(t_s, v0);
          ptx::tmem_ld_32x32b_x32(t_s + 32, v1);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            sv[i] = __uint_as_float(v0[i]);
            sv[32 + i] = __uint_as_float(v1[i]);
          }
        }
        if (j == qt) {  // diagonal tile: key > query is masked
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (kh * 64 + i > r) sv[i] = -INFINITY;
        }
        float pm[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pm[i] = fmaxf(sv[i], sv[i + 8]);
#pragma unroll
        for (int i = 16; i < 64; i += 8) {
#pragma unroll
          for (int k = 0; k < 8; ++k) pm[k] = fmaxf(pm[k], sv[i + k]);
        }
        float* red = red0 + (cnt & 1) * 256;
        sts_f32(&red[kh * 128 + r], fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                          fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))));
        asm volatile("bar.sync %0, 64;" ::"r"(nbar) : "memory");
        const float mx = fmaxf(lds_f32(&red[r]), lds_f32(&red[128 + r])) * scale_log2;
        ATRF(5 + 4 * g, j, tr);
        const bool raise = mx > m + kRescaleLog2;
        const float alpha = raise ? ex2(m - mx) : 1.f;
        if (raise) m = mx;
        uint32_t pk[32];
        float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        // two halves: the first half's P store (S columns already in registers; P.V(j-1) is complete)
        // overlaps the second half's exponentials
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int i = 32 * hh; i < 32 * hh + 32; i += 2) {
            const float x0 = fmaf(sv[i], scale_log2, -m), x1 = fmaf(sv[i + 1], scale_log2, -m);
            const bool poly = ((i >> 1) & 3) < POLY;
            const float p0 = poly ? ex2_poly(x0) : ex2(x0), p1 = poly ? ex2_poly(x1) : ex2(x1);
            ps[(i >> 1) & 7] += p0 + p1;
            pk[i >> 1] = pack_bf16(p0, p1);
          }
          uint32_t (&half)[16] = *reinterpret_cast<uint32_t(*)[16]>(&pk[16 * hh]);
          ptx::tmem_st_32x32b_x16(t_p + 16 * hh, half);
        }
        ATRF(6 + 4 * g, j, tr);
        // O += P.V of the previous tile is complete (it precedes this tile's S in the tensor pipe)
        if (j > 0 && __any_sync(0xffffffffu, raise)) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(t_o + c * 32, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            ptx::tmem_st_32x32b_x32(t_o + c * 32, v);
          }
        }
        l = l * alpha + (((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7])));
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ATRF(7 + 4 * g, j, tr);
        ptx::mbar_arrive(&p_full[g]);
      }
      // epilogue: the last P.V, the halves' row sums, O / l -> bf16, LSE
      ptx::mbar_wait(&pv_done[g], (cnt - 1) & 1);
      ptx::tc_fence_after();
      uint32_t o[2][32];
      ptx::tmem_ld_32x32b_x32(t_o, o[0]);
      ptx::tmem_ld_32x32b_x32(t_o + 32, o[1]);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&o_free[g]);
      ++ntk;
      float* red = red0 + 512;  // buffer 2: rewritten only after the next task's tile barriers
      sts_f32(&red[kh * 128 + r], l);
      asm volatile("bar.sync %0, 64;" ::"r"(nbar) : "memory");
      const float lt = lds_f32(&red[r]) + lds_f32(&red[128 + r]);
      const float inv = 1.f / lt;
      const int64_t row = int64_t(smp) * seq + int64_t(qt) * kT + r;
      bf16* dst = out + row * h + head * kD2 + kh * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(o[c][e]) * inv, __uint_as_float(o[c][e + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(o[c][e + 2]) * inv, __uint_as_float(o[c][e + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(o[c][e + 4]) * inv, __uint_as_float(o[c][e + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(o[c][e + 6]) * inv, __uint_as_float(o[c][e + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + c * 32 + e) = u;
        }
      if (kh == 0) lse[int64_t(tk.z) * seq + int64_t(qt) * kT + r] = (m + log2f(lt)) / kLog2e;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kF2Producer) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ============================================================================ backward, head_dim 128
// Transposed formulation as for head_dim 64: one CTA task = 128 keys of one (head, sample); for
// every query tile i at or above the diagonal the single MMA warp computes S^T = K Q^T and
// dP^T = V dO^T into TMEM (keys on the lanes). TMEM has room for exactly four 128-column fp32
// tiles, so every region is reused in place:
//   ST [0,128)   S^T, then P^T packed (each query half over its own S^T columns)
//   DP [128,256) dP^T, then dS'^T packed (likewise), then dQ = dS' K (fp32, queries on the lanes)
//   DV [256,384), DK [384,512) the task's accumulators.
// Task order: groups of kGroupZ (sample, head) pairs, key tile 0 (the longest) first within a
// group, dealt round-robin to the CTAs: the key tiles in flight share their heads' Q / dO tiles
// and dQ rows in L2 instead of streaming every head's from DRAM.
// MMA issue order per tile: dV(i) | S^T(i+1) | dK(i) | dQ(i) | dP^T(i+1): S^T of the next tile is
// issued as soon as dV has consumed P^T (the tensor pipe executes in order), so the eight builder
// warps compute the next tile's exponentials while dK / dQ run; dP^T(i+1) waits until the four dQ
// warps have read dQ(i) out of TMEM. dS'^T also goes to shared memory as the MN-major B operand of
// dQ^T = K^T dS'^T: with the head dims on the TMEM lanes, every fp32 reduction instruction of the dQ
// warps adds 128 contiguous bytes of one query row (red.global.add, no shared-memory staging that
// the next tile would wait on; the fp32 reductions run at the L2's ~20 B/clk/SM, measured by
// tools/microbench/red_bench.cu). Q(i) / dO(i) are released after dK(i), so the next loads start
// before the dQ product.
// Warp roles: 0-7 builders (lane quarter w % 4, query half w / 4), 8-11 dQ out + dK/dV epilogue,
// 12 TMA producer, 13 MMA issuer. K/V single-buffered per task; Q/dO(+LSE, D) two stages.
constexpr int kB2Threads = 14 * 32;

constexpr int kB2TS = 0, kB2TDP = 128, kB2TDV = 256, kB2TDK = 384;

struct B2Smem {
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTile2;
  static constexpr int kQ = kV + kTile2;           // 2 stages
  static constexpr int kDO = kQ + 2 * kTile2;      // 2 stages
  static constexpr int kDS = kDO + 2 * kTile2;     // dS'^T [128 keys, 128 queries]; dQ staging
  static constexpr int kLD = kDS + kTile2;         // 2 stages x {LSE, D}[128] fp32
  static constexpr int kBar = kLD + 2 * 1024;
  static constexpr int kBytes = kBar + 256;        // dynamic smem is 1 KiB aligned (checked)
};
static_assert(B2Smem::kBytes <= 232448, "backward d128 shared memory");

__global__ void __launch_bounds__(kB2Threads, 1)
    attn_bwd_d128_kernel(const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_do,
                         const float* __restrict__ lse, const float* __restrict__ dvec, float* __restrict__ dq32,
                         bf16* __restrict__ dqkv, const float2* __restrict__ rope_tab, int seq, int heads, int nz,
                         float scale, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  if (ptx::smem_u32(smem_raw) & 1023) __trap();  // the SWIZZLE_128B tiles need 1 KiB alignment
  uint8_t* sm = smem_raw;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + B2Smem::kBar);
  uint64_t* kv_full = bar + 0;
  uint64_t* kv_empty = bar + 1;
  uint64_t* qd_full = bar + 2;    // [2]
  uint64_t* qd_empty = bar + 4;   // [2]
  uint64_t* s_full = bar + 6;     // S^T in TMEM
  uint64_t* dp_full = bar + 7;    // dP^T in TMEM
  uint64_t* pt_full = bar + 8;    // P^T packed in TMEM (builders, 256)
  uint64_t* dst_full = bar + 9;   // dS'^T packed in TMEM (builders, 256)
  uint64_t* ds_full = bar + 10;   // dS'^T in shared memory (builders, 256)
  uint64_t* mm_done = bar + 11;   // dQ in TMEM (MMA)
  uint64_t* dq_free = bar + 12;   // dQ read out of TMEM (dQ warps, 128)
  uint64_t* acc_full = bar + 14;  // dK, dV complete (MMA)
  uint64_t* acc_free = bar + 15;  // dK, dV read out (epilogue, 128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = int(ptx::warp_id());
  const int lane = threadIdx.x & 31;
  const int nt = seq / kT;
  const int ntasks = nt * nz;
  const int h = heads * kD2;

  if (warp == 12 && lane == 0) {
    ptx::tma_prefetch_desc(&map_qkv);
    ptx::tma_prefetch_desc(&map_do);
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(kv_empty, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&qd_full[i], 1);
      ptx::mbar_init(&qd_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(dp_full, 1);
    ptx::mbar_init(pt_full, 256);
    ptx::mbar_init(dst_full, 256);
    ptx::mbar_init(ds_full, 256);
    ptx::mbar_init(mm_done, 1);
    ptx::mbar_init(dq_free, 128);
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(acc_free, 128);
    ptx::fence_barrier_init();
  }
  if (warp == 12) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 12) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0, item = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++item) {
        const AttnTask tk = group_task(t, nz, nt, false);
        const int smp = tk.z / heads, head = tk.z % heads;
        const int row0 = smp * seq;
        ptx::mbar_wait(kv_empty, (item & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(kv_full, 2 * kTile2);
        for (int c = 0; c < 2; ++c) {
          ptx::tma_load_4d(sm + B2Smem::kK + c * kBlk, &map_qkv, kv_full, h + head * kD2 + 64 * c,
                           row0 + tk.tile * kT, 0, 0);
          ptx::tma_load_4d(sm + B2Smem::kV + c * kBlk, &map_qkv, kv_full, 2 * h + head * kD2 + 64 * c,
                           row0 + tk.tile * kT, 0, 0);
        }
        for (int i = tk.tile; i < nt; ++i) {
          ptx::mbar_wait(&qd_empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&qd_full[stage], 2 * kTile2 + 2 * 128 * 4);
          for (int c = 0; c < 2; ++c) {
            ptx::tma_load_4d(sm + B2Smem::kQ + stage * kTile2 + c * kBlk, &map_qkv, &qd_full[stage],
                             head * kD2 + 64 * c, row0 + i * kT, 0, 0);
            ptx::tma_load_4d(sm + B2Smem::kDO + stage * kTile2 + c * kBlk, &map_do, &qd_full[stage],
                             head * kD2 + 64 * c, row0 + i * kT, 0, 0);
          }
          const int64_t q0 = int64_t(tk.z) * seq + int64_t(i) * kT;
          ptx::bulk_load(sm + B2Smem::kLD + stage * 1024, lse + q0, 512, &qd_full[stage]);
          ptx::bulk_load(sm + B2Smem::kLD + stage * 1024 + 512, dvec + q0, 512, &qd_full[stage]);
          if (++stage == 2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 13) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      constexpr uint32_t id_ss = ptx::idesc_bf16_f32(128, 128, 0, 0);  // S^T, dP^T: K-major both
      constexpr uint32_t id_t = ptx::idesc_bf16_f32(128, 128, 0, 1);   // dV, dK: A in TMEM, B MN-major
      constexpr uint32_t id_q = ptx::idesc_bf16_f32(128, 128, 1, 1);   // dQ: A = dS' (MN-major), B = K
      const uint32_t sk = ptx::smem_u32(sm + B2Smem::kK), sv = ptx::smem_u32(sm + B2Smem::kV);
      const uint32_t sds = ptx::smem_u32(sm + B2Smem::kDS);
      uint32_t item = 0, it = 0;
      auto sq = [&](uint32_t i) { return ptx::smem_u32(sm + B2Smem::kQ + (i & 1) * kTile2); };
      auto sdo = [&](uint32_t i) { return ptx::smem_u32(sm + B2Smem::kDO + (i & 1) * kTile2); };
      auto issue_st = [&](uint32_t i) {  // S^T(i) = K Q(i)^T
        ptx::mbar_wait(&qd_full[i & 1], (i >> 1) & 1);
        ptx::tc_fence_after();
        ATR(2, i);
#pragma unroll
        for (int k = 0; k < 8; ++k) ptx::umma_bf16(tmem + kB2TS, kdesc128(sk, k), kdesc128(sq(i), k), id_ss, k > 0);
        ptx::umma_commit(s_full);
      };
      auto issue_dpt = [&](uint32_t i) {  // dP^T(i) = V dO(i)^T, once dQ(i-1) has left the columns
        ptx::mbar_wait(dq_free, (i & 1) ^ 1);
        ptx::tc_fence_after();
        ATR(0, i);
#pragma unroll
        for (int k = 0; k < 8; ++k) ptx::umma_bf16(tmem + kB2TDP, kdesc128(sv, k), kdesc128(sdo(i), k), id_ss, k > 0);
        ptx::umma_commit(dp_full);
      };
      auto tcol = [](int k) { return uint32_t(k < 4 ? 8 * k : 64 + 8 * (k - 4)); };  // packed query columns
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++item) {
        const AttnTask tk = group_task(t, nz, nt, false);
        const int n = nt - tk.tile;  // query tiles of this key tile
        ptx::mbar_wait(kv_full, item & 1);
        issue_st(it);
        issue_dpt(it);
        for (int q = 0; q < n; ++q, ++it) {
          const bool first = q == 0, last = q + 1 == n;
          if (first) ptx::mbar_wait(acc_free, (item & 1) ^ 1);  // previous task's dK/dV read out
          ptx::mbar_wait(pt_full, it & 1);
          ptx::tc_fence_after();
          ATR(1, it);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::umma_bf16_ts(tmem + kB2TDV, tmem + kB2TS + tcol(k), mndesc(sdo(it), k), id_t, !first || k > 0);
          if (!last) issue_st(it + 1);  // overwrites P^T only after dV (in-order tensor pipe)
          ptx::mbar_wait(dst_full, it & 1);
          ptx::tc_fence_after();
          ATR(3, it);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::umma_bf16_ts(tmem + kB2TDK, tmem + kB2TDP + tcol(k), mndesc(sq(it), k), id_t, !first || k > 0);
          ptx::umma_commit(&qd_empty[it & 1]);  // Q(i), dO(i) are not dQ operands: release the stage now
          ptx::mbar_wait(ds_full, it & 1);
          ptx::tc_fence_after();
          ATR(4, it);
#pragma unroll
          for (int k = 0; k < 8; ++k)  // dQ^T = K^T dS'^T (head dims on the lanes)
            ptx::umma_bf16(tmem + kB2TDP, mndesc(sk, k), mndesc(sds, k), id_q, k > 0);
          ptx::umma_commit(mm_done);
          if (last) {
            ptx::umma_commit(acc_full);
            ptx::umma_commit(kv_empty);
          } else {
            issue_dpt(it + 1);
          }
        }
      }
    }
  } else if (warp < 8) {  // ------------------------------------------ P^T / dS'^T builders
    const int q4 = warp & 3, qh = warp >> 2;
    const int r = q4 * 32 + lane;  // key row of the tile == TMEM lane
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    const uint32_t sds = ptx::smem_u32(sm + B2Smem::kDS);
    const float sl2 = scale * kLog2e;
    uint32_t it = 0;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
      const AttnTask tk = group_task(t, nz, nt, false);
      for (int i = tk.tile; i < nt; ++i, ++it) {
        const float* ld = reinterpret_cast<const float*>(sm + B2Smem::kLD + (it & 1) * 1024);
        ptx::mbar_wait(s_full, it & 1);  // S^T(i) landed; Q(i) / LSE(i) are in this stage
        ptx::tc_fence_after();
        if (warp == 0 && lane == 0) ATR(5, it);
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t vs[32];
          ptx::tmem_ld_32x32b_x32(tmem + kB2TS + lane_off + qh * 64 + c * 32, vs);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const int q = qh * 64 + c * 32 + e;
            const float4 l4 = lds_v4(ld + q);  // LSE of queries q..q+3 (broadcast)
            float p[4] = {ex2(fmaf(__uint_as_float(vs[e]), sl2, -l4.x * kLog2e)),
                          ex2(fmaf(__uint_as_float(vs[e + 1]), sl2, -l4.y * kLog2e)),
                          ex2(fmaf(__uint_as_float(vs[e + 2]), sl2, -l4.z * kLog2e)),
                          ex2(fmaf(__uint_as_float(vs[e + 3]), sl2, -l4.w * kLog2e))};
            if (i == tk.tile) {  // diagonal tile: key r > query q gives P = 0
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (r > q + u) p[u] = 0.f;
            }
            pk[c * 16 + e / 2] = pack_bf16(p[0], p[1]);
            pk[c * 16 + e / 2 + 1] = pack_bf16(p[2], p[3]);
          }
          // P^T over this half's S^T, chunk by chunk: chunk c's 16 packed columns land on S^T columns
          // already read (chunk 1's scores sit in columns 32..63), so the store overlaps the next load
          ptx::tmem_st_32x32b_x16(tmem + kB2TS + lane_off + qh * 64 + c * 16,
                                  *reinterpret_cast<const uint32_t(*)[16]>(&pk[c * 16]));
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        if (warp == 0 && lane == 0) ATR(6, it);
        ptx::mbar_arrive(pt_full);
        // dS'^T = P^T (dP^T - D), from the bf16 P (the value the dV product also uses)
        ptx::mbar_wait(dp_full, it & 1);
        ptx::tc_fence_after();
        if (warp == 0 && lane == 0) ATR(7, it);
        uint32_t dk[32];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t vp[32];
          ptx::tmem_ld_32x32b_x32(tmem + kB2TDP + lane_off + qh * 64 + c * 32, vp);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const int q = qh * 64 + c * 32 + e;
            const float4 d4 = lds_v4(ld + 128 + q);  // D of queries q..q+3 (broadcast)
            const uint32_t pa = pk[c * 16 + e / 2], pb = pk[c * 16 + e / 2 + 1];
            dk[c * 16 + e / 2] = pack_bf16(__uint_as_float(pa << 16) * (__uint_as_float(vp[e]) - d4.x),
                                           __uint_as_float(pa & 0xffff0000u) * (__uint_as_float(vp[e + 1]) - d4.y));
            dk[c * 16 + e / 2 + 1] = pack_bf16(__uint_as_float(pb << 16) * (__uint_as_float(vp[e + 2]) - d4.z),
                                               __uint_as_float(pb & 0xffff0000u) * (__uint_as_float(vp[e + 3]) - d4.w));
          }
          ptx::tmem_st_32x32b_x16(tmem + kB2TDP + lane_off + qh * 64 + c * 16,
                                  *reinterpret_cast<const uint32_t(*)[16]>(&dk[c * 16]));
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        if (warp == 0 && lane == 0) ATR(8, it);
        ptx::mbar_arrive(dst_full);
        // dS'^T into shared memory: the B operand of dQ^T = K^T dS'^T. dQ^T(i-1) has finished reading
        // it: it precedes dP^T(i) in the in-order tensor pipe.
#pragma unroll
        for (int g = 0; g < 8; ++g)
          st_shared_v4(sds + p_off(r, qh * 64 + g * 8), dk[4 * g], dk[4 * g + 1], dk[4 * g + 2], dk[4 * g + 3]);
        fence_proxy_async();
        if (warp == 0 && lane == 0) ATR(10, it);
        ptx::mbar_arrive(ds_full);
      }
    }
  } else if (warp < 12) {  // ------------------------------------------ warps 8-11: dQ + dK/dV out
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;  // TMEM lane: head dim of dQ^T, key row of dK / dV
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    uint32_t it = 0, item = 0;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++item) {
      const AttnTask tk = group_task(t, nz, nt, false);
      const int smp = tk.z / heads, head = tk.z % heads;
      for (int i = tk.tile; i < nt; ++i, ++it) {
        ptx::mbar_wait(mm_done, it & 1);  // dQ^T(i) in TMEM
        ptx::tc_fence_after();
        if (warp == 8 && lane == 0) ATR(11, it);
        uint32_t v[4][32];
        ptx::tmem_ld_32x32b_x32(tmem + kB2TDP + lane_off, v[0]);
        ptx::tmem_ld_32x32b_x32(tmem + kB2TDP + lane_off + 32, v[1]);
        ptx::tmem_ld_32x32b_x32(tmem + kB2TDP + lane_off + 64, v[2]);
        ptx::tmem_ld_32x32b_x32(tmem + kB2TDP + lane_off + 96, v[3]);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        if (warp == 8 && lane == 0) ATR(12, it);
        ptx::mbar_arrive(dq_free);  // the MMA warp may put dP^T(i+1) into these columns
        // dQ^T: lane = head dim r, column = query. Lane pairs swap one value per query pair, so each
        // lane holds two adjacent head dims of one query: a red.v2 instruction adds two query rows'
        // 32 consecutive head dims (2 x 128 B, coalesced) into fp32 dQ. The reductions need no shared
        // memory, so nothing waits for them to drain.
        if (!(dbg & 1)) {
            const bool odd = lane & 1;
            float* dst = dq32 + (int64_t(smp) * seq + int64_t(i) * kT + (odd ? 1 : 0)) * h + head * kD2 +
                         q4 * 32 + (lane & ~1);
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float a0 = __uint_as_float(v[c][j]), a1 = __uint_as_float(v[c][j + 1]);
                const float got = __shfl_xor_sync(0xffffffffu, odd ? a0 : a1, 1);
                red_add_v2_f32(dst + int64_t(c * 32 + j) * h, odd ? got : a0, odd ? a1 : got);
              }
        }
        if (warp == 8 && lane == 0) ATR(13, it);
      }
      // epilogue: dK (scaled), dV rows of this key tile -> bf16 into dqkv. With rope_tab, dK leaves
      // through the inverse rotary embedding (the forward rotated K in the QKV GEMM epilogue):
      // column pairs (j, j + 64) are chunks c and c + 2 of the same thread's row.
      ptx::mbar_wait(acc_full, item & 1);
      ptx::tc_fence_after();
      const int64_t krow = int64_t(smp) * seq + int64_t(tk.tile) * kT + r;
      auto store32 = [&](bf16* dst, const uint32_t (&w)[32], float f) {  // bf16(f * w) (w: fp32 bits)
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(w[e]) * f, __uint_as_float(w[e + 1]) * f);
          u.y = pack_bf16(__uint_as_float(w[e + 2]) * f, __uint_as_float(w[e + 3]) * f);
          u.z = pack_bf16(__uint_as_float(w[e + 4]) * f, __uint_as_float(w[e + 5]) * f);
          u.w = pack_bf16(__uint_as_float(w[e + 6]) * f, __uint_as_float(w[e + 7]) * f);
          *reinterpret_cast<uint4*>(dst + e) = u;
        }
      };
      if (rope_tab) {
        bf16* dst = dqkv + krow * 3 * h + h + head * kD2;
        const float4* cs4 = reinterpret_cast<const float4*>(rope_tab + int64_t(tk.tile * kT + r) * (kD2 / 2));
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t ua[32], ub[32];
          ptx::tmem_ld_32x32b_x32(tmem + kB2TDK + lane_off + c * 32, ua);
          ptx::tmem_ld_32x32b_x32(tmem + kB2TDK + lane_off + 64 + c * 32, ub);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {  // in place; the softmax scale is applied by store32
            const float4 w = cs4[(c * 32 + e) >> 1];  // (cos, sin) of frequencies 32c + e, +1
            const float a0 = __uint_as_float(ua[e]), b0 = __uint_as_float(ub[e]);
            const float a1 = __uint_as_float(ua[e + 1]), b1 = __uint_as_float(ub[e + 1]);
            ua[e] = __float_as_uint(fmaf(a0, w.x, b0 * w.y));  // inverse rotation: a cos + b sin,
            ub[e] = __float_as_uint(fmaf(b0, w.x, -a0 * w.y));  //                   b cos - a sin
            ua[e + 1] = __float_as_uint(fmaf(a1, w.z, b1 * w.w));
            ub[e + 1] = __float_as_uint(fmaf(b1, w.z, -a1 * w.w));
          }
          store32(dst + c * 32, ua, scale);
          store32(dst + 64 + c * 32, ub, scale);
        }
      }
#pragma unroll 1
      for (int which = rope_tab ? 1 : 0; which < 2; ++which) {
        bf16* dst = dqkv + krow * 3 * h + (which == 0 ? h : 2 * h) + head * kD2;
        const uint32_t src = tmem + (which == 0 ? kB2TDK : kB2TDV) + lane_off;
        const float f = which == 0 ? scale : 1.f;  // dK = scale * dS'^T Q
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t w[32];
          ptx::tmem_ld_32x32b_x32(src + c * 32, w);
          ptx::tmem_ld_wait();
          store32(dst + c * 32, w, f);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(acc_free);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// D[z, q] = sum_d dO[q, head*D + d] * O[q, head*D + d]. One warp per token row: lane l reads
// 16-byte chunks l, l+32, ... (D/8 lanes per head per pass), reduced over groups of D/8 lanes.
template <int D>
__global__ void attn_dvec_kernel(const bf16* __restrict__ dO, const bf16* __restrict__ O, float* __restrict__ dvec,
                                 int64_t tokens, int seq, int heads) {
  static_assert(D == 64 || D == 128, "head_dim");
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  const int h = heads * D;
  const int nchunks = h / 8;  // 16-byte chunks per row; D / 8 chunks per head
  for (int64_t tok = blockIdx.x * int64_t(blockDim.x / 32) + threadIdx.x / 32; tok < tokens; tok += warps) {
    const int64_t smp = tok / seq;
    const int q = int(tok % seq);
    for (int k = 0; k * 32 < nchunks; ++k) {
      const int chunk = lane + 32 * k;
      float v = 0.f;
      if (chunk < nchunks) {
        const uint4 a = *reinterpret_cast<const uint4*>(dO + tok * h + chunk * 8);
        const uint4 b = *reinterpret_cast<const uint4*>(O + tok * h + chunk * 8);
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 x = __bfloat1622float2(a2[e]), y = __bfloat1622float2(b2[e]);
          v += x.x * y.x + x.y * y.y;
        }
      }
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      if (D == 128) v += __shfl_xor_sync(0xffffffffu, v, 8);
      if ((lane & (D / 8 - 1)) == 0 && chunk < nchunks) {
        const int head = chunk / (D / 8);
        dvec[(smp * heads + head) * seq + q] = v;
      }
    }
  }
}

// dqkv[:, 0:h] (bf16, row stride 3h) = dq32 [T, h]
__global__ void attn_dq_cast_kernel(const float* __restrict__ dq32, bf16* __restrict__ dqkv, int64_t tokens, int h,
                                    float scale) {
  // 8 elements per item: two 16-byte loads, one 16-byte store
  const int per_row = h / 8;
  const int64_t n8 = tokens * per_row;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t tok = i / per_row;
    const int col = int(i - tok * per_row) * 8;
    const float4 a = reinterpret_cast<const float4*>(dq32)[2 * i], b = reinterpret_cast<const float4*>(dq32)[2 * i + 1];
    uint4 o;
    o.x = pack_bf16(a.x * scale, a.y * scale);  // dQ = scale * dS' K
    o.y = pack_bf16(a.z * scale, a.w * scale);
    o.z = pack_bf16(b.x * scale, b.y * scale);
    o.w = pack_bf16(b.z * scale, b.w * scale);
    *reinterpret_cast<uint4*>(dqkv + tok * 3 * h + col) = o;
  }
}

// The same cast through the inverse rotary embedding (head_dim D): one item = 8 rotation pairs
// (j, j + D/2) of one (token, head), read from fp32 dQ, rotated back by the token's position.
template <int D>
__global__ void attn_dq_cast_rope_kernel(const float* __restrict__ dq32, bf16* __restrict__ dqkv,
                                         const float2* __restrict__ tab, int64_t tokens, int seq, int h,
                                         float scale) {
  constexpr int half = D / 2, groups = half / 8;
  const int per_row = (h / D) * groups;
  const int64_t n = tokens * per_row;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t tok = i / per_row;
    const int r = int(i - tok * per_row);
    const int col = (r / groups) * D + (r % groups) * 8;  // head start + first pair's column
    const int j0 = (r % groups) * 8;
    const float4* pa = reinterpret_cast<const float4*>(dq32 + tok * h + col);
    const float4* pb = reinterpret_cast<const float4*>(dq32 + tok * h + col + half);
    const float4 a0 = pa[0], a1 = pa[1], b0 = pb[0], b1 = pb[1];
    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    const float4* cs = reinterpret_cast<const float4*>(tab + int64_t(tok % seq) * half + j0);
    float oa[8], ob[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 w = cs[k];  // (cos, sin) of pairs 2k, 2k + 1
      oa[2 * k] = scale * fmaf(a[2 * k], w.x, b[2 * k] * w.y);  // a cos + b sin
      ob[2 * k] = scale * fmaf(b[2 * k], w.x, -a[2 * k] * w.y);  // b cos - a sin
      oa[2 * k + 1] = scale * fmaf(a[2 * k + 1], w.z, b[2 * k + 1] * w.w);
      ob[2 * k + 1] = scale * fmaf(b[2 * k + 1], w.z, -a[2 * k + 1] * w.w);
    }
    bf16* d = dqkv + tok * 3 * h + col;
    *reinterpret_cast<uint4*>(d) = make_uint4(pack_bf16(oa[0], oa[1]), pack_bf16(oa[2], oa[3]),
                                              pack_bf16(oa[4], oa[5]), pack_bf16(oa[6], oa[7]));
    *reinterpret_cast<uint4*>(d + half) = make_uint4(pack_bf16(ob[0], ob[1]), pack_bf16(ob[2], ob[3]),
                                                     pack_bf16(ob[4], ob[5]), pack_bf16(ob[6], ob[7]));
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 2-D map over a row-major [rows, cols] bf16 matrix, box = 64 columns x 128 rows, SWIZZLE_128B.
bool map_rows(CUtensorMap* m, const void* base, int64_t rows, int64_t cols) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {cuuint64_t(cols), cuuint64_t(rows), 1, 1};
  cuuint64_t strides[3] = {cuuint64_t(cols * 2), cuuint64_t(rows * cols * 2), cuuint64_t(rows * cols * 2)};
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D map over a row-major [rows, cols] fp32 matrix, box = 32 columns (128 B) x 32 rows,
// SWIZZLE_128B (the dQ reduce-add target).
bool map_f32_rows(CUtensorMap* m, const void* base, int64_t rows, int64_t cols) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int device_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

cudaError_t attention_fwd_d128(const bf16* qkv, bf16* out, float* lse, int64_t batch, int seq, int heads,
                               int ctas, cudaStream_t s) {
  static int poly = -1;
  if (poly < 0) {
    const char* e = std::getenv("ZP_ATTN_POLY");
    poly = e ? std::max(0, std::min(2, std::atoi(e))) : kFwdPolyDefault;
  }
  auto kern = poly == 0 ? attn_fwd_d128_kernel<0> : poly == 1 ? attn_fwd_d128_kernel<1> : attn_fwd_d128_kernel<2>;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    for (auto k : {attn_fwd_d128_kernel<0>, attn_fwd_d128_kernel<1>, attn_fwd_d128_kernel<2>}) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, F2Smem::kBytes);
      if (e != cudaSuccess) return e;
    }
  }
  CUtensorMap m;
  const int h = heads * kD2;
  if (!map_rows(&m, qkv, batch * seq, 3 * h)) return cudaErrorInvalidValue;
  const int nz = int(batch) * heads;
  const int nb = (seq / kT + 1) / 2;
  const int ntasks = nb * nz;
  const int grid = std::min(ntasks, ctas > 0 ? std::min(ctas, device_sms()) : device_sms());
  const float scale_log2 = (1.0f / std::sqrt(float(kD2))) * kLog2e;
  kern<<<grid, kF2Threads, F2Smem::kBytes, s>>>(m, out, lse, seq, heads, nz, scale_log2);
  note_launch();
  return cudaGetLastError();
}

cudaError_t attention_fwd(const bf16* qkv, bf16* out, float* lse, int64_t batch, int seq, int heads,
                          int ctas, cudaStream_t s, int head_dim) {
  if (seq % kT || batch < 1 || (head_dim != 64 && head_dim != 128)) return cudaErrorInvalidValue;
  if (head_dim == 128) return attention_fwd_d128(qkv, out, lse, batch, seq, heads, ctas, s);
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         FwdSmem::kBytes);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap m;
  const int h = heads * kD;
  if (!map_rows(&m, qkv, batch * seq, 3 * h)) return cudaErrorInvalidValue;
  const int nz = int(batch) * heads;
  const int ntasks = (seq / kT) * nz;
  int grid = std::min((ntasks + kFwdPipes - 1) / kFwdPipes, ctas > 0 ? std::min(ctas, device_sms()) : device_sms());
  const float scale_log2 = (1.0f / std::sqrt(float(kD))) * kLog2e;
  attn_fwd_kernel<<<grid, kFwdThreads, FwdSmem::kBytes, s>>>(m, out, lse, seq, heads, nz, scale_log2);
  note_launch();
  return cudaGetLastError();
}

cudaError_t attention_bwd_d128(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, float* dvec,
                               float* dq32, bf16* dqkv, int64_t batch, int seq, int heads, int ctas, cudaStream_t s,
                               const float2* rope_tab, bool dvec_ready) {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_d128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         B2Smem::kBytes);
    if (e != cudaSuccess) return e;
  }
  const int h = heads * kD2;
  const int64_t T = batch * seq;
  CUtensorMap mq, md;
  if (!map_rows(&mq, qkv, T, 3 * h) || !map_rows(&md, dout, T, h)) return cudaErrorInvalidValue;
  const int cap = ctas > 0 ? std::min(ctas, device_sms()) : device_sms();
  if (!dvec_ready) {  // else the producer of dout (its GEMM epilogue) wrote D and cleared dq32
    attn_dvec_kernel<128><<<std::min<int64_t>(cap * 8, (T + 7) / 8), 256, 0, s>>>(dout, out, dvec, T, seq, heads);
    note_launch();
    cudaError_t e = cudaMemsetAsync(dq32, 0, size_t(T) * h * 4, s);
    if (e != cudaSuccess) return e;
  }
  const int nz = int(batch) * heads;
  const int ntasks = (seq / kT) * nz;
  const float scale = 1.0f / std::sqrt(float(kD2));
  static int dbg = -1;  // diagnostics (ZP_ATTN_DBG): bit 0 = skip the dQ reductions (wrong dQ)
  if (dbg < 0) dbg = std::getenv("ZP_ATTN_DBG") ? std::atoi(std::getenv("ZP_ATTN_DBG")) : 0;
  attn_bwd_d128_kernel<<<std::min(ntasks, cap), kB2Threads, B2Smem::kBytes, s>>>(mq, md, lse, dvec, dq32, dqkv,
                                                                                rope_tab, seq, heads, nz, scale, dbg);
  note_launch();
  if (rope_tab)
    attn_dq_cast_rope_kernel<kD2><<<std::min<int64_t>(cap * 4, (T * h / 16 + 255) / 256), 256, 0, s>>>(
        dq32, dqkv, rope_tab, T, seq, h, scale);
  else
    attn_dq_cast_kernel<<<std::min<int64_t>(cap * 4, (T * h / 8 + 255) / 256), 256, 0, s>>>(dq32, dqkv, T, h, scale);
  note_launch();
  return cudaGetLastError();
}

cudaError_t attention_bwd(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, float* dvec,
                          float* dq32, bf16* dqkv, int64_t batch, int seq, int heads, int ctas, cudaStream_t s,
                          int head_dim, const float2* rope_tab, bool dvec_ready) {
  if (seq % kT || batch < 1 || (head_dim != 64 && head_dim != 128)) return cudaErrorInvalidValue;
  if (head_dim == 128)
    return attention_bwd_d128(qkv, out, dout, lse, dvec, dq32, dqkv, batch, seq, heads, ctas, s, rope_tab,
                              dvec_ready);
  if (rope_tab || dvec_ready) return cudaErrorInvalidValue;  // head_dim 64: caller-side rotation and D
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         BwdSmem::kBytes);
    if (e != cudaSuccess) return e;
  }
  const int h = heads * kD;
  const int64_t T = batch * seq;
  CUtensorMap mq, md, mdq;
  if (!map_rows(&mq, qkv, T, 3 * h) || !map_rows(&md, dout, T, h) || !map_f32_rows(&mdq, dq32, T, h))
    return cudaErrorInvalidValue;
  const int cap = ctas > 0 ? std::min(ctas, device_sms()) : device_sms();
  attn_dvec_kernel<64><<<std::min<int64_t>(cap * 8, (T + 7) / 8), 256, 0, s>>>(dout, out, dvec, T, seq, heads);
  note_launch();
  cudaError_t e = cudaMemsetAsync(dq32, 0, size_t(T) * h * 4, s);
  if (e != cudaSuccess) return e;
  const int nz = int(batch) * heads;
  const int ntasks = (seq / kT) * nz;
  attn_bwd_kernel<<<std::min(ntasks, cap), kBwdThreads, BwdSmem::kBytes, s>>>(mq, md, mdq, lse, dvec, dqkv, seq,
                                                                          heads, nz, 1.0f / std::sqrt(float(kD)));
  note_launch();
  attn_dq_cast_kernel<<<std::min<int64_t>(cap * 4, (T * h / 8 + 255) / 256), 256, 0, s>>>(dq32, dqkv, T, h,
                                                                                       1.0f / std::sqrt(float(kD)));
  note_launch();
  return cudaGetLastError();
}

}  // namespace zp
