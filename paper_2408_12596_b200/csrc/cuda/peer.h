// NVLink peer-memory collectives of the ZeRO synchronisation path.
//
// Every rank maps every other rank's arena (one cudaMalloc, exported with CUDA IPC) and a small
// flag block. The b_i/B-weighted gradient reduce-scatter is a PULL: the owner of a shard reads
// the peers' bf16 (or fp32) gradients of that shard over NVLink and sums them in fp32 (the b_i/B
// weight is already folded into each rank's loss scale 1/(B*s)). At the synchronisation point the
// same kernel runs AdamW on the owned shard and PUSHES the new bf16 parameters into every rank's
// parameter buffer, so reduce-scatter + optimizer + all-gather is one launch.
//
// Ordering: an entry barrier (each rank's gradients are final) and an exit barrier (no rank
// overwrites gradients or reads parameters that a peer is still pulling / pushing) made of
// epoch-stamped flags written with st.release.sys into the peers' flag blocks. Waits are
// bounded: a peer that never arrives traps the kernel instead of hanging the GPU.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace zp {

constexpr int kMaxPeers = 8;

struct PeerFlags {       // one per rank, IPC-mapped by every peer
  uint32_t ready[kMaxPeers];
  uint32_t done[kMaxPeers];
  uint32_t ctr;          // local CTA arrival counter of the exit barrier (wraps per launch)
  uint32_t pad[15];
  // ZeRO-3 copy-engine reduce-scatter (runtime.cu z3_reduce_async), written by stream memory
  // operations of the peers into this rank's block, waited on locally:
  uint32_t rs_ready[kMaxPeers][2];   // [peer][buffer]: peer's group gradient in that buffer is final
  uint32_t rs_pulled[kMaxPeers][2];  // [peer][buffer]: peer has copied its slice out of ours
};

struct PeerView {
  int n = 0, rank = 0;
  char* base[kMaxPeers] = {};        // every rank's arena base, mapped into this process
  PeerFlags* flags[kMaxPeers] = {};  // every rank's flag block
};

// Single-device emulation of all n ranks in ONE cooperative launch (test harness, include/
// zp_kernels.h): blocks [r*g, (r+1)*g) run rank r's instance, so instances that wait on one
// another are co-resident by construction. Rank r's per-rank pointers are the given (rank 0)
// pointers + r*stride bytes, its shard offset + r*shard elements. g == 0: a normal per-rank launch.
struct PeerEmu {
  int g = 0;
  int64_t stride = 0, shard = 0;
};

// acc[i] = (overwrite ? 0 : acc[i]) + sum_j src_j[shard_off + i], i < len. src_off = byte offset
// of src (bf16 [total]) inside every rank's arena.
cudaError_t peer_rs_accumulate(const PeerView& pv, int64_t src_off, int64_t shard_off, float* acc,
                               int64_t len, bool overwrite, uint32_t epoch, int ctas, cudaStream_t s,
                               const PeerEmu& emu = PeerEmu());

// g[i] = (acc ? acc[i] : 0) + sum_j src_j[shard_off + i] (src bf16, or fp32 when src_f32);
// AdamW on (p32, m, v)[i]; bf16(p32[i]) stored to every rank's p16 at element shard_off + i
// (p16_off = byte offset of p16 [total] in every arena). gout (optional) receives g (fp32).
cudaError_t peer_rs_adam_ag(const PeerView& pv, int64_t src_off, bool src_f32, int64_t shard_off,
                            const float* acc, float* p32, float* m, float* v, int64_t p16_off,
                            float* gout, int64_t len, const AdamParams& ap, uint32_t epoch, int ctas,
                            cudaStream_t s, const PeerEmu& emu = PeerEmu());

// dst[i] = src_j[...] gather: every rank's shard j (len elements of bf16 at byte offset
// src_off + j*len*2 ... ) is pulled into dst at element j*len. Used by ZeRO-3 group gathers.
cudaError_t peer_all_gather(const PeerView& pv, int64_t shard_src_off, bf16* dst, int64_t len,
                            uint32_t epoch, int ctas, cudaStream_t s, const PeerEmu& emu = PeerEmu());

}  // namespace zp
