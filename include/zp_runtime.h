/*
 * zp_runtime.h — C ABI of the B200 device back end: one runtime per rank (one process per
 * GPU), executing real heterogeneous-ZeRO micro-steps on sm_100a kernels with NCCL
 * collectives over NVLink.
 *
 * This is the drop-in for the reference's device seam:
 *   run_step         proj/core/include/zeroplan/hardware.hpp:111-114 -> zp_runtime_run_step
 *   memory_probe     proj/core/include/zeroplan/hardware.hpp:118-120 -> zp_runtime_memory_probe
 *   simulate_iteration  proj/core/include/zeroplan/simulator.hpp:49-52
 *                                                    -> zp_runtime_execute_iteration
 * with the same result structs (zp_step_trace / zp_probe / zp_iteration_report from
 * zp_host.h) and the same OOM signal (ZP_OOM instead of std::nullopt).
 *
 * Collective calls (run_step at stage 2/3, execute_iteration at every stage with world > 1)
 * must be made by every rank in the same order; a rank that sits out a micro-step passes
 * batch 0 and still joins the collectives with a zero gradient.
 */
#ifndef ZP_RUNTIME_H_
#define ZP_RUNTIME_H_

#include <stdint.h>

#include "zp_host.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Decoder config. arch 0: GPT-2 family (pre-LN LayerNorm with bias, learned positions, tied LM
 * head, GELU-tanh MLP, biases). arch 1: Llama family (RMSNorm, rotary positions theta 1e4,
 * SwiGLU MLP with d_ff hidden units, no biases, untied LM head). head_dim = d_model / n_head must be
 * 64 or 128. */
typedef struct zp_gpt_config {
  int32_t n_layer, d_model, n_head, d_ff, vocab, seq_len;
  int32_t arch;
} zp_gpt_config;

typedef struct zp_runtime_desc {
  int32_t rank, world_size, device;
  uint8_t nccl_id[128];       /* ncclUniqueId from rank 0; ignored when world_size == 1 */
  int32_t sm_budget;          /* emulated SM count: CTA cap of every kernel (0 = all SMs) */
  int64_t hbm_cap_bytes;      /* emulated HBM capacity of the rank's arena (0 = free - 4 GiB) */
  zp_gpt_config model;
  uint64_t seed;              /* weight-init seed */
  float lr, beta1, beta2, eps, weight_decay;
} zp_runtime_desc;

typedef struct zp_runtime zp_runtime;

/* Per-rank measured timings of one executed iteration (the local half of zp_iteration_report;
 * the caller combines ranks, e.g. with the comm-floor rule of DESIGN.md). */
typedef struct zp_rank_timing {
  double compute;        /* sum of forward+backward event time of this rank's micro-steps */
  double forward, backward;
  double comm;           /* sum of collective event time (includes waiting for slower ranks) */
  double optimizer;      /* AdamW (+ cast) event time */
  double wall;           /* first event to last event of the iteration on this rank */
  double loss_sum;       /* sum over this rank's tokens of CE / (B * seq) */
  int64_t micro_steps;   /* micro-steps with batch > 0 */
  int32_t n_collectives; /* collectives issued in the iteration (every one, never truncated) */
  int32_t coll_capacity; /* caller: entries available at coll_times (0 = do not record) */
  double* coll_times;    /* caller-owned [coll_capacity]: per-collective event durations in issue
                            order; the first min(n_collectives, coll_capacity) are filled and
                            coll_truncated is set when the buffer was too small */
  int32_t coll_truncated;
  int32_t pad_;
  double ag_fwd, ag_bwd, rs; /* sums of the ZeRO-3 forward / backward gathers and reduce-scatters */
  double sync;           /* synchronisation-point collective time (Z0/1 all-reduce, Z2 gather, or the
                            fused reduce-scatter + AdamW + all-gather kernel) */
} zp_rank_timing;

const char* zp_runtime_last_error(void);
int zp_nccl_unique_id(uint8_t out[128]);
int zp_runtime_create(const zp_runtime_desc* desc, zp_runtime** out);
int zp_runtime_destroy(zp_runtime* rt);

/* Flat parameter count (padded layout) and the true GPT parameter count. */
int zp_runtime_param_count(zp_runtime* rt, int64_t* padded, int64_t* logical);
/* Activation bytes of one micro-step of batch b (the arena reservation run_step makes). */
int zp_runtime_activation_bytes(zp_runtime* rt, int64_t batch, int64_t* out);
/* Bytes resident in the arena for ZeRO stage `stage` (params, grads, optimizer state, fixed
 * workspaces). */
int zp_runtime_resident_bytes(zp_runtime* rt, int32_t stage, int64_t* out);

/* Alg. 1 memory probe: allocator high-water mark before / after a batch-1 forward. Local. */
int zp_runtime_memory_probe(zp_runtime* rt, int32_t stage, zp_probe* out);

/* Token pool for the next step/iteration: `count` samples of seq_len+1 tokens. from_host=1
 * copies from `host_tokens` (pinned recommended); from_host=0 synthesises on device from
 * (seed, iteration, first_sample + j). */
int zp_runtime_load_tokens(zp_runtime* rt, const int32_t* host_tokens, int64_t first_sample,
                           int64_t count, uint64_t iteration, int32_t from_host);

/* One profiling step at local batch `batch` (0 = sit out): forward, backward, the stage's
 * micro-step collectives and the optimizer step, each timed with CUDA events.
 * Collective over ranks. Returns ZP_OOM (after joining the collectives with batch 0) when the
 * activation reservation exceeds the rank's HBM cap. */
int zp_runtime_run_step(zp_runtime* rt, int64_t batch, int32_t stage, int64_t global_batch,
                        zp_step_trace* out);

/* One training iteration of `plan` (zp_host.h AllocationPlan) on this rank: gas micro-steps
 * of b (then lbs) samples at stage 2/3, device_gas steps at stage 0/1, the stage's
 * collectives and the sharded AdamW update. Samples come from the token pool in order.
 * Collective over ranks. timing may be NULL. */
int zp_runtime_execute_iteration(zp_runtime* rt, const zp_allocation_plan* plan, int32_t stage,
                                 zp_rank_timing* timing);

/* Parity access. kind: 0 master fp32 params, 1 Adam m, 2 Adam v, 3 summed gradient of the last
 * iteration (fp32; needs zp_runtime_keep_grads(rt, 1) before it). Copies this rank's shard
 * [begin, end) of the flat layout to host `out` (capacity >= end - begin floats). */
int zp_runtime_get_state(zp_runtime* rt, int32_t kind, float* out, int64_t* begin, int64_t* end);
int zp_runtime_get_params_bf16(zp_runtime* rt, uint16_t* out); /* full bf16 params (Z3: owned slices) */
int zp_runtime_set_params(zp_runtime* rt, const float* full_fp32); /* resets master + bf16 copy */
int zp_runtime_keep_grads(zp_runtime* rt, int32_t on);
/* SM confinement of the rank: *sms = SMs its kernels may use, *green = 1 when a green context
 * (driver SM partition, a multiple of 8 SMs <= sm_budget) confines every kernel on the rank's
 * stream, including NCCL's and the HBM-bound ones; 0 = grid caps only (ZP_GREEN=0 or no support). */
int zp_runtime_sm_info(zp_runtime* rt, int32_t* sms, int32_t* green);
/* *on = 1 when the ZeRO-1/2/3 collectives run over NVLink peer memory (CUDA IPC mappings of every
 * rank's arena: pull reduce-scatter and all-gather, and the fused reduce-scatter + AdamW +
 * all-gather kernel at the ZeRO-1/2 synchronisation point),
 * 0 when they run over NCCL (world size 1, ZP_PEER=0, or a rank that cannot map its peers). */
int zp_runtime_peer_collectives(zp_runtime* rt, int32_t* on);
/* NVLink microbenchmark on the ZeRO-2 layout (every rank calls it with the same arguments):
 * which 0 = pull reduce-scatter of the bf16 gradient (peer_rs_acc_k), 1 = pull all-gather of the
 * bf16 parameter shards (peer_ag_k), 2 = copy-engine pulls of every peer's shard (the ZeRO-3
 * prefetch path). *seconds = mean device time per call over reps (CUDA events on the runtime
 * stream, after one warm-up call); *pulled = bytes this rank reads from its peers per call. */
int zp_runtime_bench_collective(zp_runtime* rt, int32_t which, int32_t reps, double* seconds, int64_t* pulled);
/* Measured alpha-beta link model for the planner's collective_time (reference comm.cpp:88-99:
 * latency + volume / min(link_bandwidths)), collective over ranks: the stage's reduce-scatter
 * path (NVLink pull kernel, or NCCL without peer access) timed on a 1 GiB bf16 buffer and on
 * n*256 elements, max over ranks. *latency = small-buffer time (s); *bandwidth = buffer bytes /
 * (large-buffer time - latency) (B/s), i.e. the reference's per-launch volume convention. */
int zp_runtime_link_model(zp_runtime* rt, int32_t stage, int32_t reps, double* bandwidth, double* latency);
/* Flat-layout ranges this rank owns, as (flat_begin, flat_end, shard_begin) triples: one range
 * at stages 0-2, one per parameter group (embedding, each layer, final LN) at stage 3, where the
 * shard buffers of zp_runtime_get_state are the concatenation of the owned slices. */
int zp_runtime_owned_ranges(zp_runtime* rt, int64_t* triples, int32_t cap, int32_t* count);
/* Flat-layout offset/shape of a named tensor ("wte", "wpe", "lnf_g", "lnf_b", "h{i}.ln1_g", ...,
 * "h{i}.w_qkv", "h{i}.b_qkv", "h{i}.w_o", "h{i}.b_o", "h{i}.w_fc", "h{i}.b_fc", "h{i}.w_proj",
 * "h{i}.b_proj", "h{i}.ln2_g", "h{i}.ln2_b"). */
int zp_runtime_tensor_info(zp_runtime* rt, const char* name, int64_t* offset, int64_t* rows,
                           int64_t* cols);
/* Poplar Alg. 1 on the real devices, collective over ranks: per-rank memory probe, mbs
 * estimate and the reference's exponential + bisection probe sequence (each probe a real
 * run_step), stage escalation when any rank cannot fit batch 1; the ranks' DeviceProfiles are
 * all-gathered so every rank returns the same ProfileResult (reference profile_cluster,
 * proj/core/src/profiler.cpp:129-171). stage_request < 0 = auto. */
int zp_runtime_profile(zp_runtime* rt, int32_t stage_request, zp_profile* out);
/* Device-side timing: record event `slot` (0..7) on the runtime stream; elapsed(a, b) waits for
 * b and returns the seconds between the two events. */
int zp_runtime_mark(zp_runtime* rt, int32_t slot);
int zp_runtime_elapsed(zp_runtime* rt, int32_t a, int32_t b, double* seconds);
/* Per-launch CUDA-event timing of the dense (linear-layer) GEMMs. mode 1: enable + reset,
 * 0: disable, 2: synchronise and return the summed algorithmic FLOPs, event seconds and launch
 * count since the last reset. */
int zp_runtime_gemm_stats(zp_runtime* rt, int32_t mode, double* flops, double* seconds,
                          int64_t* launches);
int zp_runtime_sync(zp_runtime* rt);

#ifdef __cplusplus
}
#endif
#endif /* ZP_RUNTIME_H_ */
