/*
 * zp_host.h — C ABI over the zeroplan host API (profiler / curves / planner / executor).
 *
 * Plain structs with fixed capacity, caller-owned outputs, integer status codes, no
 * exceptions across the boundary. Each function mirrors one reference entry point and
 * maps its exception taxonomy (proj/core/include/zeroplan/error.hpp:24-47) onto codes:
 *
 *   ZP_OK 0 | ZP_EINVAL 1 (InvalidInputError) | ZP_EINFEASIBLE 2 (InfeasibleError)
 *   ZP_EINTERNAL 3 (InternalError) | ZP_OOM 4 (std::nullopt from run_step / memory_probe)
 *   ZP_ECUDA 5 | ZP_ENCCL 6
 *
 * The message of the last failure on the calling thread is returned by zp_last_error().
 * The oracle library built from the reference sources (oracle/_ref/libzpref.so) exports
 * the same functions with the prefix `zpref_` so parity tests can call both sides with
 * identical inputs.
 */
#ifndef ZP_HOST_H_
#define ZP_HOST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZP_OK 0
#define ZP_EINVAL 1
#define ZP_EINFEASIBLE 2
#define ZP_EINTERNAL 3
#define ZP_OOM 4
#define ZP_ECUDA 5
#define ZP_ENCCL 6

#define ZP_MAX_DEVICES 64
#define ZP_MAX_SAMPLES 128

/* reference hardware.hpp:33-63 (DeviceGroundTruth / ClusterGroundTruth) */
typedef struct zp_device_gt {
  double total_mem, act_mem_per_batch, compute_fixed, compute_per_batch, optimizer_time;
} zp_device_gt;

typedef struct zp_cluster {
  int32_t n;
  zp_device_gt devices[ZP_MAX_DEVICES];
  double link_bandwidths[ZP_MAX_DEVICES];
  double link_latency;
  uint64_t seed;
  double jitter;
} zp_cluster;

/* reference hardware.hpp:66-78 */
typedef struct zp_model {
  double param_count;
  int64_t hidden_size, num_layers;
  double bytes_per_param, optimizer_state_multiplier;
} zp_model;

/* reference hardware.hpp:85-99 */
typedef struct zp_step_trace {
  double forward_compute, backward_compute, fwd_allgather, bwd_allgather, reduce_scatter,
      allreduce, optimizer_step;
} zp_step_trace;

typedef struct zp_probe {
  double before_forward, after_forward, total;
} zp_probe;

/* reference comm.hpp:74-81 */
typedef struct zp_comm_profile {
  int32_t stage;
  double volume_forward, volume_backward, volume_optimizer, time_per_step, sync_time;
} zp_comm_profile;

/* reference profiler.hpp:29-56 */
typedef struct zp_sample {
  int64_t batch;
  double time;
} zp_sample;

typedef struct zp_device_profile {
  int32_t device_id;
  int64_t mbs;
  int32_t probes_used;
  double optimizer_time;
  int32_t n_samples;
  zp_sample samples[ZP_MAX_SAMPLES];
} zp_device_profile;

typedef struct zp_profile {
  int32_t effective_stage;
  int32_t n;
  zp_device_profile devices[ZP_MAX_DEVICES];
} zp_profile;

/* reference perf_curve.hpp:32-76 (speeds / step times are returned through caller arrays) */
typedef struct zp_curve_info {
  int32_t device_id;
  int64_t mbs;
  double peak_speed;
  int64_t peak_lo, peak_hi;
} zp_curve_info;

/* reference planner.hpp:30-65 */
typedef struct zp_device_alloc {
  int32_t device_id;
  int64_t b, gmbs, lbs;
  double predicted_time;
} zp_device_alloc;

typedef struct zp_allocation_plan {
  int32_t stage;
  int64_t gbs, gas;
  int32_t n;
  zp_device_alloc devices[ZP_MAX_DEVICES];
  double iteration_time;
  double idle[ZP_MAX_DEVICES];
  double under_utilization[ZP_MAX_DEVICES];
  double objective;
  double weights[ZP_MAX_DEVICES];
  double predicted_wall_time;
} zp_allocation_plan;

/* reference simulator.hpp:31-46 */
typedef struct zp_iteration_report {
  double iteration_time;
  int32_t n;
  double busy[ZP_MAX_DEVICES];
  double idle[ZP_MAX_DEVICES];
  double compute[ZP_MAX_DEVICES];
  double comm_total;
  double throughput;
} zp_iteration_report;

const char* zp_last_error(void);

/* Latent back end and cost model (reference hardware.cpp / comm.cpp). */
int zp_resident_state_bytes(const zp_model* model, int32_t stage, int32_t n, double* out);
int zp_run_step(const zp_cluster* c, int32_t device_id, const zp_model* m, int64_t batch,
                int32_t stage, uint64_t noise_index, zp_step_trace* out);
int zp_memory_probe(const zp_cluster* c, int32_t device_id, const zp_model* m, int32_t stage,
                    zp_probe* out);
int zp_collective_time(double volume, const zp_cluster* c, double* out);
int zp_make_comm_profile(const zp_model* m, int32_t stage, const zp_cluster* c,
                         zp_comm_profile* out);
int zp_ffn_volumes(int64_t hidden, int64_t layers, uint64_t out3[3]);

/* Profiler (reference profiler.cpp). stage_request < 0 = auto escalation. */
int zp_time_consumed_during_step(const zp_step_trace* t, int32_t stage, double* out);
int zp_estimate_theoretical_mbs(const zp_cluster* c, int32_t device_id, const zp_model* m,
                                int32_t stage, int64_t* out);
int zp_search_mbs(const zp_cluster* c, int32_t device_id, const zp_model* m, int32_t stage,
                  int64_t estimate, zp_device_profile* out);
int zp_profile_cluster(const zp_cluster* c, const zp_model* m, int32_t stage_request,
                       zp_profile* out);

/* Spline and curves (reference spline.cpp / perf_curve.cpp). segs_out: 4 doubles per segment. */
int zp_spline_fit(int32_t n, const double* xs, const double* ys, double* knots_out,
                  double* segs_out);
int zp_spline_eval(int32_t n, const double* xs, const double* ys, int32_t nq, const double* xq,
                   int32_t deriv, double* out);
int zp_build_curve(int32_t n_samples, const zp_sample* samples, int64_t mbs, int32_t device_id,
                   zp_curve_info* info, double* speeds_out, double* times_out);

/* Planner (reference planner.cpp). Curves are built from the profile's devices. */
int zp_plan(int64_t gbs, const zp_profile* profile, int32_t stage, const zp_model* m,
            const zp_cluster* c, zp_allocation_plan* out);
int zp_plan_zero01(int64_t gbs, const zp_profile* profile, zp_allocation_plan* out);
int zp_plan_zero23(int64_t gbs, const zp_profile* profile, const zp_comm_profile* comm,
                   zp_allocation_plan* out);
int zp_make_uniform_plan(int64_t gbs, const zp_profile* profile, int32_t stage,
                         const zp_comm_profile* comm, double optimizer_tail, zp_allocation_plan* out);
int zp_allocate_remainder(int32_t n, const int64_t* gmbs, const zp_profile* profile,
                          int64_t batch_remain, int64_t* out);

/* Latent executor (reference simulator.cpp). */
int zp_simulate_iteration(const zp_cluster* c, const zp_model* m, const zp_allocation_plan* plan,
                          int32_t stage, uint64_t iteration, zp_iteration_report* out);
int zp_simulate_run(const zp_cluster* c, const zp_model* m, const zp_allocation_plan* plan, int32_t stage,
                    int32_t iterations, zp_iteration_report* out);

#ifdef __cplusplus
}
#endif
#endif /* ZP_HOST_H_ */
