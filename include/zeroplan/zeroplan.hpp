// zeroplan host API on B200 — declarations.
//
// Same names, argument meaning and error behaviour as the reference planner's
// public C++ API (proj/core/include/zeroplan/*.hpp), so a caller of the reference
// can switch to this library unchanged. Two device back ends sit under the
// `run_step` / `memory_probe` seam (reference hardware.hpp:111-120):
//   * ClusterGroundTruth  — the reference's latent closed-form device model, kept as the
//                           test double that lets the host stack be parity-checked on CPU;
//   * the B200 runtime    — real sm_100a execution (csrc/cuda) behind the C ABI of
//                           include/zp_runtime.h; integration/hardware_b200.{hpp,cpp} binds it to
//                           the reference's own run_step / memory_probe signatures.
// Planner arithmetic (spline, curves, Alg. 2) reproduces the reference bit-for-bit:
// every floating-point operation keeps the reference's order.
#ifndef ZEROPLAN_B200_ZEROPLAN_HPP_
#define ZEROPLAN_B200_ZEROPLAN_HPP_

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace zeroplan {

// ------------------------------------------------------------------ errors
// Exception taxonomy of reference error.hpp:24-47 (exit codes 1 / 2 / internal).
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidInputError : Error {
  explicit InvalidInputError(const std::string& m) : Error(m) {}
};
struct InfeasibleError : Error {
  explicit InfeasibleError(const std::string& m) : Error(m) {}
};
struct InternalError : Error {
  explicit InternalError(const std::string& m) : Error(m) {}
};

// ------------------------------------------------------------------ ZeRO stage
// Reference zero_stage.hpp:27-50.
enum class ZeroStage : int { kStage0 = 0, kStage1 = 1, kStage2 = 2, kStage3 = 3 };
inline int stage_index(ZeroStage s) { return static_cast<int>(s); }
ZeroStage stage_from_index(int value);
inline bool shards_gradients(ZeroStage s) { return stage_index(s) >= 2; }
inline bool shards_parameters(ZeroStage s) { return s == ZeroStage::kStage3; }

// ------------------------------------------------------------------ device model types
// Reference hardware.hpp:33-99.
struct DeviceGroundTruth {
  int id = 0;
  std::string name;
  double total_mem = 0.0;
  double act_mem_per_batch = 0.0;
  double compute_fixed = 0.0;
  double compute_per_batch = 0.0;
  double optimizer_time = 0.0;
  friend bool operator==(const DeviceGroundTruth&, const DeviceGroundTruth&) = default;
};

struct ClusterGroundTruth {
  std::vector<DeviceGroundTruth> devices;
  std::vector<double> link_bandwidths;
  double link_latency = 0.0;
  std::uint64_t seed = 0;
  double jitter = 0.0;
  int device_count() const { return static_cast<int>(devices.size()); }
  void validate() const;
  friend bool operator==(const ClusterGroundTruth&, const ClusterGroundTruth&) = default;
};

struct ModelSpec {
  double param_count = 0.0;
  std::int64_t hidden_size = 0;
  std::int64_t num_layers = 0;
  double bytes_per_param = 2.0;
  double optimizer_state_multiplier = 16.0;
  void validate() const;
  friend bool operator==(const ModelSpec&, const ModelSpec&) = default;
};

struct StepTrace {
  double forward_compute = 0.0;
  double backward_compute = 0.0;
  double fwd_allgather = 0.0;
  double bwd_allgather = 0.0;
  double reduce_scatter = 0.0;
  double allreduce = 0.0;
  double optimizer_step = 0.0;
};

struct MemoryProbe {
  double before_forward = 0.0;
  double after_forward = 0.0;
  double total = 0.0;
};

double resident_state_bytes(const ModelSpec& model, ZeroStage stage, int n);

// Latent (test-double) device back end: reference hardware.cpp:144-203.
std::optional<StepTrace> run_step(const ClusterGroundTruth& cluster, int device_id,
                                  const ModelSpec& model, std::int64_t batch_size, ZeroStage stage,
                                  std::uint64_t noise_index = 0);
std::optional<MemoryProbe> memory_probe(const ClusterGroundTruth& cluster, int device_id,
                                        const ModelSpec& model, ZeroStage stage);

// ------------------------------------------------------------------ communication model
// Reference comm.hpp:25-84.
std::uint64_t ffn_comm_volume(std::int64_t hidden_size, std::int64_t layers);
std::uint64_t ffn_forward_volume(std::int64_t hidden_size, std::int64_t layers);
std::uint64_t ffn_backward_volume(std::int64_t hidden_size, std::int64_t layers);
double stage_comm_volume(const ModelSpec& model, ZeroStage stage);
double micro_step_comm_volume(const ModelSpec& model, ZeroStage stage);
double sync_comm_volume(const ModelSpec& model, ZeroStage stage);
double collective_time(double volume_bytes, const ClusterGroundTruth& cluster);
double micro_step_comm_time(const ModelSpec& model, ZeroStage stage,
                            const ClusterGroundTruth& cluster);
double sync_comm_time(const ModelSpec& model, ZeroStage stage, const ClusterGroundTruth& cluster);

struct CommProfile {
  ZeroStage stage = ZeroStage::kStage0;
  double volume_forward = 0.0;
  double volume_backward = 0.0;
  double volume_optimizer = 0.0;
  double time_per_step = 0.0;
  double sync_time = 0.0;
};
CommProfile make_comm_profile(const ModelSpec& model, ZeroStage stage,
                              const ClusterGroundTruth& cluster);

// ------------------------------------------------------------------ natural cubic spline
// Reference spline.hpp:25-79.
struct SamplePoint {
  double x = 0.0;
  double y = 0.0;
};

class CubicSpline {
 public:
  struct Segment {
    double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
  };
  double eval(double x) const;
  double first_derivative(double x) const;
  double second_derivative(double x) const;
  const std::vector<double>& knots() const { return x_; }
  const std::vector<double>& values() const { return y_; }
  const std::vector<Segment>& segments() const { return seg_; }

 private:
  friend CubicSpline fit_natural_spline(std::vector<SamplePoint> points);
  std::size_t locate(double x) const;
  std::vector<double> x_, y_;
  std::vector<Segment> seg_;
};

CubicSpline fit_natural_spline(std::vector<SamplePoint> points);
double eval_spline(const CubicSpline& spline, double x);

// ------------------------------------------------------------------ profiler (Alg. 1)
// Reference profiler.hpp:29-83.
struct BatchSample {
  std::int64_t batch = 0;
  double time = 0.0;
};
struct DeviceProfile {
  int device_id = 0;
  std::int64_t mbs = 0;
  std::vector<BatchSample> samples;
  int probes_used = 0;
  double optimizer_time = 0.0;
};
struct ProfileResult {
  ZeroStage effective_stage = ZeroStage::kStage0;
  std::vector<DeviceProfile> devices;
};
struct SearchResult {
  std::int64_t mbs = 0;
  std::vector<BatchSample> samples;
  int probes_used = 0;
  double optimizer_time = 0.0;
};

double time_consumed_during_step(const StepTrace& trace, ZeroStage stage);
std::optional<std::int64_t> estimate_theoretical_mbs(const ClusterGroundTruth& cluster,
                                                     int device_id, const ModelSpec& model,
                                                     ZeroStage stage);
SearchResult search_mbs(const ClusterGroundTruth& cluster, int device_id, const ModelSpec& model,
                        ZeroStage stage, std::int64_t mbs_estimate);
ProfileResult profile_cluster(const ClusterGroundTruth& cluster, const ModelSpec& model,
                              std::optional<ZeroStage> stage_request);

// ------------------------------------------------------------------ performance curves
// Reference perf_curve.hpp:32-85.
class PerfCurve {
 public:
  static constexpr double kPeakEpsilon = 0.05;
  static constexpr double kSpeedFloor = 1e-9;
  struct PeakRange {
    std::int64_t lo = 1;
    std::int64_t hi = 1;
  };
  int device_id() const { return device_id_; }
  std::int64_t mbs() const { return mbs_; }
  double peak_speed() const { return peak_speed_; }
  PeakRange peak_range() const { return peak_range_; }
  const std::optional<CubicSpline>& spline() const { return spline_; }
  const std::vector<BatchSample>& samples() const { return samples_; }
  double speed_at(double batch) const;
  double predict_step_time(std::int64_t b) const;
  std::int64_t find_max_batch_within_time(double t) const;
  const std::vector<double>& step_times() const { return times_; }

 private:
  friend PerfCurve build_curve(std::vector<BatchSample> samples, std::int64_t mbs, int device_id);
  int device_id_ = 0;
  std::int64_t mbs_ = 0;
  std::optional<CubicSpline> spline_;
  double constant_speed_ = 0.0;
  double peak_speed_ = 0.0;
  PeakRange peak_range_;
  std::vector<double> speeds_;
  std::vector<double> times_;
  std::vector<BatchSample> samples_;
};

PerfCurve build_curve(std::vector<BatchSample> samples, std::int64_t mbs, int device_id = 0);
std::vector<PerfCurve> build_curves(const ProfileResult& profile);

// ------------------------------------------------------------------ planner (Alg. 2)
// Reference planner.hpp:30-103.
struct PlanMetrics {
  double iteration_time = 0.0;
  std::vector<double> idle;
  std::vector<double> under_utilization;
  double objective = 0.0;
};
PlanMetrics compute_plan_metrics(const std::vector<double>& finish_times,
                                 const std::vector<double>& weights);

struct DeviceAllocation {
  int device_id = 0;
  std::int64_t b = 0;
  std::int64_t gmbs = 0;
  std::int64_t lbs = 0;
  double predicted_time = 0.0;
};

struct AllocationPlan {
  ZeroStage stage = ZeroStage::kStage0;
  std::int64_t gbs = 0;
  std::vector<DeviceAllocation> devices;
  std::int64_t gas = 1;
  PlanMetrics metrics;
  std::vector<double> weights;
  double predicted_wall_time = 0.0;
  std::int64_t device_gas(std::size_t i) const;
  std::int64_t total_assigned() const;
};

std::vector<std::int64_t> allocate_remainder(std::vector<std::int64_t> gmbs,
                                             const std::vector<PerfCurve>& curves,
                                             std::int64_t batch_remain);
AllocationPlan plan_zero01(std::int64_t gbs, const std::vector<PerfCurve>& curves);
AllocationPlan plan_zero23(std::int64_t gbs, const std::vector<PerfCurve>& curves,
                           const CommProfile& comm);
AllocationPlan plan(std::int64_t gbs, const ProfileResult& profile, ZeroStage stage,
                    const ModelSpec& model, const ClusterGroundTruth& cluster);
AllocationPlan make_uniform_plan(std::int64_t gbs, const std::vector<PerfCurve>& curves,
                                 ZeroStage stage, const CommProfile& comm, double optimizer_tail);
void attach_overheads(AllocationPlan& plan, const CommProfile& comm, double optimizer_tail);

// ------------------------------------------------------------------ iteration executor
// Reference simulator.hpp:31-63. `simulate_iteration` replays a plan against the latent
// back end; the B200 executor with the same report contract is zp_runtime_execute_iteration.
struct IterationReport {
  double iteration_time = 0.0;
  std::vector<double> busy;
  std::vector<double> idle;
  std::vector<double> compute;
  double comm_total = 0.0;
  double throughput = 0.0;
};
struct SimReport {
  int iterations = 0;
  IterationReport mean;
  double speedup_vs_baseline = 1.0;
};
IterationReport simulate_iteration(const ClusterGroundTruth& cluster, const ModelSpec& model,
                                   const AllocationPlan& plan, ZeroStage stage,
                                   std::uint64_t iteration_index = 0);
SimReport simulate_run(const ClusterGroundTruth& cluster, const ModelSpec& model,
                       const AllocationPlan& plan, ZeroStage stage, int iterations);
double compare_plans(const ClusterGroundTruth& cluster, const ModelSpec& model, ZeroStage stage,
                     const AllocationPlan& plan_a, const AllocationPlan& plan_b, int iterations);

}  // namespace zeroplan

#endif  // ZEROPLAN_B200_ZEROPLAN_HPP_
