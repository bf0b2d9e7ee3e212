// B200 device back end for the reference's own zeroplan library (the drop-in at its device seam).
//
// The reference models every device with a latent closed form behind two free functions,
// `zeroplan::run_step` and `zeroplan::memory_probe` (proj/core/include/zeroplan/hardware.hpp:
// 111-120), called by profile_cluster (profiler.cpp:52, 74, 140) and simulate_iteration
// (simulator.cpp:33-34). A maintainer switches that library to real GPUs by compiling its
// unchanged hardware.cpp with the latent pair renamed
//     -Drun_step=latent_run_step -Dmemory_probe=latent_memory_probe
// and adding hardware_b200.cpp, which defines the seam functions again: while a `ScopedBackend`
// is alive they execute on the B200 ranks of a `Backend` (libzp.so, include/zp_runtime.h);
// otherwise they forward to the latent model, so every existing caller and test keeps working.
// oracle/Makefile builds exactly that (oracle/_ref/seam_b200) and INTEGRATION.md describes it.
//
// One process drives all ranks, one host thread per GPU per call (the C ABI is per rank and its
// collectives need every rank inside them). The reference calls run_step for one device at a
// time (profiler.cpp:150-164); the backend serves that sequential caller by running the probed
// device at its batch while every other rank sits out (batch 0) and still joins the stage's
// collectives, so ZeRO-2/3 probes are real collective steps.
#ifndef ZEROPLAN_HARDWARE_B200_HPP_
#define ZEROPLAN_HARDWARE_B200_HPP_

#include <cstdint>
#include <optional>
#include <vector>

#include "zeroplan/hardware.hpp"
#include "zeroplan/planner.hpp"
#include "zeroplan/profiler.hpp"
#include "zeroplan/simulator.hpp"
#include "zp_runtime.h"

namespace zeroplan::b200 {

struct RankConfig {
  int device = 0;                  // CUDA device ordinal
  int sm_budget = 0;               // emulated SM count (0 = all)
  std::int64_t hbm_cap_bytes = 0;  // emulated HBM capacity (0 = free memory - 4 GiB)
};

struct BackendConfig {
  zp_gpt_config model{};  // the decoder every rank trains (include/zp_runtime.h)
  std::vector<RankConfig> ranks;
  std::uint64_t seed = 0;
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.0f;
};

class Backend {
 public:
  explicit Backend(const BackendConfig& cfg);
  ~Backend();
  Backend(const Backend&) = delete;
  Backend& operator=(const Backend&) = delete;

  int size() const { return static_cast<int>(rt_.size()); }
  zp_runtime* rank(int i) const { return rt_[static_cast<std::size_t>(i)]; }
  // True GPT parameter count (what ModelSpec::param_count must say).
  double param_count() const { return param_count_; }

  // Reference run_step semantics for one device: `device_id` runs `batch`, every other rank sits
  // out with batch 0 and joins the collectives. nullopt = the device's arena refused the batch.
  std::optional<StepTrace> run_step(int device_id, std::int64_t batch, ZeroStage stage);
  // Batch-1 forward high-water marks of one rank (local, no collectives).
  std::optional<MemoryProbe> memory_probe(int device_id, ZeroStage stage);
  // Alg. 1 with every rank probing in lockstep (zp_runtime_profile); same result type as the
  // reference's profile_cluster.
  ProfileResult profile_cluster(std::optional<ZeroStage> stage_request);
  // One real iteration of `plan` on every rank (samples synthesised on device, contiguous per
  // rank); the measured IterationReport: busy_i = compute_i + sum over collectives of the
  // fastest rank's time + optimizer_i, T = max wall, idle_i = T - busy_i, throughput = gbs / T.
  IterationReport execute_iteration(const AllocationPlan& plan, ZeroStage stage,
                                    std::uint64_t iteration = 0);

 private:
  template <class F>
  void on_all_ranks(F&& f);
  std::vector<zp_runtime*> rt_;
  double param_count_ = 0.0;
};

// While alive, zeroplan::run_step / memory_probe for any cluster with `backend.size()` devices run
// on the backend (the cluster's latent device fields are then unused); one at a time.
class ScopedBackend {
 public:
  explicit ScopedBackend(Backend& backend);
  ~ScopedBackend();
  ScopedBackend(const ScopedBackend&) = delete;
  ScopedBackend& operator=(const ScopedBackend&) = delete;
};

Backend* active();

}  // namespace zeroplan::b200

#endif  // ZEROPLAN_HARDWARE_B200_HPP_
