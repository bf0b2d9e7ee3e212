// Resumable max-batch search shared by the latent profiler and the lockstep GPU profiler.
#pragma once
#include <cstdint>
#include <map>
#include <optional>

#include "zeroplan/zeroplan.hpp"

namespace zeroplan {

// floor((total - before) / (after - before)) capped to [1, 1e15] (reference profiler.cpp:49-60).
std::optional<std::int64_t> mbs_from_probe(const MemoryProbe& p);

// Probe sequence of reference search_mbs (profiler.cpp:62-127): 1, 2, 4, ... capped at the
// estimate; on the first OOM, upper-middle bisection over [last success, OOM batch - 1].
class MbsSearch {
 public:
  explicit MbsSearch(std::int64_t estimate);
  bool done() const { return phase_ == Phase::kDone; }
  std::int64_t next_batch() const;
  // step_time = nullopt means the probe ran out of memory.
  void record(std::int64_t batch, std::optional<double> step_time, double optimizer_time);
  SearchResult result() const;

 private:
  enum class Phase { kGrow, kBisect, kDone };
  void finish(std::int64_t mbs);
  std::int64_t estimate_;
  Phase phase_ = Phase::kGrow;
  std::int64_t grow_ = 1, last_ok_ = 0, lo_ = 0, hi_ = 0, mbs_ = 0;
  int probes_ = 0;
  double optimizer_time_ = 0.0;
  std::map<std::int64_t, double> times_;
};

}  // namespace zeroplan
