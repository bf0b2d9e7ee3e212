// Poplar Alg. 1: per-stage time accounting, memory-probe mbs estimate, and the
// exponential + bisection max-batch search (reference profiler.cpp:25-171).
//
// The search is written as a resumable state machine (zeroplan_b200::MbsSearch) so
// the GPU profiler can drive all ranks in lockstep — one collective step per probe,
// each rank at its own probe batch — while issuing exactly the probe sequence the
// reference's sequential loop would (SURVEY.md §7 hard part 2).
#include "profiler_search.hpp"

#include <cmath>
#include <map>

namespace zeroplan {

double time_consumed_during_step(const StepTrace& t, ZeroStage stage) {
  // Stage-dependent wall path minus the collectives on it. The
  // add-then-subtract is kept literally: acceptance c3 compares against exactly this.
  double wall = t.forward_compute + t.backward_compute;
  double excluded = 0.0;
  if (stage == ZeroStage::kStage2) {
    wall += t.reduce_scatter;
    excluded = t.reduce_scatter;
  } else if (stage == ZeroStage::kStage3) {
    wall += t.fwd_allgather + t.bwd_allgather + t.reduce_scatter;
    excluded = t.fwd_allgather + t.bwd_allgather + t.reduce_scatter;
  }
  const double own = wall - excluded;
  if (own < 0.0) throw InternalError("negative compute time after collective subtraction");
  return own;
}

std::optional<std::int64_t> mbs_from_probe(const MemoryProbe& p) {
  const double per_batch = p.after_forward - p.before_forward;
  const double fits = std::floor((p.total - p.before_forward) / per_batch);
  const double bounded = std::min(fits, 1e15);  // keep the int cast exact (< 2^53)
  return std::max<std::int64_t>(static_cast<std::int64_t>(bounded), 1);
}

std::optional<std::int64_t> estimate_theoretical_mbs(const ClusterGroundTruth& cluster,
                                                     int device_id, const ModelSpec& model,
                                                     ZeroStage stage) {
  const auto p = memory_probe(cluster, device_id, model, stage);
  if (!p) return std::nullopt;
  return mbs_from_probe(*p);
}

// ------------------------------------------------------------------ MbsSearch

MbsSearch::MbsSearch(std::int64_t estimate) : estimate_(estimate) {
  if (estimate < 1) throw InvalidInputError("mbs_estimate must be >= 1");
}

std::int64_t MbsSearch::next_batch() const {
  if (phase_ == Phase::kGrow) return grow_;
  return lo_ + (hi_ - lo_ + 1) / 2;  // upper middle
}

void MbsSearch::record(std::int64_t batch, std::optional<double> step_time, double optimizer_time) {
  ++probes_;
  const bool ok = step_time.has_value();
  if (ok) {
    times_[batch] = *step_time;
    optimizer_time_ = optimizer_time;
  }
  if (phase_ == Phase::kGrow) {
    if (ok) {
      last_ok_ = batch;
      if (batch == estimate_) return finish(last_ok_);
      grow_ = std::min(batch * 2, estimate_);
      return;
    }
    if (last_ok_ == 0) throw InternalError("search_mbs: batch size 1 does not fit");
    // The largest workable batch lies in [last_ok, batch).
    lo_ = last_ok_;
    hi_ = batch - 1;
    phase_ = Phase::kBisect;
    if (!(lo_ < hi_)) finish(lo_);
    return;
  }
  if (ok)
    lo_ = batch;
  else
    hi_ = batch - 1;
  if (!(lo_ < hi_)) finish(lo_);
}

void MbsSearch::finish(std::int64_t mbs) {
  phase_ = Phase::kDone;
  mbs_ = mbs;
}

SearchResult MbsSearch::result() const {
  SearchResult r;
  r.mbs = mbs_;
  r.probes_used = probes_;
  r.optimizer_time = optimizer_time_;
  for (const auto& [b, t] : times_)
    if (b <= mbs_) r.samples.push_back(BatchSample{b, t});
  return r;
}

SearchResult search_mbs(const ClusterGroundTruth& cluster, int device_id, const ModelSpec& model,
                        ZeroStage stage, std::int64_t mbs_estimate) {
  MbsSearch s(mbs_estimate);
  while (!s.done()) {
    const std::int64_t b = s.next_batch();
    const auto trace = run_step(cluster, device_id, model, b, stage);
    if (trace)
      s.record(b, time_consumed_during_step(*trace, stage), trace->optimizer_step);
    else
      s.record(b, std::nullopt, 0.0);
  }
  return s.result();
}

ProfileResult profile_cluster(const ClusterGroundTruth& cluster, const ModelSpec& model,
                              std::optional<ZeroStage> stage_request) {
  cluster.validate();
  model.validate();
  const int n = cluster.device_count();
  for (int s = stage_request ? stage_index(*stage_request) : 0; s <= 3; ++s) {
    const ZeroStage stage = stage_from_index(s);
    bool fits = true;
    for (int d = 0; d < n && fits; ++d) fits = memory_probe(cluster, d, model, stage).has_value();
    if (!fits) continue;  // a device cannot hold batch 1: escalate the stage
    ProfileResult out;
    out.effective_stage = stage;
    out.devices.reserve(static_cast<std::size_t>(n));
    for (int d = 0; d < n; ++d) {
      const auto est = estimate_theoretical_mbs(cluster, d, model, stage);
      if (!est) throw InternalError("memory probe and estimate disagree");
      SearchResult r = search_mbs(cluster, d, model, stage, *est);
      DeviceProfile p;
      p.device_id = d;
      p.mbs = r.mbs;
      p.samples = std::move(r.samples);
      p.probes_used = r.probes_used;
      p.optimizer_time = r.optimizer_time;
      out.devices.push_back(std::move(p));
    }
    return out;
  }
  throw InfeasibleError(
      "model too large: a single batch does not fit on every device even at ZeRO stage 3");
}

}  // namespace zeroplan
