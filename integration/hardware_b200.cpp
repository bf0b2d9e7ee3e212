// B200 device back end at the reference's device seam — see hardware_b200.hpp.
#include "hardware_b200.hpp"

#include <algorithm>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>

#include "zeroplan/error.hpp"

namespace zeroplan {

// The reference's own latent implementations (proj/core/src/hardware.cpp compiled with the pair
// renamed; see hardware_b200.hpp).
std::optional<StepTrace> latent_run_step(const ClusterGroundTruth& cluster, int device_id,
                                         const ModelSpec& model, std::int64_t batch_size,
                                         ZeroStage stage, std::uint64_t noise_index);
std::optional<MemoryProbe> latent_memory_probe(const ClusterGroundTruth& cluster, int device_id,
                                               const ModelSpec& model, ZeroStage stage);

namespace b200 {
namespace {

Backend* g_active = nullptr;
std::mutex g_mu;

// C-ABI status -> the reference's exception taxonomy (error.hpp:24-47).
[[noreturn]] void raise(int rc, const std::string& where) {
  const std::string msg = where + ": " + zp_runtime_last_error();
  switch (rc) {
    case ZP_EINVAL:
      throw InvalidInputError(msg);
    case ZP_EINFEASIBLE:
      throw InfeasibleError(msg);
    default:
      throw InternalError(msg);
  }
}

void check(int rc, const char* where) {
  if (rc != ZP_OK) raise(rc, where);
}

StepTrace to_trace(const zp_step_trace& t) {
  StepTrace s;
  s.forward_compute = t.forward_compute;
  s.backward_compute = t.backward_compute;
  s.fwd_allgather = t.fwd_allgather;
  s.bwd_allgather = t.bwd_allgather;
  s.reduce_scatter = t.reduce_scatter;
  s.allreduce = t.allreduce;
  s.optimizer_step = t.optimizer_step;
  return s;
}

ProfileResult to_profile(const zp_profile& p) {
  ProfileResult r;
  r.effective_stage = stage_from_index(p.effective_stage);
  for (int i = 0; i < p.n; ++i) {
    const zp_device_profile& d = p.devices[i];
    DeviceProfile o;
    o.device_id = d.device_id;
    o.mbs = d.mbs;
    o.probes_used = d.probes_used;
    o.optimizer_time = d.optimizer_time;
    for (int k = 0; k < d.n_samples; ++k) o.samples.push_back({d.samples[k].batch, d.samples[k].time});
    r.devices.push_back(std::move(o));
  }
  return r;
}

void to_c_plan(const AllocationPlan& p, zp_allocation_plan* o) {
  std::memset(o, 0, sizeof(*o));
  o->stage = stage_index(p.stage);
  o->gbs = p.gbs;
  o->gas = p.gas;
  o->n = static_cast<int32_t>(p.devices.size());
  for (std::size_t i = 0; i < p.devices.size() && i < ZP_MAX_DEVICES; ++i) {
    const DeviceAllocation& d = p.devices[i];
    o->devices[i] = {d.device_id, d.b, d.gmbs, d.lbs, d.predicted_time};
    if (i < p.metrics.idle.size()) o->idle[i] = p.metrics.idle[i];
    if (i < p.metrics.under_utilization.size()) o->under_utilization[i] = p.metrics.under_utilization[i];
    if (i < p.weights.size()) o->weights[i] = p.weights[i];
  }
  o->iteration_time = p.metrics.iteration_time;
  o->objective = p.metrics.objective;
  o->predicted_wall_time = p.predicted_wall_time;
}

}  // namespace

template <class F>
void Backend::on_all_ranks(F&& f) {
  std::vector<std::exception_ptr> err(rt_.size());
  std::vector<std::thread> th;
  for (std::size_t i = 0; i < rt_.size(); ++i)
    th.emplace_back([&, i] {
      try {
        f(static_cast<int>(i));
      } catch (...) {
        err[i] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

Backend::Backend(const BackendConfig& cfg) {
  const int n = static_cast<int>(cfg.ranks.size());
  if (n < 1 || n > ZP_MAX_DEVICES) throw InvalidInputError("backend needs 1..64 ranks");
  uint8_t id[128] = {};
  if (n > 1) check(zp_nccl_unique_id(id), "zp_nccl_unique_id");
  rt_.assign(static_cast<std::size_t>(n), nullptr);
  std::vector<int> rc(static_cast<std::size_t>(n), ZP_OK);
  std::vector<std::string> msg(static_cast<std::size_t>(n));
  // NCCL communicator setup is collective: every rank is created concurrently on its own thread
  std::vector<std::thread> th;
  for (int i = 0; i < n; ++i)
    th.emplace_back([&, i] {
      zp_runtime_desc d{};
      d.rank = i;
      d.world_size = n;
      d.device = cfg.ranks[static_cast<std::size_t>(i)].device;
      std::memcpy(d.nccl_id, id, sizeof(id));
      d.sm_budget = cfg.ranks[static_cast<std::size_t>(i)].sm_budget;
      d.hbm_cap_bytes = cfg.ranks[static_cast<std::size_t>(i)].hbm_cap_bytes;
      d.model = cfg.model;
      d.seed = cfg.seed;
      d.lr = cfg.lr;
      d.beta1 = cfg.beta1;
      d.beta2 = cfg.beta2;
      d.eps = cfg.eps;
      d.weight_decay = cfg.weight_decay;
      rc[static_cast<std::size_t>(i)] = zp_runtime_create(&d, &rt_[static_cast<std::size_t>(i)]);
      if (rc[static_cast<std::size_t>(i)] != ZP_OK) msg[static_cast<std::size_t>(i)] = zp_runtime_last_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < n; ++i)
    if (rc[static_cast<std::size_t>(i)] != ZP_OK) {
      for (zp_runtime* r : rt_)
        if (r) zp_runtime_destroy(r);
      rt_.clear();
      throw InternalError("zp_runtime_create (rank " + std::to_string(i) + "): " + msg[static_cast<std::size_t>(i)]);
    }
  int64_t padded = 0, logical = 0;
  check(zp_runtime_param_count(rt_[0], &padded, &logical), "zp_runtime_param_count");
  param_count_ = static_cast<double>(logical);
}

Backend::~Backend() {
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (g_active == this) g_active = nullptr;
  }
  for (zp_runtime* r : rt_)
    if (r) zp_runtime_destroy(r);
}

std::optional<StepTrace> Backend::run_step(int device_id, std::int64_t batch, ZeroStage stage) {
  std::vector<zp_step_trace> tr(rt_.size());
  std::vector<int> rc(rt_.size(), ZP_OK);
  std::vector<std::string> msg(rt_.size());
  on_all_ranks([&](int i) {
    const std::int64_t b = i == device_id ? batch : 0;  // the others sit out
    rc[static_cast<std::size_t>(i)] =
        zp_runtime_run_step(rt_[static_cast<std::size_t>(i)], b, stage_index(stage), batch, &tr[static_cast<std::size_t>(i)]);
    if (rc[static_cast<std::size_t>(i)] != ZP_OK) msg[static_cast<std::size_t>(i)] = zp_runtime_last_error();
  });
  for (std::size_t i = 0; i < rt_.size(); ++i) {
    const int r = rc[i];
    if (r == ZP_OK || (r == ZP_OOM && static_cast<int>(i) == device_id)) continue;
    throw InternalError("zp_runtime_run_step (rank " + std::to_string(i) + "): " + msg[i]);
  }
  if (rc[static_cast<std::size_t>(device_id)] == ZP_OOM) return std::nullopt;
  return to_trace(tr[static_cast<std::size_t>(device_id)]);
}

std::optional<MemoryProbe> Backend::memory_probe(int device_id, ZeroStage stage) {
  zp_probe p{};
  const int rc = zp_runtime_memory_probe(rt_[static_cast<std::size_t>(device_id)], stage_index(stage), &p);
  if (rc == ZP_OOM) return std::nullopt;
  check(rc, "zp_runtime_memory_probe");
  MemoryProbe m;
  m.before_forward = p.before_forward;
  m.after_forward = p.after_forward;
  m.total = p.total;
  return m;
}

ProfileResult Backend::profile_cluster(std::optional<ZeroStage> stage_request) {
  std::vector<zp_profile> out(rt_.size());
  std::vector<int> rc(rt_.size(), ZP_OK);
  std::vector<std::string> msg(rt_.size());
  const int req = stage_request ? stage_index(*stage_request) : -1;
  on_all_ranks([&](int i) {
    const std::size_t k = static_cast<std::size_t>(i);
    rc[k] = zp_runtime_profile(rt_[k], req, &out[k]);
    if (rc[k] != ZP_OK) msg[k] = zp_runtime_last_error();
  });
  for (std::size_t i = 0; i < rt_.size(); ++i)
    if (rc[i] != ZP_OK) {
      if (rc[i] == ZP_EINFEASIBLE) throw InfeasibleError(msg[i]);
      throw InternalError("zp_runtime_profile (rank " + std::to_string(i) + "): " + msg[i]);
    }
  return to_profile(out[0]);
}

IterationReport Backend::execute_iteration(const AllocationPlan& plan, ZeroStage stage, std::uint64_t iteration) {
  const std::size_t n = rt_.size();
  if (plan.devices.size() != n) throw InvalidInputError("plan does not match the backend's rank count");
  zp_allocation_plan cp;
  to_c_plan(plan, &cp);
  std::vector<zp_rank_timing> tm(n);
  std::vector<std::vector<double>> coll(n, std::vector<double>(1 << 16));
  std::vector<int> rc(n, ZP_OK);
  std::vector<std::string> msg(n);
  on_all_ranks([&](int i) {
    const std::size_t k = static_cast<std::size_t>(i);
    std::int64_t first = 0;
    for (std::size_t j = 0; j < k; ++j) first += plan.devices[j].gmbs;
    rc[k] = zp_runtime_load_tokens(rt_[k], nullptr, first, std::max<std::int64_t>(plan.devices[k].gmbs, 1), iteration, 0);
    if (rc[k] == ZP_OK) {
      tm[k].coll_times = coll[k].data();
      tm[k].coll_capacity = static_cast<int32_t>(coll[k].size());
      rc[k] = zp_runtime_execute_iteration(rt_[k], &cp, stage_index(stage), &tm[k]);
    }
    if (rc[k] != ZP_OK) msg[k] = zp_runtime_last_error();
  });
  for (std::size_t i = 0; i < n; ++i)
    if (rc[i] != ZP_OK) {
      if (rc[i] == ZP_EINVAL) throw InvalidInputError(msg[i]);
      throw InternalError("zp_runtime_execute_iteration (rank " + std::to_string(i) + "): " + msg[i]);
    }
  for (std::size_t i = 0; i < n; ++i)
    if (tm[i].coll_truncated || tm[i].n_collectives != tm[0].n_collectives)
      throw InternalError("ranks issued different collective counts (or the timing buffer overflowed)");
  // Collective k costs every rank the fastest rank's duration (the last to arrive does not wait);
  // anything above it on a faster rank is synchronisation idle.
  double floor = 0.0;
  for (int k = 0; k < tm[0].n_collectives; ++k) {
    double m = coll[0][static_cast<std::size_t>(k)];
    for (std::size_t i = 1; i < n; ++i) m = std::min(m, coll[i][static_cast<std::size_t>(k)]);
    floor += m;
  }
  IterationReport r;
  r.comm_total = floor;
  for (std::size_t i = 0; i < n; ++i) {
    r.compute.push_back(tm[i].compute);
    r.busy.push_back(tm[i].compute + floor + tm[i].optimizer);
    r.iteration_time = std::max(r.iteration_time, tm[i].wall);
  }
  for (std::size_t i = 0; i < n; ++i) r.idle.push_back(r.iteration_time - r.busy[i]);
  r.throughput = static_cast<double>(plan.total_assigned()) / r.iteration_time;
  return r;
}

ScopedBackend::ScopedBackend(Backend& backend) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_active) throw InvalidInputError("another B200 backend is already active");
  g_active = &backend;
}

ScopedBackend::~ScopedBackend() {
  std::lock_guard<std::mutex> lock(g_mu);
  g_active = nullptr;
}

Backend* active() {
  std::lock_guard<std::mutex> lock(g_mu);
  return g_active;
}

}  // namespace b200

// ---------------------------------------------------------------- the seam (hardware.hpp:111-120)
namespace {
b200::Backend* backend_for(const ClusterGroundTruth& cluster, const ModelSpec& model, int device_id) {
  b200::Backend* be = b200::active();
  if (!be || cluster.device_count() != be->size()) return nullptr;
  if (device_id < 0 || device_id >= cluster.device_count())
    throw InvalidInputError("device_id out of range: " + std::to_string(device_id));
  if (model.param_count != be->param_count())
    throw InvalidInputError("model.param_count: does not match the B200 backend's model (" +
                            std::to_string(be->param_count()) + ")");
  return be;
}
}  // namespace

std::optional<StepTrace> run_step(const ClusterGroundTruth& cluster, int device_id, const ModelSpec& model,
                                  std::int64_t batch_size, ZeroStage stage, std::uint64_t noise_index) {
  b200::Backend* be = backend_for(cluster, model, device_id);
  if (!be) return latent_run_step(cluster, device_id, model, batch_size, stage, noise_index);
  if (batch_size < 1) throw InvalidInputError("batch_size must be >= 1");
  return be->run_step(device_id, batch_size, stage);  // noise is real on hardware
}

std::optional<MemoryProbe> memory_probe(const ClusterGroundTruth& cluster, int device_id, const ModelSpec& model,
                                        ZeroStage stage) {
  b200::Backend* be = backend_for(cluster, model, device_id);
  if (!be) return latent_memory_probe(cluster, device_id, model, stage);
  return be->memory_probe(device_id, stage);
}

}  // namespace zeroplan
