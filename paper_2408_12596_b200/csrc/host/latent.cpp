// Latent device model (test double) and the collective cost model.
//
// Restates reference hardware.cpp:29-203 and comm.cpp:36-144 operation for operation,
// because profiles measured through this back end must equal the reference's bit for bit.
// On the GPU the same seam is served by the CUDA runtime (csrc/cuda/runtime.cu).
#include <algorithm>
#include <string>

#include "zeroplan/zeroplan.hpp"

namespace zeroplan {

ZeroStage stage_from_index(int value) {
  if (value < 0 || value > 3)
    throw InvalidInputError("stage: must be 0, 1, 2 or 3, got " + std::to_string(value));
  return static_cast<ZeroStage>(value);
}

namespace {

// splitmix64 finaliser (reference hardware.cpp:29-34).
std::uint64_t splitmix(std::uint64_t v) {
  v += 0x9e3779b97f4a7c15ull;
  v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ull;
  v = (v ^ (v >> 27)) * 0x94d049bb133111ebull;
  return v ^ (v >> 31);
}

// Multiplicative timing noise in [1 - jitter, 1 + jitter) (reference hardware.cpp:36-47).
double noise_scale(const ClusterGroundTruth& c, int dev, ZeroStage s, std::int64_t b,
                   std::uint64_t index) {
  if (c.jitter <= 0.0) return 1.0;
  const std::uint64_t keys[4] = {static_cast<std::uint64_t>(dev),
                                 static_cast<std::uint64_t>(stage_index(s)),
                                 static_cast<std::uint64_t>(b), index};
  std::uint64_t h = c.seed;
  for (std::uint64_t k : keys) h = splitmix(h ^ k);
  const double u = static_cast<double>(h >> 11) * 0x1.0p-53;
  return 1.0 + c.jitter * (2.0 * u - 1.0);
}

const DeviceGroundTruth& device_ref(const ClusterGroundTruth& c, int id) {
  if (id < 0 || id >= c.device_count())
    throw InvalidInputError("device_id out of range: " + std::to_string(id));
  return c.devices[static_cast<std::size_t>(id)];
}

void fail_if(bool bad, const std::string& what) {
  if (bad) throw InvalidInputError(what);
}

}  // namespace

// Field checks in the reference's comparison direction (hardware.cpp:60-119), so NaN
// inputs are accepted or rejected exactly as the reference does.
void ClusterGroundTruth::validate() const {
  fail_if(devices.empty(), "cluster.devices: must contain at least one device");
  fail_if(link_bandwidths.size() != devices.size(),
          "cluster.link_bandwidths: must have one entry per device");
  for (std::size_t i = 0; i < devices.size(); ++i) {
    const DeviceGroundTruth& d = devices[i];
    const std::string at = "cluster.devices[" + std::to_string(i) + "].";
    fail_if(d.total_mem <= 0.0, at + "total_mem: must be positive");
    fail_if(d.act_mem_per_batch <= 0.0, at + "act_mem_per_batch: must be positive");
    fail_if(d.compute_fixed < 0.0, at + "compute_fixed: must be >= 0");
    fail_if(d.compute_per_batch <= 0.0, at + "compute_per_batch: must be positive");
    fail_if(d.optimizer_time < 0.0, at + "optimizer_time: must be >= 0");
  }
  for (std::size_t i = 0; i < link_bandwidths.size(); ++i)
    fail_if(link_bandwidths[i] <= 0.0,
            "cluster.link_bandwidths[" + std::to_string(i) + "]: must be positive");
  fail_if(link_latency < 0.0, "cluster.link_latency: must be >= 0");
  fail_if(jitter < 0.0 || jitter >= 1.0, "cluster.jitter: must be in [0, 1)");
}

void ModelSpec::validate() const {
  fail_if(param_count <= 0.0, "model.param_count: must be positive");
  fail_if(hidden_size <= 0, "model.hidden_size: must be positive");
  fail_if(num_layers <= 0, "model.num_layers: must be positive");
  fail_if(bytes_per_param <= 0.0, "model.bytes_per_param: must be positive");
  fail_if(optimizer_state_multiplier < 2.0 * bytes_per_param,
          "model.optimizer_state_multiplier: must cover parameter and gradient state "
          "(>= 2 * bytes_per_param)");
}

// ZeRO resident bytes per rank (reference hardware.cpp:121-142): stage s shards
// the optimizer state (s>=1), then gradients (s>=2), then parameters (s=3) over n.
double resident_state_bytes(const ModelSpec& model, ZeroStage stage, int n) {
  if (n < 1) throw InvalidInputError("device count must be >= 1");
  const double psi = model.param_count;
  const double p = model.bytes_per_param;
  const double g = model.bytes_per_param;
  const double opt = model.optimizer_state_multiplier - p - g;
  const double ranks = static_cast<double>(n);
  if (stage == ZeroStage::kStage0) return model.optimizer_state_multiplier * psi;
  if (stage == ZeroStage::kStage1) return (p + g) * psi + opt * psi / ranks;
  if (stage == ZeroStage::kStage2) return p * psi + (g + opt) * psi / ranks;
  return model.optimizer_state_multiplier * psi / ranks;
}

std::optional<StepTrace> run_step(const ClusterGroundTruth& cluster, int device_id,
                                  const ModelSpec& model, std::int64_t batch_size, ZeroStage stage,
                                  std::uint64_t noise_index) {
  const DeviceGroundTruth& dev = device_ref(cluster, device_id);
  if (batch_size < 1) throw InvalidInputError("batch_size must be >= 1");
  const double bsz = static_cast<double>(batch_size);
  const double resident = resident_state_bytes(model, stage, cluster.device_count());
  if (resident + dev.act_mem_per_batch * bsz > dev.total_mem) return std::nullopt;

  const double compute = (dev.compute_fixed + dev.compute_per_batch * bsz) *
                         noise_scale(cluster, device_id, stage, batch_size, noise_index);
  StepTrace t;
  t.forward_compute = compute / 3.0;
  t.backward_compute = compute * 2.0 / 3.0;
  t.optimizer_step = dev.optimizer_time;
  const double wire = model.param_count * model.bytes_per_param;
  switch (stage) {
    case ZeroStage::kStage0:
    case ZeroStage::kStage1:
      t.allreduce = collective_time(2.0 * wire, cluster);
      break;
    case ZeroStage::kStage2:
      t.reduce_scatter = collective_time(wire, cluster);
      t.allreduce = collective_time(wire, cluster);
      break;
    case ZeroStage::kStage3:
      t.fwd_allgather = collective_time(wire, cluster);
      t.bwd_allgather = collective_time(wire, cluster);
      t.reduce_scatter = collective_time(wire, cluster);
      break;
  }
  return t;
}

std::optional<MemoryProbe> memory_probe(const ClusterGroundTruth& cluster, int device_id,
                                        const ModelSpec& model, ZeroStage stage) {
  const DeviceGroundTruth& dev = device_ref(cluster, device_id);
  const double resident = resident_state_bytes(model, stage, cluster.device_count());
  if (resident + dev.act_mem_per_batch > dev.total_mem) return std::nullopt;
  return MemoryProbe{resident, resident + dev.act_mem_per_batch, dev.total_mem};
}

// ------------------------------------------------------------------ comm model

namespace {
std::uint64_t ffn_h(std::int64_t hidden, std::int64_t layers) {
  if (hidden < 1 || layers < 1)
    throw InvalidInputError("ffn volume requires hidden_size >= 1 and layers >= 1");
  return static_cast<std::uint64_t>(hidden);
}
double wire_bytes(const ModelSpec& m) { return m.param_count * m.bytes_per_param; }
}  // namespace

// Paper FFN volumes: 8 d h^2 forward, 16 d h^2 backward.
std::uint64_t ffn_forward_volume(std::int64_t hidden, std::int64_t layers) {
  const std::uint64_t h = ffn_h(hidden, layers);
  return 8ull * static_cast<std::uint64_t>(layers) * h * h;
}
std::uint64_t ffn_backward_volume(std::int64_t hidden, std::int64_t layers) {
  const std::uint64_t h = ffn_h(hidden, layers);
  return 16ull * static_cast<std::uint64_t>(layers) * h * h;
}
std::uint64_t ffn_comm_volume(std::int64_t hidden, std::int64_t layers) {
  return ffn_forward_volume(hidden, layers) + ffn_backward_volume(hidden, layers);
}

double stage_comm_volume(const ModelSpec& model, ZeroStage stage) {
  return (stage == ZeroStage::kStage3 ? 3.0 : 2.0) * wire_bytes(model);
}

double micro_step_comm_volume(const ModelSpec& model, ZeroStage stage) {
  if (stage == ZeroStage::kStage2) return wire_bytes(model);
  if (stage == ZeroStage::kStage3) return 3.0 * wire_bytes(model);
  return 0.0;
}

double sync_comm_volume(const ModelSpec& model, ZeroStage stage) {
  if (stage == ZeroStage::kStage0 || stage == ZeroStage::kStage1) return 2.0 * wire_bytes(model);
  if (stage == ZeroStage::kStage2) return wire_bytes(model);
  return 0.0;
}

// alpha-beta cost over the slowest link (reference comm.cpp:88-99).
double collective_time(double volume_bytes, const ClusterGroundTruth& cluster) {
  if (volume_bytes < 0.0) throw InvalidInputError("collective volume must be >= 0");
  if (cluster.link_bandwidths.empty())
    throw InvalidInputError("cluster.link_bandwidths: must not be empty");
  const double slowest =
      *std::min_element(cluster.link_bandwidths.begin(), cluster.link_bandwidths.end());
  return cluster.link_latency + volume_bytes / slowest;
}

double micro_step_comm_time(const ModelSpec& model, ZeroStage stage,
                            const ClusterGroundTruth& cluster) {
  if (stage == ZeroStage::kStage2) return collective_time(wire_bytes(model), cluster);
  // ZeRO-3: three separate launches (fwd AG, bwd AG, RS), each paying the latency.
  if (stage == ZeroStage::kStage3) return 3.0 * collective_time(wire_bytes(model), cluster);
  return 0.0;
}

double sync_comm_time(const ModelSpec& model, ZeroStage stage, const ClusterGroundTruth& cluster) {
  if (stage == ZeroStage::kStage3) return 0.0;
  return collective_time(sync_comm_volume(model, stage), cluster);
}

CommProfile make_comm_profile(const ModelSpec& model, ZeroStage stage,
                              const ClusterGroundTruth& cluster) {
  const double w = wire_bytes(model);
  CommProfile p;
  p.stage = stage;
  if (stage == ZeroStage::kStage0 || stage == ZeroStage::kStage1) {
    p.volume_optimizer = 2.0 * w;
  } else if (stage == ZeroStage::kStage2) {
    p.volume_backward = w;
    p.volume_optimizer = w;
  } else {
    p.volume_forward = w;
    p.volume_backward = 2.0 * w;
  }
  p.time_per_step = micro_step_comm_time(model, stage, cluster);
  p.sync_time = sync_comm_time(model, stage, cluster);
  return p;
}

}  // namespace zeroplan
