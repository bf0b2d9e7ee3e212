// Device-seam check: the reference's own zeroplan pipeline (profile_cluster -> plan ->
// simulate_iteration, compiled from its unchanged sources) driving real B200 ranks through
// hardware_b200.cpp, and the product planner (libzp.so, zp_plan) re-planning the same measured
// profiles bit for bit. Built by oracle/Makefile into oracle/_ref/seam_b200; run by
// tests/test_seam_gpu.py. Prints one JSON object; exit code 0 iff every plan matches.
//
//   seam_b200 [--ranks N] [--stage S] [--gbs G] [--model tiny|gpt2-small] [--sm a,b,..]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "hardware_b200.hpp"
#include "zeroplan/error.hpp"
#include "zeroplan/planner.hpp"
#include "zeroplan/profiler.hpp"
#include "zeroplan/simulator.hpp"
#include "zp_host.h"

using namespace zeroplan;

namespace {

std::string num(double v) {
  if (std::isinf(v)) return "\"inf\"";
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::string plan_json(const AllocationPlan& p) {
  std::ostringstream o;
  o << "{\"gas\": " << p.gas << ", \"b\": [";
  for (std::size_t i = 0; i < p.devices.size(); ++i) o << (i ? ", " : "") << p.devices[i].b;
  o << "], \"gmbs\": [";
  for (std::size_t i = 0; i < p.devices.size(); ++i) o << (i ? ", " : "") << p.devices[i].gmbs;
  o << "], \"lbs\": [";
  for (std::size_t i = 0; i < p.devices.size(); ++i) o << (i ? ", " : "") << p.devices[i].lbs;
  o << "], \"predicted_wall_time\": " << num(p.predicted_wall_time) << "}";
  return o.str();
}

std::string report_json(const IterationReport& r) {
  std::ostringstream o;
  o << "{\"iteration_time\": " << num(r.iteration_time) << ", \"throughput\": " << num(r.throughput)
    << ", \"comm_total\": " << num(r.comm_total) << ", \"compute\": [";
  for (std::size_t i = 0; i < r.compute.size(); ++i) o << (i ? ", " : "") << num(r.compute[i]);
  o << "], \"idle\": [";
  for (std::size_t i = 0; i < r.idle.size(); ++i) o << (i ? ", " : "") << num(r.idle[i]);
  o << "]}";
  return o.str();
}

std::string profile_json(const ProfileResult& p) {
  std::ostringstream o;
  o << "{\"effective_stage\": " << stage_index(p.effective_stage) << ", \"devices\": [";
  for (std::size_t i = 0; i < p.devices.size(); ++i) {
    const DeviceProfile& d = p.devices[i];
    o << (i ? ", " : "") << "{\"mbs\": " << d.mbs << ", \"probes_used\": " << d.probes_used
      << ", \"optimizer_time\": " << num(d.optimizer_time) << ", \"samples\": [";
    for (std::size_t k = 0; k < d.samples.size(); ++k)
      o << (k ? ", " : "") << "[" << d.samples[k].batch << ", " << num(d.samples[k].time) << "]";
    o << "]}";
  }
  o << "]}";
  return o.str();
}

// The product planner (libzp.so C ABI) on the same profile; returns the fields that differ from
// the reference's plan (bitwise on every double).
std::vector<std::string> product_plan_diffs(std::int64_t gbs, const ProfileResult& p, ZeroStage stage,
                                            const ModelSpec& m, const ClusterGroundTruth& c,
                                            const AllocationPlan& ref) {
  static zp_profile zp;
  std::memset(&zp, 0, sizeof zp);
  zp.effective_stage = stage_index(p.effective_stage);
  zp.n = static_cast<int32_t>(p.devices.size());
  for (std::size_t i = 0; i < p.devices.size(); ++i) {
    const DeviceProfile& d = p.devices[i];
    zp.devices[i].device_id = d.device_id;
    zp.devices[i].mbs = d.mbs;
    zp.devices[i].probes_used = d.probes_used;
    zp.devices[i].optimizer_time = d.optimizer_time;
    zp.devices[i].n_samples = static_cast<int32_t>(d.samples.size());
    for (std::size_t k = 0; k < d.samples.size(); ++k) zp.devices[i].samples[k] = {d.samples[k].batch, d.samples[k].time};
  }
  zp_model zm{m.param_count, m.hidden_size, m.num_layers, m.bytes_per_param, m.optimizer_state_multiplier};
  static zp_cluster zc;
  std::memset(&zc, 0, sizeof zc);
  zc.n = c.device_count();
  for (int i = 0; i < zc.n; ++i) {
    const DeviceGroundTruth& d = c.devices[static_cast<std::size_t>(i)];
    zc.devices[i] = {d.total_mem, d.act_mem_per_batch, d.compute_fixed, d.compute_per_batch, d.optimizer_time};
    zc.link_bandwidths[i] = c.link_bandwidths[static_cast<std::size_t>(i)];
  }
  zc.link_latency = c.link_latency;
  zc.seed = c.seed;
  zc.jitter = c.jitter;
  static zp_allocation_plan out;
  std::vector<std::string> d;
  if (zp_plan(gbs, &zp, stage_index(stage), &zm, &zc, &out) != ZP_OK) {
    d.push_back(std::string("zp_plan failed: ") + zp_last_error());
    return d;
  }
  auto same = [](double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; };
  if (out.stage != stage_index(ref.stage)) d.push_back("stage");
  if (out.gbs != ref.gbs) d.push_back("gbs");
  if (out.gas != ref.gas) d.push_back("gas");
  if (out.n != static_cast<int32_t>(ref.devices.size())) d.push_back("n");
  for (std::size_t i = 0; i < ref.devices.size(); ++i) {
    const DeviceAllocation& r = ref.devices[i];
    const zp_device_alloc& q = out.devices[i];
    if (q.device_id != r.device_id || q.b != r.b || q.gmbs != r.gmbs || q.lbs != r.lbs ||
        !same(q.predicted_time, r.predicted_time))
      d.push_back("devices[" + std::to_string(i) + "]");
    if (!same(out.idle[i], ref.metrics.idle[i]) || !same(out.under_utilization[i], ref.metrics.under_utilization[i]) ||
        !same(out.weights[i], ref.weights[i]))
      d.push_back("metrics[" + std::to_string(i) + "]");
  }
  if (!same(out.iteration_time, ref.metrics.iteration_time)) d.push_back("iteration_time");
  if (!same(out.objective, ref.metrics.objective)) d.push_back("objective");
  if (!same(out.predicted_wall_time, ref.predicted_wall_time)) d.push_back("predicted_wall_time");
  return d;
}

std::string diffs_json(const std::vector<std::string>& d) {
  std::string s = "[";
  for (std::size_t i = 0; i < d.size(); ++i) s += (i ? ", \"" : "\"") + d[i] + "\"";
  return s + "]";
}

}  // namespace

int main(int argc, char** argv) {
  int ranks = 1, stage_i = 2;
  std::int64_t gbs = 24;
  std::string model_name = "tiny";
  std::vector<int> sms;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const char* v = argv[i + 1];
    if (k == "--ranks") ranks = std::atoi(v);
    else if (k == "--stage") stage_i = std::atoi(v);
    else if (k == "--gbs") gbs = std::atoll(v);
    else if (k == "--model") model_name = v;
    else if (k == "--sm") {
      std::stringstream ss(v);
      std::string t;
      while (std::getline(ss, t, ',')) sms.push_back(std::atoi(t.c_str()));
    }
  }
  if (argc > 1 && std::string(argv[1]) == "--latent") {
    // No backend active: the seam forwards to the reference's latent model (the renamed
    // hardware.cpp), so the unchanged pipeline must reproduce the reference library exactly.
    // Cluster = the reference's tests/data/mixed_cluster.json shape (2:1 speeds, 4 devices).
    ClusterGroundTruth cluster;
    const double c1[4] = {0.002, 0.002, 0.004, 0.004};
    for (int r = 0; r < 4; ++r) {
      DeviceGroundTruth d;
      d.id = r;
      d.total_mem = 80e9;
      d.act_mem_per_batch = 2e9;
      d.compute_fixed = 0.01;
      d.compute_per_batch = c1[r];
      d.optimizer_time = 0.005;
      cluster.devices.push_back(d);
      cluster.link_bandwidths.push_back(100e9);
    }
    cluster.link_latency = 1e-4;
    ModelSpec model;
    model.param_count = 1e9;
    model.hidden_size = 2048;
    model.num_layers = 24;
    std::printf("[");
    for (int st = 0; st < 4; ++st) {
      const ProfileResult p = profile_cluster(cluster, model, stage_from_index(st));
      const AllocationPlan a = plan(256, p, p.effective_stage, model, cluster);
      const IterationReport r = simulate_iteration(cluster, model, a, p.effective_stage);
      std::printf("%s{\"stage\": %d, \"profile\": %s, \"plan\": %s, \"report\": %s}", st ? ",\n " : "",
                  st, profile_json(p).c_str(), plan_json(a).c_str(), report_json(r).c_str());
    }
    std::printf("]\n");
    return 0;
  }
  try {
    b200::BackendConfig cfg;
    cfg.model = model_name == "gpt2-small" ? zp_gpt_config{12, 768, 12, 3072, 50257, 1024, 0}
                                           : zp_gpt_config{2, 256, 4, 1024, 512, 128, 0};
    cfg.seed = 1;
    for (int r = 0; r < ranks; ++r)
      cfg.ranks.push_back({r, sms.empty() ? 0 : sms[static_cast<std::size_t>(r) % sms.size()],
                           std::int64_t(model_name == "tiny" ? 8 : 60) << 30});
    b200::Backend backend(cfg);
    const ZeroStage stage = stage_from_index(stage_i);

    // The reference's cluster/model vocabulary. Under the backend only the device count and the
    // link model are read (by plan(), planner.cpp:343-347); one rank launches no collectives.
    ClusterGroundTruth cluster;
    for (int r = 0; r < ranks; ++r) {
      DeviceGroundTruth d;
      d.id = r;
      d.total_mem = 1.0;
      d.act_mem_per_batch = 1.0;
      d.compute_per_batch = 1.0;
      cluster.devices.push_back(d);
      cluster.link_bandwidths.push_back(ranks > 1 ? 770e9 : std::numeric_limits<double>::infinity());
    }
    cluster.link_latency = ranks > 1 ? 25e-6 : 0.0;
    ModelSpec model;
    model.param_count = backend.param_count();
    model.hidden_size = cfg.model.d_model;
    model.num_layers = cfg.model.n_layer;

    b200::ScopedBackend scope(backend);
    // (1) the reference's sequential profiler over the GPU seam
    const ProfileResult p1 = profile_cluster(cluster, model, stage);
    const AllocationPlan a1 = plan(gbs, p1, p1.effective_stage, model, cluster);
    const auto d1 = product_plan_diffs(gbs, p1, p1.effective_stage, model, cluster, a1);
    // (2) the reference's simulator replaying that plan through the GPU run_step
    const IterationReport s1 = simulate_iteration(cluster, model, a1, p1.effective_stage);
    // (3) lockstep profiling on all ranks, the reference's plan of it, and the real iteration
    const ProfileResult p2 = backend.profile_cluster(stage);
    const AllocationPlan a2 = plan(gbs, p2, p2.effective_stage, model, cluster);
    const auto d2 = product_plan_diffs(gbs, p2, p2.effective_stage, model, cluster, a2);
    const IterationReport e2 = backend.execute_iteration(a2, p2.effective_stage);
    // (4) OOM through the seam: a batch far above the measured mbs is std::nullopt
    const auto oom = run_step(cluster, 0, model, p1.devices[0].mbs * 64 + 64, p1.effective_stage, 0);

    std::printf("{\"ranks\": %d, \"model\": \"%s\", \"params\": %s, \"gbs\": %lld,\n", ranks, model_name.c_str(),
                num(backend.param_count()).c_str(), static_cast<long long>(gbs));
    std::printf(" \"reference_profile\": %s,\n \"reference_plan\": %s,\n \"plan_parity_reference_profile\": %s,\n",
                profile_json(p1).c_str(), plan_json(a1).c_str(), diffs_json(d1).c_str());
    std::printf(" \"reference_simulate_on_gpu\": %s,\n", report_json(s1).c_str());
    std::printf(" \"lockstep_profile\": %s,\n \"lockstep_plan\": %s,\n \"plan_parity_lockstep_profile\": %s,\n",
                profile_json(p2).c_str(), plan_json(a2).c_str(), diffs_json(d2).c_str());
    std::printf(" \"executed_iteration\": %s,\n \"oom_is_nullopt\": %s}\n", report_json(e2).c_str(),
                oom ? "false" : "true");
    return (d1.empty() && d2.empty() && !oom) ? 0 : 1;
  } catch (const Error& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 3;
  }
}
