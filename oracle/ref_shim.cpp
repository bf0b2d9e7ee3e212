// ORACLE / TEST INFRASTRUCTURE — never linked into the product.
//
// C-ABI shim over the *reference's own* zeroplan sources, compiled in place from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/libzpref.so.
// It exports the zp_host.h functions with the prefix `zpref_`, marshalled by the same
// header (include/zp_host_marshal.inl) as the product, so a parity test feeds both
// libraries byte-identical inputs. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load this library.
//
// It also restates the reference acceptance suite's fuzz-instance generator
// (proj/tests/acceptance.cpp:72-110). The instances depend on libstdc++'s distribution
// algorithms, so they are generated here with the same compiler and library.
#include <cmath>
#include <random>

#include "zeroplan/comm.hpp"
#include "zeroplan/error.hpp"
#include "zeroplan/hardware.hpp"
#include "zeroplan/perf_curve.hpp"
#include "zeroplan/planner.hpp"
#include "zeroplan/profiler.hpp"
#include "zeroplan/simulator.hpp"
#include "zeroplan/spline.hpp"
#include "zeroplan/zero_stage.hpp"
#include "zp_host.h"

#define ZP_FN(name) zpref_##name
#define ZP_EXPORT __attribute__((visibility("default")))
#include "zp_host_marshal.inl"

extern "C" ZP_EXPORT int zpref_fuzz_instance(uint64_t index, zp_cluster* c, zp_model* m,
                                             int64_t* gbs, int32_t* stage_request) {
  // Draw order follows proj/tests/acceptance.cpp:72-110 exactly.
  std::mt19937_64 rng(0x5eed0000 + index);
  std::uniform_int_distribution<int> n_dist(1, 6);
  std::uniform_int_distribution<std::int64_t> mbs_dist(1, 64);
  std::uniform_int_distribution<std::int64_t> act_dist(1 << 20, 1 << 26);
  std::uniform_real_distribution<double> c0_dist(0.01, 0.3);
  std::uniform_real_distribution<double> c1_dist(0.005, 0.2);
  std::uniform_real_distribution<double> bw_dist(8.0, 11.0);
  std::uniform_real_distribution<double> lat_dist(0.0, 1e-3);
  std::uniform_int_distribution<std::int64_t> gbs_dist(1, 512);
  std::uniform_int_distribution<int> stage_dist(-1, 3);

  const int n = n_dist(rng);
  zeroplan::ModelSpec model;
  model.param_count = static_cast<double>(n) * 100000.0;
  model.hidden_size = 256;
  model.num_layers = 4;
  const double resident = zeroplan::resident_state_bytes(model, zeroplan::ZeroStage::kStage0, n);
  std::memset(c, 0, sizeof(*c));
  c->n = n;
  for (int i = 0; i < n; ++i) {
    zp_device_gt& d = c->devices[i];
    d.act_mem_per_batch = static_cast<double>(act_dist(rng));
    std::uniform_int_distribution<std::int64_t> slack_dist(
        0, static_cast<std::int64_t>(d.act_mem_per_batch) - 1);
    d.total_mem = resident + d.act_mem_per_batch * static_cast<double>(mbs_dist(rng)) +
                  static_cast<double>(slack_dist(rng));
    d.compute_fixed = c0_dist(rng);
    d.compute_per_batch = c1_dist(rng);
    d.optimizer_time = 0.0;
    c->link_bandwidths[i] = std::pow(10.0, bw_dist(rng));
  }
  c->link_latency = lat_dist(rng);
  *gbs = gbs_dist(rng);
  *stage_request = stage_dist(rng);
  m->param_count = model.param_count;
  m->hidden_size = model.hidden_size;
  m->num_layers = model.num_layers;
  m->bytes_per_param = model.bytes_per_param;
  m->optimizer_state_multiplier = model.optimizer_state_multiplier;
  return 0;
}
