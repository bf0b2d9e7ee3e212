// Conversion between the zp_host.h C structs and the zeroplan C++ API, plus the
// exported C functions. Header-only on purpose: it is compiled twice —
//   * into libzp.so against include/zeroplan/zeroplan.hpp (prefix zp_), and
//   * into the oracle library against the reference's own headers (prefix zpref_),
// so both sides of a parity test are called through byte-identical marshalling.
// The including file defines ZP_FN(name) and includes the zeroplan headers first.
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <vector>

namespace zp_marshal {

namespace zpns = ::zeroplan;

inline thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const zpns::InvalidInputError& e) {
    g_last_error = e.what();
    return ZP_EINVAL;
  } catch (const zpns::InfeasibleError& e) {
    g_last_error = e.what();
    return ZP_EINFEASIBLE;
  } catch (const zpns::InternalError& e) {
    g_last_error = e.what();
    return ZP_EINTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ZP_EINTERNAL;
  }
}

inline zpns::ClusterGroundTruth to_cluster(const zp_cluster* c) {
  zpns::ClusterGroundTruth out;
  const int n = c->n < 0 ? 0 : (c->n > ZP_MAX_DEVICES ? ZP_MAX_DEVICES : c->n);
  for (int i = 0; i < n; ++i) {
    zpns::DeviceGroundTruth d;
    d.id = i;
    d.total_mem = c->devices[i].total_mem;
    d.act_mem_per_batch = c->devices[i].act_mem_per_batch;
    d.compute_fixed = c->devices[i].compute_fixed;
    d.compute_per_batch = c->devices[i].compute_per_batch;
    d.optimizer_time = c->devices[i].optimizer_time;
    out.devices.push_back(d);
    out.link_bandwidths.push_back(c->link_bandwidths[i]);
  }
  out.link_latency = c->link_latency;
  out.seed = c->seed;
  out.jitter = c->jitter;
  return out;
}

inline zpns::ModelSpec to_model(const zp_model* m) {
  zpns::ModelSpec s;
  s.param_count = m->param_count;
  s.hidden_size = m->hidden_size;
  s.num_layers = m->num_layers;
  s.bytes_per_param = m->bytes_per_param;
  s.optimizer_state_multiplier = m->optimizer_state_multiplier;
  return s;
}

inline zpns::StepTrace to_trace(const zp_step_trace* t) {
  zpns::StepTrace s;
  s.forward_compute = t->forward_compute;
  s.backward_compute = t->backward_compute;
  s.fwd_allgather = t->fwd_allgather;
  s.bwd_allgather = t->bwd_allgather;
  s.reduce_scatter = t->reduce_scatter;
  s.allreduce = t->allreduce;
  s.optimizer_step = t->optimizer_step;
  return s;
}

inline void from_trace(const zpns::StepTrace& s, zp_step_trace* t) {
  t->forward_compute = s.forward_compute;
  t->backward_compute = s.backward_compute;
  t->fwd_allgather = s.fwd_allgather;
  t->bwd_allgather = s.bwd_allgather;
  t->reduce_scatter = s.reduce_scatter;
  t->allreduce = s.allreduce;
  t->optimizer_step = s.optimizer_step;
}

inline zpns::CommProfile to_comm(const zp_comm_profile* c) {
  zpns::CommProfile p;
  p.stage = zpns::stage_from_index(c->stage);
  p.volume_forward = c->volume_forward;
  p.volume_backward = c->volume_backward;
  p.volume_optimizer = c->volume_optimizer;
  p.time_per_step = c->time_per_step;
  p.sync_time = c->sync_time;
  return p;
}

inline void from_comm(const zpns::CommProfile& p, zp_comm_profile* c) {
  c->stage = zpns::stage_index(p.stage);
  c->volume_forward = p.volume_forward;
  c->volume_backward = p.volume_backward;
  c->volume_optimizer = p.volume_optimizer;
  c->time_per_step = p.time_per_step;
  c->sync_time = p.sync_time;
}

inline void from_device_profile(int dev, std::int64_t mbs, const std::vector<zpns::BatchSample>& s,
                                int probes, double opt, zp_device_profile* o) {
  if (s.size() > ZP_MAX_SAMPLES) throw zpns::InternalError("too many samples for zp_device_profile");
  o->device_id = dev;
  o->mbs = mbs;
  o->probes_used = probes;
  o->optimizer_time = opt;
  o->n_samples = static_cast<int32_t>(s.size());
  for (std::size_t i = 0; i < s.size(); ++i) {
    o->samples[i].batch = s[i].batch;
    o->samples[i].time = s[i].time;
  }
}

inline zpns::ProfileResult to_profile(const zp_profile* p) {
  zpns::ProfileResult r;
  r.effective_stage = zpns::stage_from_index(p->effective_stage);
  for (int i = 0; i < p->n; ++i) {
    const zp_device_profile& d = p->devices[i];
    zpns::DeviceProfile o;
    o.device_id = d.device_id;
    o.mbs = d.mbs;
    o.probes_used = d.probes_used;
    o.optimizer_time = d.optimizer_time;
    for (int k = 0; k < d.n_samples; ++k) o.samples.push_back({d.samples[k].batch, d.samples[k].time});
    r.devices.push_back(std::move(o));
  }
  return r;
}

inline void from_plan(const zpns::AllocationPlan& p, zp_allocation_plan* o) {
  std::memset(o, 0, sizeof(*o));
  o->stage = zpns::stage_index(p.stage);
  o->gbs = p.gbs;
  o->gas = p.gas;
  o->n = static_cast<int32_t>(p.devices.size());
  for (std::size_t i = 0; i < p.devices.size(); ++i) {
    o->devices[i].device_id = p.devices[i].device_id;
    o->devices[i].b = p.devices[i].b;
    o->devices[i].gmbs = p.devices[i].gmbs;
    o->devices[i].lbs = p.devices[i].lbs;
    o->devices[i].predicted_time = p.devices[i].predicted_time;
    o->idle[i] = p.metrics.idle[i];
    o->under_utilization[i] = p.metrics.under_utilization[i];
    o->weights[i] = p.weights[i];
  }
  o->iteration_time = p.metrics.iteration_time;
  o->objective = p.metrics.objective;
  o->predicted_wall_time = p.predicted_wall_time;
}

inline zpns::AllocationPlan to_plan(const zp_allocation_plan* o) {
  zpns::AllocationPlan p;
  p.stage = zpns::stage_from_index(o->stage);
  p.gbs = o->gbs;
  p.gas = o->gas;
  for (int i = 0; i < o->n; ++i) {
    zpns::DeviceAllocation d;
    d.device_id = o->devices[i].device_id;
    d.b = o->devices[i].b;
    d.gmbs = o->devices[i].gmbs;
    d.lbs = o->devices[i].lbs;
    d.predicted_time = o->devices[i].predicted_time;
    p.devices.push_back(d);
    p.metrics.idle.push_back(o->idle[i]);
    p.metrics.under_utilization.push_back(o->under_utilization[i]);
    p.weights.push_back(o->weights[i]);
  }
  p.metrics.iteration_time = o->iteration_time;
  p.metrics.objective = o->objective;
  p.predicted_wall_time = o->predicted_wall_time;
  return p;
}

inline void from_report(const zpns::IterationReport& r, zp_iteration_report* o) {
  std::memset(o, 0, sizeof(*o));
  o->iteration_time = r.iteration_time;
  o->n = static_cast<int32_t>(r.busy.size());
  for (std::size_t i = 0; i < r.busy.size(); ++i) {
    o->busy[i] = r.busy[i];
    o->idle[i] = r.idle[i];
    o->compute[i] = r.compute[i];
  }
  o->comm_total = r.comm_total;
  o->throughput = r.throughput;
}

inline std::optional<zpns::ZeroStage> stage_req(int s) {
  if (s < 0) return std::nullopt;
  return zpns::stage_from_index(s);
}

}  // namespace zp_marshal

extern "C" {

ZP_EXPORT const char* ZP_FN(last_error)(void) { return zp_marshal::g_last_error.c_str(); }

ZP_EXPORT int ZP_FN(resident_state_bytes)(const zp_model* m, int32_t stage, int32_t n, double* out) {
  return zp_marshal::guarded([&] {
    *out = ::zeroplan::resident_state_bytes(zp_marshal::to_model(m), ::zeroplan::stage_from_index(stage), n);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(run_step)(const zp_cluster* c, int32_t dev, const zp_model* m, int64_t batch,
                              int32_t stage, uint64_t noise, zp_step_trace* out) {
  return zp_marshal::guarded([&] {
    const auto t = ::zeroplan::run_step(zp_marshal::to_cluster(c), dev, zp_marshal::to_model(m), batch,
                                        ::zeroplan::stage_from_index(stage), noise);
    if (!t) return ZP_OOM;
    zp_marshal::from_trace(*t, out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(memory_probe)(const zp_cluster* c, int32_t dev, const zp_model* m, int32_t stage,
                                  zp_probe* out) {
  return zp_marshal::guarded([&] {
    const auto p = ::zeroplan::memory_probe(zp_marshal::to_cluster(c), dev, zp_marshal::to_model(m),
                                            ::zeroplan::stage_from_index(stage));
    if (!p) return ZP_OOM;
    out->before_forward = p->before_forward;
    out->after_forward = p->after_forward;
    out->total = p->total;
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(collective_time)(double volume, const zp_cluster* c, double* out) {
  return zp_marshal::guarded([&] {
    *out = ::zeroplan::collective_time(volume, zp_marshal::to_cluster(c));
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(make_comm_profile)(const zp_model* m, int32_t stage, const zp_cluster* c,
                                       zp_comm_profile* out) {
  return zp_marshal::guarded([&] {
    zp_marshal::from_comm(::zeroplan::make_comm_profile(zp_marshal::to_model(m),
                                                        ::zeroplan::stage_from_index(stage),
                                                        zp_marshal::to_cluster(c)),
                          out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(ffn_volumes)(int64_t hidden, int64_t layers, uint64_t out3[3]) {
  return zp_marshal::guarded([&] {
    out3[0] = ::zeroplan::ffn_forward_volume(hidden, layers);
    out3[1] = ::zeroplan::ffn_backward_volume(hidden, layers);
    out3[2] = ::zeroplan::ffn_comm_volume(hidden, layers);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(time_consumed_during_step)(const zp_step_trace* t, int32_t stage, double* out) {
  return zp_marshal::guarded([&] {
    *out = ::zeroplan::time_consumed_during_step(zp_marshal::to_trace(t), ::zeroplan::stage_from_index(stage));
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(estimate_theoretical_mbs)(const zp_cluster* c, int32_t dev, const zp_model* m,
                                              int32_t stage, int64_t* out) {
  return zp_marshal::guarded([&] {
    const auto e = ::zeroplan::estimate_theoretical_mbs(zp_marshal::to_cluster(c), dev, zp_marshal::to_model(m),
                                                        ::zeroplan::stage_from_index(stage));
    if (!e) return ZP_OOM;
    *out = *e;
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(search_mbs)(const zp_cluster* c, int32_t dev, const zp_model* m, int32_t stage,
                                int64_t estimate, zp_device_profile* out) {
  return zp_marshal::guarded([&] {
    const auto r = ::zeroplan::search_mbs(zp_marshal::to_cluster(c), dev, zp_marshal::to_model(m),
                                          ::zeroplan::stage_from_index(stage), estimate);
    zp_marshal::from_device_profile(dev, r.mbs, r.samples, r.probes_used, r.optimizer_time, out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(profile_cluster)(const zp_cluster* c, const zp_model* m, int32_t stage_request,
                                     zp_profile* out) {
  return zp_marshal::guarded([&] {
    const auto r = ::zeroplan::profile_cluster(zp_marshal::to_cluster(c), zp_marshal::to_model(m),
                                               zp_marshal::stage_req(stage_request));
    out->effective_stage = ::zeroplan::stage_index(r.effective_stage);
    out->n = static_cast<int32_t>(r.devices.size());
    for (std::size_t i = 0; i < r.devices.size(); ++i) {
      const auto& d = r.devices[i];
      zp_marshal::from_device_profile(d.device_id, d.mbs, d.samples, d.probes_used, d.optimizer_time,
                                      &out->devices[i]);
    }
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(spline_fit)(int32_t n, const double* xs, const double* ys, double* knots_out,
                                double* segs_out) {
  return zp_marshal::guarded([&] {
    std::vector<::zeroplan::SamplePoint> pts;
    for (int i = 0; i < n; ++i) pts.push_back({xs[i], ys[i]});
    const auto s = ::zeroplan::fit_natural_spline(pts);
    for (std::size_t i = 0; i < s.knots().size(); ++i) knots_out[i] = s.knots()[i];
    for (std::size_t i = 0; i < s.segments().size(); ++i) {
      segs_out[4 * i + 0] = s.segments()[i].a;
      segs_out[4 * i + 1] = s.segments()[i].b;
      segs_out[4 * i + 2] = s.segments()[i].c;
      segs_out[4 * i + 3] = s.segments()[i].d;
    }
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(spline_eval)(int32_t n, const double* xs, const double* ys, int32_t nq,
                                 const double* xq, int32_t deriv, double* out) {
  return zp_marshal::guarded([&] {
    std::vector<::zeroplan::SamplePoint> pts;
    for (int i = 0; i < n; ++i) pts.push_back({xs[i], ys[i]});
    const auto s = ::zeroplan::fit_natural_spline(pts);
    for (int i = 0; i < nq; ++i)
      out[i] = deriv == 0 ? s.eval(xq[i])
                          : (deriv == 1 ? s.first_derivative(xq[i]) : s.second_derivative(xq[i]));
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(build_curve)(int32_t ns, const zp_sample* samples, int64_t mbs, int32_t dev,
                                 zp_curve_info* info, double* speeds_out, double* times_out) {
  return zp_marshal::guarded([&] {
    std::vector<::zeroplan::BatchSample> s;
    for (int i = 0; i < ns; ++i) s.push_back({samples[i].batch, samples[i].time});
    const auto c = ::zeroplan::build_curve(s, mbs, dev);
    info->device_id = c.device_id();
    info->mbs = c.mbs();
    info->peak_speed = c.peak_speed();
    info->peak_lo = c.peak_range().lo;
    info->peak_hi = c.peak_range().hi;
    for (int64_t b = 1; b <= mbs; ++b) {
      if (speeds_out) speeds_out[b - 1] = c.speed_at(static_cast<double>(b));
      if (times_out) times_out[b - 1] = c.predict_step_time(b);
    }
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(plan)(int64_t gbs, const zp_profile* profile, int32_t stage, const zp_model* m,
                          const zp_cluster* c, zp_allocation_plan* out) {
  return zp_marshal::guarded([&] {
    zp_marshal::from_plan(::zeroplan::plan(gbs, zp_marshal::to_profile(profile),
                                           ::zeroplan::stage_from_index(stage), zp_marshal::to_model(m),
                                           zp_marshal::to_cluster(c)),
                          out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(plan_zero01)(int64_t gbs, const zp_profile* profile, zp_allocation_plan* out) {
  return zp_marshal::guarded([&] {
    zp_marshal::from_plan(
        ::zeroplan::plan_zero01(gbs, ::zeroplan::build_curves(zp_marshal::to_profile(profile))), out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(plan_zero23)(int64_t gbs, const zp_profile* profile, const zp_comm_profile* comm,
                                 zp_allocation_plan* out) {
  return zp_marshal::guarded([&] {
    zp_marshal::from_plan(::zeroplan::plan_zero23(gbs, ::zeroplan::build_curves(zp_marshal::to_profile(profile)),
                                                  zp_marshal::to_comm(comm)),
                          out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(make_uniform_plan)(int64_t gbs, const zp_profile* profile, int32_t stage,
                                       const zp_comm_profile* comm, double tail, zp_allocation_plan* out) {
  return zp_marshal::guarded([&] {
    zp_marshal::from_plan(
        ::zeroplan::make_uniform_plan(gbs, ::zeroplan::build_curves(zp_marshal::to_profile(profile)),
                                      ::zeroplan::stage_from_index(stage), zp_marshal::to_comm(comm), tail),
        out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(allocate_remainder)(int32_t n, const int64_t* gmbs, const zp_profile* profile,
                                        int64_t remain, int64_t* out) {
  return zp_marshal::guarded([&] {
    std::vector<std::int64_t> g(gmbs, gmbs + n);
    const auto r = ::zeroplan::allocate_remainder(g, ::zeroplan::build_curves(zp_marshal::to_profile(profile)),
                                                  remain);
    for (std::size_t i = 0; i < r.size(); ++i) out[i] = r[i];
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(simulate_iteration)(const zp_cluster* c, const zp_model* m, const zp_allocation_plan* plan,
                                        int32_t stage, uint64_t iteration, zp_iteration_report* out) {
  return zp_marshal::guarded([&] {
    zp_marshal::from_report(::zeroplan::simulate_iteration(zp_marshal::to_cluster(c), zp_marshal::to_model(m),
                                                           zp_marshal::to_plan(plan),
                                                           ::zeroplan::stage_from_index(stage), iteration),
                            out);
    return ZP_OK;
  });
}

ZP_EXPORT int ZP_FN(simulate_run)(const zp_cluster* c, const zp_model* m, const zp_allocation_plan* plan,
                                  int32_t stage, int32_t iterations, zp_iteration_report* out) {
  return zp_marshal::guarded([&] {
    zp_marshal::from_report(::zeroplan::simulate_run(zp_marshal::to_cluster(c), zp_marshal::to_model(m),
                                                     zp_marshal::to_plan(plan),
                                                     ::zeroplan::stage_from_index(stage), iterations)
                                .mean,
                            out);
    return ZP_OK;
  });
}

}  // extern "C"
