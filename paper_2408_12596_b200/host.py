"""Python view of the zeroplan host C ABI (include/zp_host.h).

`HostAPI(lib, prefix)` binds one library's functions — the product (`libzp.so`,
prefix ``zp_``) or the oracle build of the reference sources (``zpref_``) — and
exposes them with the reference's names (profile_cluster, plan, simulate_iteration, ...),
raising the reference's exception taxonomy on error codes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

MAX_DEV = 64
MAX_SAMPLES = 128

OK, EINVAL, EINFEASIBLE, EINTERNAL, OOM, ECUDA, ENCCL = range(7)


class ZeroplanError(RuntimeError):
    pass


class InvalidInputError(ZeroplanError):
    pass


class InfeasibleError(ZeroplanError):
    pass


class InternalError(ZeroplanError):
    pass


class CudaError(ZeroplanError):
    pass


class NcclError(ZeroplanError):
    pass


_ERR = {EINVAL: InvalidInputError, EINFEASIBLE: InfeasibleError, EINTERNAL: InternalError,
        ECUDA: CudaError, ENCCL: NcclError}


class DeviceGT(C.Structure):
    _fields_ = [("total_mem", C.c_double), ("act_mem_per_batch", C.c_double),
                ("compute_fixed", C.c_double), ("compute_per_batch", C.c_double),
                ("optimizer_time", C.c_double)]


class Cluster(C.Structure):
    _fields_ = [("n", C.c_int32), ("devices", DeviceGT * MAX_DEV),
                ("link_bandwidths", C.c_double * MAX_DEV), ("link_latency", C.c_double),
                ("seed", C.c_uint64), ("jitter", C.c_double)]


class Model(C.Structure):
    _fields_ = [("param_count", C.c_double), ("hidden_size", C.c_int64), ("num_layers", C.c_int64),
                ("bytes_per_param", C.c_double), ("optimizer_state_multiplier", C.c_double)]


class StepTrace(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("forward_compute", "backward_compute", "fwd_allgather",
                                          "bwd_allgather", "reduce_scatter", "allreduce",
                                          "optimizer_step")]


class Probe(C.Structure):
    _fields_ = [("before_forward", C.c_double), ("after_forward", C.c_double), ("total", C.c_double)]


class CommProfile(C.Structure):
    _fields_ = [("stage", C.c_int32), ("volume_forward", C.c_double), ("volume_backward", C.c_double),
                ("volume_optimizer", C.c_double), ("time_per_step", C.c_double),
                ("sync_time", C.c_double)]


class Sample(C.Structure):
    _fields_ = [("batch", C.c_int64), ("time", C.c_double)]


class DeviceProfile(C.Structure):
    _fields_ = [("device_id", C.c_int32), ("mbs", C.c_int64), ("probes_used", C.c_int32),
                ("optimizer_time", C.c_double), ("n_samples", C.c_int32),
                ("samples", Sample * MAX_SAMPLES)]


class Profile(C.Structure):
    _fields_ = [("effective_stage", C.c_int32), ("n", C.c_int32), ("devices", DeviceProfile * MAX_DEV)]


class CurveInfo(C.Structure):
    _fields_ = [("device_id", C.c_int32), ("mbs", C.c_int64), ("peak_speed", C.c_double),
                ("peak_lo", C.c_int64), ("peak_hi", C.c_int64)]


class DeviceAlloc(C.Structure):
    _fields_ = [("device_id", C.c_int32), ("b", C.c_int64), ("gmbs", C.c_int64), ("lbs", C.c_int64),
                ("predicted_time", C.c_double)]


class Plan(C.Structure):
    _fields_ = [("stage", C.c_int32), ("gbs", C.c_int64), ("gas", C.c_int64), ("n", C.c_int32),
                ("devices", DeviceAlloc * MAX_DEV), ("iteration_time", C.c_double),
                ("idle", C.c_double * MAX_DEV), ("under_utilization", C.c_double * MAX_DEV),
                ("objective", C.c_double), ("weights", C.c_double * MAX_DEV),
                ("predicted_wall_time", C.c_double)]


class IterationReport(C.Structure):
    _fields_ = [("iteration_time", C.c_double), ("n", C.c_int32), ("busy", C.c_double * MAX_DEV),
                ("idle", C.c_double * MAX_DEV), ("compute", C.c_double * MAX_DEV),
                ("comm_total", C.c_double), ("throughput", C.c_double)]


# ----------------------------------------------------------------- python-side value types

@dataclass
class Device:
    total_mem: float
    act_mem_per_batch: float
    compute_fixed: float
    compute_per_batch: float
    optimizer_time: float = 0.0
    name: str = ""


@dataclass
class ClusterSpec:
    devices: list
    link_bandwidths: list
    link_latency: float = 0.0
    seed: int = 0
    jitter: float = 0.0

    def to_c(self) -> Cluster:
        c = Cluster()
        c.n = len(self.devices)
        for i, d in enumerate(self.devices):
            c.devices[i].total_mem = d.total_mem
            c.devices[i].act_mem_per_batch = d.act_mem_per_batch
            c.devices[i].compute_fixed = d.compute_fixed
            c.devices[i].compute_per_batch = d.compute_per_batch
            c.devices[i].optimizer_time = d.optimizer_time
            c.link_bandwidths[i] = self.link_bandwidths[i]
        c.link_latency = self.link_latency
        c.seed = self.seed
        c.jitter = self.jitter
        return c


@dataclass
class ModelSpec:
    param_count: float
    hidden_size: int = 1024
    num_layers: int = 8
    bytes_per_param: float = 2.0
    optimizer_state_multiplier: float = 16.0

    def to_c(self) -> Model:
        return Model(self.param_count, self.hidden_size, self.num_layers, self.bytes_per_param,
                     self.optimizer_state_multiplier)


def profile_to_py(p: Profile) -> dict:
    devs = []
    for i in range(p.n):
        d = p.devices[i]
        devs.append({"device_id": d.device_id, "mbs": d.mbs, "probes_used": d.probes_used,
                     "optimizer_time": d.optimizer_time,
                     "samples": [(d.samples[k].batch, d.samples[k].time) for k in range(d.n_samples)]})
    return {"effective_stage": p.effective_stage, "devices": devs}


def profile_from_py(d: dict) -> Profile:
    p = Profile()
    p.effective_stage = d["effective_stage"]
    p.n = len(d["devices"])
    for i, dev in enumerate(d["devices"]):
        t = p.devices[i]
        t.device_id = dev["device_id"]
        t.mbs = dev["mbs"]
        t.probes_used = dev.get("probes_used", 0)
        t.optimizer_time = dev.get("optimizer_time", 0.0)
        t.n_samples = len(dev["samples"])
        for k, (b, tm) in enumerate(dev["samples"]):
            t.samples[k].batch = b
            t.samples[k].time = tm
    return p


def plan_to_py(p: Plan) -> dict:
    n = p.n
    return {"stage": p.stage, "gbs": p.gbs, "gas": p.gas,
            "devices": [{"device_id": p.devices[i].device_id, "b": p.devices[i].b,
                         "gmbs": p.devices[i].gmbs, "lbs": p.devices[i].lbs,
                         "predicted_time": p.devices[i].predicted_time} for i in range(n)],
            "iteration_time": p.iteration_time, "idle": list(p.idle[:n]),
            "under_utilization": list(p.under_utilization[:n]), "objective": p.objective,
            "weights": list(p.weights[:n]), "predicted_wall_time": p.predicted_wall_time}


def plan_from_py(d: dict) -> Plan:
    p = Plan()
    p.stage, p.gbs, p.gas, p.n = d["stage"], d["gbs"], d["gas"], len(d["devices"])
    for i, dev in enumerate(d["devices"]):
        p.devices[i] = DeviceAlloc(dev["device_id"], dev["b"], dev["gmbs"], dev["lbs"], dev["predicted_time"])
        p.idle[i] = d["idle"][i]
        p.under_utilization[i] = d["under_utilization"][i]
        p.weights[i] = d["weights"][i]
    p.iteration_time = d["iteration_time"]
    p.objective = d["objective"]
    p.predicted_wall_time = d["predicted_wall_time"]
    return p


def report_to_py(r: IterationReport) -> dict:
    n = r.n
    return {"iteration_time": r.iteration_time, "busy": list(r.busy[:n]), "idle": list(r.idle[:n]),
            "compute": list(r.compute[:n]), "comm_total": r.comm_total, "throughput": r.throughput}


_SIGS = {
    "last_error": ([], C.c_char_p),
    "resident_state_bytes": ([C.POINTER(Model), C.c_int32, C.c_int32, C.POINTER(C.c_double)], C.c_int),
    "run_step": ([C.POINTER(Cluster), C.c_int32, C.POINTER(Model), C.c_int64, C.c_int32, C.c_uint64,
                  C.POINTER(StepTrace)], C.c_int),
    "memory_probe": ([C.POINTER(Cluster), C.c_int32, C.POINTER(Model), C.c_int32, C.POINTER(Probe)], C.c_int),
    "collective_time": ([C.c_double, C.POINTER(Cluster), C.POINTER(C.c_double)], C.c_int),
    "make_comm_profile": ([C.POINTER(Model), C.c_int32, C.POINTER(Cluster), C.POINTER(CommProfile)], C.c_int),
    "ffn_volumes": ([C.c_int64, C.c_int64, C.POINTER(C.c_uint64)], C.c_int),
    "time_consumed_during_step": ([C.POINTER(StepTrace), C.c_int32, C.POINTER(C.c_double)], C.c_int),
    "estimate_theoretical_mbs": ([C.POINTER(Cluster), C.c_int32, C.POINTER(Model), C.c_int32,
                                  C.POINTER(C.c_int64)], C.c_int),
    "search_mbs": ([C.POINTER(Cluster), C.c_int32, C.POINTER(Model), C.c_int32, C.c_int64,
                    C.POINTER(DeviceProfile)], C.c_int),
    "profile_cluster": ([C.POINTER(Cluster), C.POINTER(Model), C.c_int32, C.POINTER(Profile)], C.c_int),
    "spline_fit": ([C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                    C.POINTER(C.c_double)], C.c_int),
    "spline_eval": ([C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32,
                     C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double)], C.c_int),
    "build_curve": ([C.c_int32, C.POINTER(Sample), C.c_int64, C.c_int32, C.POINTER(CurveInfo),
                     C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "plan": ([C.c_int64, C.POINTER(Profile), C.c_int32, C.POINTER(Model), C.POINTER(Cluster),
              C.POINTER(Plan)], C.c_int),
    "plan_zero01": ([C.c_int64, C.POINTER(Profile), C.POINTER(Plan)], C.c_int),
    "plan_zero23": ([C.c_int64, C.POINTER(Profile), C.POINTER(CommProfile), C.POINTER(Plan)], C.c_int),
    "make_uniform_plan": ([C.c_int64, C.POINTER(Profile), C.c_int32, C.POINTER(CommProfile), C.c_double,
                           C.POINTER(Plan)], C.c_int),
    "allocate_remainder": ([C.c_int32, C.POINTER(C.c_int64), C.POINTER(Profile), C.c_int64,
                            C.POINTER(C.c_int64)], C.c_int),
    "simulate_iteration": ([C.POINTER(Cluster), C.POINTER(Model), C.POINTER(Plan), C.c_int32, C.c_uint64,
                            C.POINTER(IterationReport)], C.c_int),
    "simulate_run": ([C.POINTER(Cluster), C.POINTER(Model), C.POINTER(Plan), C.c_int32, C.c_int32,
                      C.POINTER(IterationReport)], C.c_int),
}


def _darr(xs):
    return (C.c_double * max(1, len(xs)))(*xs)


class HostAPI:
    """Reference-named wrappers over one library's zp_host.h exports."""

    def __init__(self, lib: C.CDLL, prefix: str):
        self.lib = lib
        self.prefix = prefix
        self.fn = {}
        for name, (args, res) in _SIGS.items():
            f = getattr(lib, prefix + name)
            f.argtypes = args
            f.restype = res
            self.fn[name] = f

    def _check(self, rc, allow_oom=False):
        if rc == OK:
            return True
        if rc == OOM and allow_oom:
            return False
        msg = self.fn["last_error"]().decode()
        raise _ERR.get(rc, ZeroplanError)(msg)

    # ---- latent back end / cost model
    def resident_state_bytes(self, model: ModelSpec, stage: int, n: int) -> float:
        out = C.c_double()
        self._check(self.fn["resident_state_bytes"](C.byref(model.to_c()), stage, n, C.byref(out)))
        return out.value

    def run_step(self, cluster, dev, model, batch, stage, noise_index=0) -> Optional[dict]:
        t = StepTrace()
        ok = self._check(self.fn["run_step"](C.byref(cluster.to_c()), dev, C.byref(model.to_c()), batch,
                                             stage, noise_index, C.byref(t)), allow_oom=True)
        return {k: getattr(t, k) for k, _ in StepTrace._fields_} if ok else None

    def memory_probe(self, cluster, dev, model, stage) -> Optional[tuple]:
        p = Probe()
        ok = self._check(self.fn["memory_probe"](C.byref(cluster.to_c()), dev, C.byref(model.to_c()), stage,
                                                 C.byref(p)), allow_oom=True)
        return (p.before_forward, p.after_forward, p.total) if ok else None

    def collective_time(self, volume, cluster) -> float:
        out = C.c_double()
        self._check(self.fn["collective_time"](volume, C.byref(cluster.to_c()), C.byref(out)))
        return out.value

    def make_comm_profile(self, model, stage, cluster) -> CommProfile:
        out = CommProfile()
        self._check(self.fn["make_comm_profile"](C.byref(model.to_c()), stage, C.byref(cluster.to_c()),
                                                 C.byref(out)))
        return out

    def ffn_volumes(self, hidden, layers):
        out = (C.c_uint64 * 3)()
        self._check(self.fn["ffn_volumes"](hidden, layers, out))
        return tuple(out)

    # ---- profiler
    def time_consumed_during_step(self, trace: dict, stage: int) -> float:
        t = StepTrace(**trace)
        out = C.c_double()
        self._check(self.fn["time_consumed_during_step"](C.byref(t), stage, C.byref(out)))
        return out.value

    def estimate_theoretical_mbs(self, cluster, dev, model, stage) -> Optional[int]:
        out = C.c_int64()
        ok = self._check(self.fn["estimate_theoretical_mbs"](C.byref(cluster.to_c()), dev, C.byref(model.to_c()),
                                                             stage, C.byref(out)), allow_oom=True)
        return out.value if ok else None

    def search_mbs(self, cluster, dev, model, stage, estimate) -> dict:
        d = DeviceProfile()
        self._check(self.fn["search_mbs"](C.byref(cluster.to_c()), dev, C.byref(model.to_c()), stage, estimate,
                                          C.byref(d)))
        return {"mbs": d.mbs, "probes_used": d.probes_used, "optimizer_time": d.optimizer_time,
                "samples": [(d.samples[k].batch, d.samples[k].time) for k in range(d.n_samples)]}

    def profile_cluster(self, cluster, model, stage_request: Optional[int]) -> dict:
        p = Profile()
        self._check(self.fn["profile_cluster"](C.byref(cluster.to_c()), C.byref(model.to_c()),
                                               -1 if stage_request is None else stage_request, C.byref(p)))
        return profile_to_py(p)

    # ---- spline / curves
    def spline_fit(self, xs, ys):
        n = len(xs)
        knots = (C.c_double * n)()
        segs = (C.c_double * (4 * max(1, n - 1)))()
        self._check(self.fn["spline_fit"](n, _darr(xs), _darr(ys), knots, segs))
        return list(knots), [tuple(segs[4 * i:4 * i + 4]) for i in range(n - 1)]

    def spline_eval(self, xs, ys, xq, deriv=0):
        out = (C.c_double * max(1, len(xq)))()
        self._check(self.fn["spline_eval"](len(xs), _darr(xs), _darr(ys), len(xq), _darr(xq), deriv, out))
        return list(out[:len(xq)])

    def build_curve(self, samples, mbs, device_id=0):
        arr = (Sample * max(1, len(samples)))(*[Sample(b, t) for b, t in samples])
        info = CurveInfo()
        sp = (C.c_double * max(1, mbs))()
        tm = (C.c_double * max(1, mbs))()
        self._check(self.fn["build_curve"](len(samples), arr, mbs, device_id, C.byref(info), sp, tm))
        return {"device_id": info.device_id, "mbs": info.mbs, "peak_speed": info.peak_speed,
                "peak_range": (info.peak_lo, info.peak_hi), "speeds": list(sp[:mbs]), "times": list(tm[:mbs])}

    # ---- planner
    def plan(self, gbs, profile: dict, stage, model, cluster) -> dict:
        out = Plan()
        self._check(self.fn["plan"](gbs, C.byref(profile_from_py(profile)), stage, C.byref(model.to_c()),
                                    C.byref(cluster.to_c()), C.byref(out)))
        return plan_to_py(out)

    def plan_zero01(self, gbs, profile: dict) -> dict:
        out = Plan()
        self._check(self.fn["plan_zero01"](gbs, C.byref(profile_from_py(profile)), C.byref(out)))
        return plan_to_py(out)

    def plan_zero23(self, gbs, profile: dict, comm: CommProfile) -> dict:
        out = Plan()
        self._check(self.fn["plan_zero23"](gbs, C.byref(profile_from_py(profile)), C.byref(comm), C.byref(out)))
        return plan_to_py(out)

    def make_uniform_plan(self, gbs, profile: dict, stage, comm: CommProfile, optimizer_tail) -> dict:
        out = Plan()
        self._check(self.fn["make_uniform_plan"](gbs, C.byref(profile_from_py(profile)), stage, C.byref(comm),
                                                 optimizer_tail, C.byref(out)))
        return plan_to_py(out)

    def allocate_remainder(self, gmbs: Sequence[int], profile: dict, remain: int):
        n = len(gmbs)
        out = (C.c_int64 * max(1, n))()
        self._check(self.fn["allocate_remainder"](n, (C.c_int64 * max(1, n))(*gmbs),
                                                  C.byref(profile_from_py(profile)), remain, out))
        return list(out[:n])

    # ---- executor
    def simulate_iteration(self, cluster, model, plan: dict, stage, iteration=0) -> dict:
        out = IterationReport()
        self._check(self.fn["simulate_iteration"](C.byref(cluster.to_c()), C.byref(model.to_c()),
                                                  C.byref(plan_from_py(plan)), stage, iteration, C.byref(out)))
        return report_to_py(out)

    def simulate_run(self, cluster, model, plan: dict, stage, iterations) -> dict:
        out = IterationReport()
        self._check(self.fn["simulate_run"](C.byref(cluster.to_c()), C.byref(model.to_c()),
                                            C.byref(plan_from_py(plan)), stage, iterations, C.byref(out)))
        return report_to_py(out)


_product = None


def product() -> HostAPI:
    """The product library (libzp.so)."""
    global _product
    if _product is None:
        import os
        alt = os.environ.get("ZP_HOST_LIB")  # sanitizer build of the host code (tools/sanitize)
        if alt:
            _product = HostAPI(C.CDLL(alt), "zp_")
        else:
            from . import _lib
            _product = HostAPI(_lib.lib, "zp_")
    return _product
