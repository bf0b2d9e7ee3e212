"""Poplar on B200: the reference pipeline (profile -> curves -> plan -> execute) with the latent
device model replaced by the real runtime.

    profile = rt.profile(stage)                      # Alg. 1, lockstep over ranks (C++)
    plan    = poplar_plan(rt, profile, gbs, stage)   # Alg. 2, bit-exact zeroplan planner (C++)
    timing  = rt.execute_iteration(plan, stage)      # real ZeRO iteration on this rank

Reference call stack: proj/core/src/experiment.cpp:424-436 (run_through_plan) and
simulator.cpp:49-116 (simulate_iteration) — same data structures, real devices.
"""
from __future__ import annotations

from typing import Optional, Sequence

from . import host
from .host import ClusterSpec, Device, ModelSpec

# Fallback link model when none was measured (one rank, or a caller that skips the measurement):
# NVLink 5 per-direction peer-copy bandwidth on this pool and a typical collective launch latency.
# bench.py measures both per run (Runtime.link_model: the stage's reduce-scatter path timed at two
# sizes, max over ranks) and passes them in; they parameterise the planner's alpha-beta collective
# model (reference comm.cpp:88-99), which on NVSwitch is uniform across ranks.
NVLINK_BPS = 770e9
NCCL_ALPHA = 25e-6


def planner_inputs(rt, n: int, link_bw: float = NVLINK_BPS, alpha: float = NCCL_ALPHA):
    """ModelSpec / ClusterSpec for `zeroplan::plan`: only the device count and the link model are
    read by the planner (reference planner.cpp:343-347); the latent device fields are unused."""
    m = rt.model
    model = ModelSpec(float(rt.param_count), m.d_model, m.n_layer, 2.0, 16.0)
    cluster = ClusterSpec([Device(1.0, 1.0, 0.0, 1.0)] * n, [link_bw] * n, alpha)
    return model, cluster


def poplar_plan(rt, profile: dict, gbs: int, stage: int, n: int, uniform: bool = False,
                link=None, api=None) -> dict:
    """Alg. 2 through the product planner (or `api`, e.g. the compiled reference for parity).
    link = (bandwidth B/s, latency s) of the measured alpha-beta model."""
    api = api or host.product()
    model, cluster = planner_inputs(rt, n, *(link or ()))
    if not uniform:
        return api.plan(gbs, profile, stage, model, cluster)
    comm = api.make_comm_profile(model, stage, cluster)
    tail = max(d["optimizer_time"] for d in profile["devices"])
    return api.make_uniform_plan(gbs, profile, stage, comm, tail)


def recalibrate(profile: dict, plan: dict, timings: Sequence[dict], slow_only: bool = True) -> dict:
    """Profile with every rank's step-time samples rescaled by the ratio of its measured compute
    in a planned iteration to the compute the plan predicted for it.

    Alg. 1's probes are short; a long iteration settles at lower power-capped clocks, and not by
    the same factor on every tier (a rank with more SMs draws more power). One measured iteration
    corrects the curves; the planner (Alg. 2) is then re-run unchanged on the corrected profile.
    Ranks that did no work keep their samples.

    slow_only: a rank is only ever slowed, never sped up. Under the board power cap a GPU that
    idles part of the iteration (waiting in lockstep collectives) computes at higher clocks than
    one that never idles, so its faster measurement is an artefact of the plan: crediting it made
    the next plan give that rank the bigger batch, it became the bottleneck and slowed down, and
    the passes oscillated between two plans (C5 on 4 GPUs: ±10 % per rank). The full-load speed is
    what the bottleneck rank runs at, and that is what slowing-only converges to."""
    out = {**profile, "devices": []}
    for d, dp, t in zip(profile["devices"], plan["devices"], timings):
        # predicted_time = sum of the curve's step times over the rank's micro-steps
        # (reference planner.cpp:40-58, 318-326): compute only, like the measured spans
        predicted, measured = dp["predicted_time"], t["compute"]
        ratio = measured / predicted if predicted > 0 and measured > 0 else 1.0
        if slow_only:
            ratio = max(ratio, 1.0)
        out["devices"].append({**d, "samples": [(b, tt * ratio) for b, tt in d["samples"]]})
    return out


def recalibrate_link(link, stage: int, gas: int, comm_floor: float, param_count: float,
                     bytes_per_param: float = 2.0):
    """Link model (bandwidth, latency) fitted to the collective time an executed iteration actually
    exposed. The reference's cost model charges every collective in full, additively
    (comm.cpp:101-120): per iteration `gas` micro-step launches (ZeRO-2: one reduce-scatter; ZeRO-3:
    two gathers + one reduce-scatter) plus the synchronisation collective (ZeRO-0/1: an all-reduce
    of twice the model; ZeRO-2: a gather). On B200 the ZeRO-3 gathers are prefetched behind
    compute, so the additive model over-charges them. Keeping the measured latency, the bandwidth
    is solved from the measured comm floor (poplar.iteration_report) so that the planner's comm
    term equals what the iteration exposed; the unchanged planner then re-plans with it."""
    bw, alpha = link
    vol = param_count * bytes_per_param
    if stage <= 1:
        launches, volume = 1, 2.0 * vol
    elif stage == 2:
        launches, volume = gas + 1, (gas + 1) * vol
    else:
        launches, volume = 3 * gas, 3 * gas * vol
    t = comm_floor - launches * alpha
    return (volume / t if t > 0 else 1e15, alpha)


def rank_slice(plan: dict, rank: int):
    """First global sample index and sample count of `rank` (ranks take contiguous ranges in
    device order, so global sample j is the same sample for every allocation)."""
    first = sum(d["gmbs"] for d in plan["devices"][:rank])
    return first, plan["devices"][rank]["gmbs"]


def iteration_report(timings: Sequence[dict], gbs: int) -> dict:
    """Combine per-rank measured timings into the reference's IterationReport
    (simulator.cpp:104-114). Collective k costs every rank min_j t_j(k) (the last rank to
    arrive does not wait); anything above that on a faster rank is synchronisation idle.
    busy_i = compute_i + sum_k min_j t_j(k) + optimizer_i; T = max_i wall_i; idle_i = T - busy_i."""
    counts = {len(t["coll_times"]) for t in timings}
    if len(counts) != 1:
        raise ValueError(f"ranks issued different collective counts {sorted(counts)}")
    ncoll = counts.pop()
    floor = sum(min(t["coll_times"][k] for t in timings) for k in range(ncoll))
    T = max(t["wall"] for t in timings)
    busy = [t["compute"] + floor + t["optimizer"] for t in timings]
    return {"iteration_time": T, "busy": busy, "idle": [T - b for b in busy],
            "compute": [t["compute"] for t in timings], "comm_total": floor, "throughput": gbs / T,
            "sync_idle_pct": [100.0 * max(0.0, T - b) / T for b in busy]}
