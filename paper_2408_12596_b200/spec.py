"""Experiment spec and report formats of the reference, on the B200 emulated cluster.

The reference reads a JSON spec (proj/core/src/experiment.cpp:155-215: `cluster.devices[]`
with `name, total_mem, act_mem_per_batch, compute_fixed, compute_per_batch, optimizer_time`,
`cluster.link_bandwidths, link_latency, jitter`, `model.param_count, hidden_size, num_layers,
bytes_per_param, optimizer_state_multiplier`, `gbs, stage, iterations, seed, format`) and
writes reports with fixed field names (experiment.cpp:264-338). This module parses the same
spec with the same validation messages, maps each latent device onto an emulated B200 rank, and
renders the reference's report objects from measured runs.

B200 extension (optional, ignored by the reference's fields): per device `sm_budget` (CTA cap
= SMs) and `hbm_cap` (bytes; the arena size), and a top-level `b200` object naming the
transformer to run (`{"model": "gpt2-small"}`). Without them the SM budget follows the latent
speed (148 SMs for the device with the smallest compute_per_batch, proportionally fewer for
slower ones) and the HBM cap is `total_mem` (0 = the whole device when total_mem exceeds it).
"""
from __future__ import annotations

import json
from typing import Optional, Sequence

from .host import InvalidInputError

_DEVICE_KEYS = {"name", "total_mem", "act_mem_per_batch", "compute_fixed", "compute_per_batch",
                "optimizer_time", "sm_budget", "hbm_cap"}
_CLUSTER_KEYS = {"devices", "link_bandwidths", "link_latency", "jitter"}
_MODEL_KEYS = {"param_count", "hidden_size", "num_layers", "bytes_per_param", "optimizer_state_multiplier"}
_SPEC_KEYS = {"cluster", "model", "gbs", "stage", "iterations", "seed", "format", "b200"}
B200_SMS = 148
B200_HBM = 180 * (1 << 30)


class SpecError(InvalidInputError):
    """The reference's InvalidInputError for a malformed spec (status ZP_EINVAL)."""


def _fail(path: str, why: str):
    raise SpecError(f"{path}: {why}")


def _obj(v, path):
    if not isinstance(v, dict):
        _fail(path, "must be an object")
    return v


def _req(obj, path, key):
    if key not in obj:
        _fail(f"{path}.{key}", "missing required field")
    return obj[key]


def _num(v, path):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        _fail(path, "must be a number")
    return float(v)


def _int(v, path):
    if isinstance(v, bool) or not isinstance(v, int) and not (isinstance(v, float) and v.is_integer()):
        _fail(path, "must be an integer")
    return int(v)


def _unknown(obj, path, allowed):
    for k in obj:
        if k not in allowed:
            _fail(f"{path}.{k}", "unknown field")


def parse_spec(doc) -> dict:
    """Spec dict (from a JSON string, a path or a dict) validated like the reference's
    parse_spec; returns plain Python values."""
    if isinstance(doc, str):
        text = doc
        if not text.lstrip().startswith("{"):
            with open(doc) as f:
                text = f.read()
        try:
            doc = json.loads(text)
        except json.JSONDecodeError as e:
            raise SpecError(f"spec: {e}") from None
    _obj(doc, "spec")
    _unknown(doc, "spec", _SPEC_KEYS)
    cl = _obj(_req(doc, "spec", "cluster"), "cluster")
    _unknown(cl, "cluster", _CLUSTER_KEYS)
    devs = _req(cl, "cluster", "devices")
    if not isinstance(devs, list) or not devs:
        _fail("cluster.devices", "must be a non-empty array")
    devices = []
    for i, d in enumerate(devs):
        p = f"cluster.devices[{i}]"
        _obj(d, p)
        _unknown(d, p, _DEVICE_KEYS)
        name = d.get("name", f"gpu{i}")
        if not isinstance(name, str):
            _fail(p + ".name", "must be a string")
        dev = {"name": name}
        for k in ("total_mem", "act_mem_per_batch", "compute_fixed", "compute_per_batch"):
            dev[k] = _num(_req(d, p, k), f"{p}.{k}")
        dev["optimizer_time"] = _num(d.get("optimizer_time", 0.0), p + ".optimizer_time")
        if "sm_budget" in d:
            dev["sm_budget"] = _int(d["sm_budget"], p + ".sm_budget")
            if not 1 <= dev["sm_budget"] <= B200_SMS:
                _fail(p + ".sm_budget", f"must be in [1, {B200_SMS}]")
        if "hbm_cap" in d:
            dev["hbm_cap"] = _num(d["hbm_cap"], p + ".hbm_cap")
        if dev["total_mem"] <= 0 or dev["compute_per_batch"] <= 0:
            _fail(p, "total_mem and compute_per_batch must be positive")
        devices.append(dev)
    bws = _req(cl, "cluster", "link_bandwidths")
    if not isinstance(bws, list):
        _fail("cluster.link_bandwidths", "must be an array")
    bws = [_num(b, f"cluster.link_bandwidths[{i}]") for i, b in enumerate(bws)]
    if len(bws) != len(devices):
        _fail("cluster.link_bandwidths", "must have one entry per device")
    model = _obj(_req(doc, "spec", "model"), "model")
    _unknown(model, "model", _MODEL_KEYS)
    m = {"param_count": _num(_req(model, "model", "param_count"), "model.param_count"),
         "hidden_size": _int(_req(model, "model", "hidden_size"), "model.hidden_size"),
         "num_layers": _int(_req(model, "model", "num_layers"), "model.num_layers"),
         "bytes_per_param": _num(model.get("bytes_per_param", 2.0), "model.bytes_per_param"),
         "optimizer_state_multiplier": _num(model.get("optimizer_state_multiplier", 16.0),
                                            "model.optimizer_state_multiplier")}
    gbs = _int(_req(doc, "spec", "gbs"), "spec.gbs")
    if gbs < 1:
        _fail("gbs", "must be >= 1")
    stage = doc.get("stage", "auto")
    if isinstance(stage, str):
        if stage != "auto":
            _fail("stage", 'must be 0, 1, 2, 3 or "auto"')
        stage = None
    else:
        stage = _int(stage, "stage")
        if stage not in (0, 1, 2, 3):
            _fail("stage", 'must be 0, 1, 2, 3 or "auto"')
    iterations = _int(doc.get("iterations", 50), "spec.iterations")
    if iterations < 1:
        _fail("iterations", "must be >= 1")
    seed = _int(doc.get("seed", 0), "spec.seed")
    if seed < 0:
        _fail("seed", "must be >= 0")
    fmt = doc.get("format", "obj")
    if fmt not in ("obj", "table"):
        _fail("format", 'must be "obj" or "table"')
    b200 = _obj(doc.get("b200", {}), "b200")
    return {"cluster": {"devices": devices, "link_bandwidths": bws,
                        "link_latency": _num(cl.get("link_latency", 0.0), "cluster.link_latency"),
                        "jitter": _num(cl.get("jitter", 0.0), "cluster.jitter")},
            "model": m, "gbs": gbs, "stage": stage, "iterations": iterations, "seed": seed,
            "format": fmt, "b200": dict(b200)}


def emulation(spec: dict) -> list:
    """Per device (sm_budget, hbm_cap_bytes) of the emulated B200 cluster (see module doc)."""
    devs = spec["cluster"]["devices"]
    fastest = min(d["compute_per_batch"] for d in devs)
    out = []
    for d in devs:
        sm = d.get("sm_budget")
        if sm is None:
            sm = max(2, int(round(B200_SMS * fastest / d["compute_per_batch"] / 2)) * 2)
        cap = d.get("hbm_cap", d["total_mem"])
        out.append((int(sm), 0 if cap >= B200_HBM else int(cap)))
    return out


# ---------------------------------------------------------------- reports (experiment.cpp:264-338)

def profile_report(profile: dict, spec: dict) -> dict:
    names = [d["name"] for d in spec["cluster"]["devices"]]
    return {"effective_stage": profile["effective_stage"],
            "devices": [{"id": d["device_id"], "name": names[d["device_id"]], "mbs": d["mbs"],
                         "probes_used": d["probes_used"], "optimizer_time": d["optimizer_time"],
                         "samples": [[b, t] for b, t in d["samples"]]} for d in profile["devices"]]}


def plan_report(plan: dict) -> dict:
    return {"stage": plan["stage"], "gbs": plan["gbs"], "gas": plan["gas"],
            "predicted_T": plan["iteration_time"], "objective": plan["objective"],
            "predicted_wall_time": plan["predicted_wall_time"],
            "devices": [{"id": d["device_id"], "b": d["b"], "gmbs": d["gmbs"], "lbs": d["lbs"],
                         "predicted_time": d["predicted_time"], "idle": plan["idle"][i],
                         "under_utilization": plan["under_utilization"][i]}
                        for i, d in enumerate(plan["devices"])]}


def sim_report(iterations: Sequence[dict], param_count: float, baseline_T: Optional[float] = None) -> dict:
    """The reference's `simulate` object from MEASURED iteration reports
    (poplar.iteration_report per iteration): mean T, throughput, flops proxy (6 * params *
    samples/s, as the reference), comm, busy/idle/compute per rank, and the speedup over a
    baseline iteration time when given."""
    n = len(iterations)
    k = len(iterations[0]["busy"])
    mean = lambda key: sum(r[key] for r in iterations) / n  # noqa: E731
    vec = lambda key: [sum(r[key][i] for r in iterations) / n for i in range(k)]  # noqa: E731
    thr = mean("throughput")
    out = {"iterations": n,
           "mean": {"T": mean("iteration_time"), "throughput": thr, "flops_proxy": 6.0 * param_count * thr,
                    "comm_total": mean("comm_total"), "busy": vec("busy"), "idle": vec("idle"),
                    "compute": vec("compute")}}
    out["speedup_vs_baseline"] = (baseline_T / out["mean"]["T"]) if baseline_T else None
    return out
