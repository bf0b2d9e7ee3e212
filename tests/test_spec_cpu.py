"""Reference experiment-spec parsing (experiment.cpp:155-215 field names, required fields,
unknown-field rejection, ranges) and the B200 emulation mapping; CPU only."""
import json
import os

import pytest

from paper_2408_12596_b200 import spec
from paper_2408_12596_b200.host import InvalidInputError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _doc():
    return json.load(open(os.path.join(ROOT, "examples", "hetero2_gpt2.json")))


def test_example_spec_parses_and_maps():
    sp = spec.parse_spec(os.path.join(ROOT, "examples", "hetero2_gpt2.json"))
    assert sp["gbs"] == 512 and sp["stage"] == 2 and sp["iterations"] == 3 and sp["seed"] == 42
    assert [d["name"] for d in sp["cluster"]["devices"]] == ["fast0", "slow0"]
    # latent speed 2:1 -> 148 and 74 SMs; 180 GiB device uncapped (0), 80 GiB capped
    assert spec.emulation(sp) == [(148, 0), (74, 85899345920)]


def test_defaults_and_auto_stage():
    d = _doc()
    for k in ("stage", "iterations", "seed", "b200"):
        d.pop(k)
    sp = spec.parse_spec(d)
    assert sp["stage"] is None and sp["iterations"] == 50 and sp["seed"] == 0 and sp["format"] == "obj"
    assert sp["model"]["bytes_per_param"] == 2.0 and sp["model"]["optimizer_state_multiplier"] == 16.0


@pytest.mark.parametrize("mutate,msg", [
    (lambda d: d["cluster"]["devices"][0].pop("total_mem"), "cluster.devices[0].total_mem: missing required field"),
    (lambda d: d.__setitem__("extra", 1), "spec.extra: unknown field"),
    (lambda d: d["cluster"]["devices"][1].__setitem__("speed", 1), "cluster.devices[1].speed: unknown field"),
    (lambda d: d.__setitem__("gbs", 0), "gbs: must be >= 1"),
    (lambda d: d.__setitem__("stage", 5), 'stage: must be 0, 1, 2, 3 or "auto"'),
    (lambda d: d.__setitem__("stage", "max"), 'stage: must be 0, 1, 2, 3 or "auto"'),
    (lambda d: d.__setitem__("format", "csv"), 'format: must be "obj" or "table"'),
    (lambda d: d["cluster"].__setitem__("devices", []), "cluster.devices: must be a non-empty array"),
    (lambda d: d["model"].__setitem__("hidden_size", "768"), "model.hidden_size: must be an integer"),
    (lambda d: d["cluster"]["devices"][0].__setitem__("sm_budget", 200), "cluster.devices[0].sm_budget: must be in [1, 148]"),
])
def test_spec_errors(mutate, msg):
    d = _doc()
    mutate(d)
    with pytest.raises(InvalidInputError) as e:
        spec.parse_spec(d)
    assert msg in str(e.value)


def test_explicit_emulation_overrides():
    d = _doc()
    d["cluster"]["devices"][1]["sm_budget"] = 100
    d["cluster"]["devices"][1]["hbm_cap"] = 40 * (1 << 30)
    assert spec.emulation(spec.parse_spec(d))[1] == (100, 40 * (1 << 30))


def test_reports_use_reference_field_names():
    sp = spec.parse_spec(_doc())
    prof = {"effective_stage": 2, "devices": [
        {"device_id": 0, "mbs": 10, "probes_used": 4, "optimizer_time": 0.1, "samples": [(1, 0.5), (2, 0.9)]},
        {"device_id": 1, "mbs": 8, "probes_used": 4, "optimizer_time": 0.2, "samples": [(1, 0.9)]}]}
    pr = spec.profile_report(prof, sp)
    assert pr["devices"][1] == {"id": 1, "name": "slow0", "mbs": 8, "probes_used": 4, "optimizer_time": 0.2,
                                "samples": [[1, 0.9]]}
    plan = {"stage": 2, "gbs": 6, "gas": 2, "iteration_time": 1.0, "objective": 0.5, "predicted_wall_time": 1.2,
            "idle": [0.0, 0.1], "under_utilization": [0.0, 0.3],
            "devices": [{"device_id": 0, "b": 2, "gmbs": 4, "lbs": 2, "predicted_time": 1.0},
                        {"device_id": 1, "b": 1, "gmbs": 2, "lbs": 1, "predicted_time": 0.9}]}
    pl = spec.plan_report(plan)
    assert set(pl) == {"stage", "gbs", "gas", "predicted_T", "objective", "predicted_wall_time", "devices"}
    assert pl["devices"][1]["under_utilization"] == 0.3
    it = {"iteration_time": 2.0, "throughput": 3.0, "comm_total": 0.1, "busy": [2.0, 1.5], "idle": [0.0, 0.5],
          "compute": [1.8, 1.3]}
    sim = spec.sim_report([it, it], 1e6, baseline_T=3.0)
    assert sim["mean"]["T"] == 2.0 and sim["mean"]["flops_proxy"] == 6.0 * 1e6 * 3.0
    assert sim["speedup_vs_baseline"] == 1.5 and sim["iterations"] == 2
