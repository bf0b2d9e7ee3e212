"""The device-seam binding (integration/hardware_b200.cpp) linked with the reference's own zeroplan
sources (oracle/_ref/seam_b200, built by oracle/Makefile).

CPU: with no B200 backend active the seam forwards to the reference's latent model (its unchanged
hardware.cpp with the pair renamed), so profile -> plan -> simulate through the binary equals the
reference library bit for bit.
GPU: the reference's unchanged profile_cluster / plan / simulate_iteration drive real B200 ranks
through the reference's run_step / memory_probe signatures; the product planner re-plans every
measured profile bit-identically; OOM crosses the seam as std::nullopt; the executed iteration
(Backend::execute_iteration) returns the reference's IterationReport.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEAM = os.path.join(ROOT, "oracle", "_ref", "seam_b200")


def _seam():
    if not os.path.exists(SEAM):
        import oracle
        oracle.build_reference()
    if not os.path.exists(SEAM):
        pytest.skip("oracle/_ref/seam_b200 not built and /root/reference absent")
    return SEAM


def _run(args, timeout=900):
    r = subprocess.run([_seam()] + args, capture_output=True, text=True, timeout=timeout)
    out = r.stdout.strip()
    # NCCL may print its version banner to stdout first; the report starts at the first '{' / '['
    starts = [i for i in (out.find("\n{"), out.find("\n[")) if i >= 0]
    if out[:1] not in "{[" and starts:
        out = out[min(starts) + 1:]
    try:
        data = json.loads(out.replace('"inf"', "Infinity"))
    except json.JSONDecodeError:
        raise AssertionError(f"rc={r.returncode} stdout={out[:2000]} stderr={r.stderr[-2000:]}")
    return r.returncode, data


def test_latent_seam_matches_reference_library():
    import oracle
    from paper_2408_12596_b200.host import ClusterSpec, Device, ModelSpec
    rc, data = _run(["--latent"])
    assert rc == 0, data
    ref = oracle.reference()
    c1 = [0.002, 0.002, 0.004, 0.004]
    cl = ClusterSpec([Device(80e9, 2e9, 0.01, c, 0.005) for c in c1], [100e9] * 4, 1e-4)
    m = ModelSpec(1e9, 2048, 24)
    for st, got in enumerate(data):
        p = ref.profile_cluster(cl, m, st)
        a = ref.plan(256, p, p["effective_stage"], m, cl)
        r = ref.simulate_iteration(cl, m, a, p["effective_stage"])
        assert got["profile"]["effective_stage"] == p["effective_stage"]
        for gd, rd in zip(got["profile"]["devices"], p["devices"]):
            assert gd["mbs"] == rd["mbs"] and gd["probes_used"] == rd["probes_used"]
            assert [tuple(s) for s in gd["samples"]] == [tuple(s) for s in rd["samples"]]
        assert got["plan"]["gas"] == a["gas"]
        assert got["plan"]["b"] == [d["b"] for d in a["devices"]]
        assert got["plan"]["gmbs"] == [d["gmbs"] for d in a["devices"]]
        assert got["plan"]["lbs"] == [d["lbs"] for d in a["devices"]]
        assert got["plan"]["predicted_wall_time"] == a["predicted_wall_time"]
        assert got["report"]["iteration_time"] == r["iteration_time"]
        assert got["report"]["idle"] == r["idle"]


def _gpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


GPU_CASES = [(1, 2, ""), (1, 3, ""), (1, 1, ""), (2, 2, "148,74"), (2, 3, "148,74"), (2, 0, "")]


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,stage,sms", GPU_CASES)
def test_reference_pipeline_on_b200_ranks(cuda, ranks, stage, sms):
    if _gpus() < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    args = ["--ranks", str(ranks), "--stage", str(stage), "--gbs", "24"] + (["--sm", sms] if sms else [])
    rc, d = _run(args)
    assert "error" not in d, d
    assert d["plan_parity_reference_profile"] == [] and d["plan_parity_lockstep_profile"] == [], d
    assert d["oom_is_nullopt"] is True
    assert rc == 0
    for prof in (d["reference_profile"], d["lockstep_profile"]):
        assert len(prof["devices"]) == ranks
        for dev in prof["devices"]:
            assert dev["mbs"] >= 1 and len(dev["samples"]) >= 1
            assert all(t > 0 for _, t in dev["samples"])
    assert sum(d["reference_plan"]["gmbs"]) == 24 and sum(d["lockstep_plan"]["gmbs"]) == 24
    sim, ex = d["reference_simulate_on_gpu"], d["executed_iteration"]
    assert sim["iteration_time"] > 0 and all(c > 0 for c in sim["compute"] if c)
    assert ex["iteration_time"] > 0 and ex["throughput"] > 0
    assert all(i >= -1e-6 for i in ex["idle"])
