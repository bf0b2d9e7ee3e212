"""poplar.recalibrate: every rank's profile samples are rescaled by measured / predicted compute of
one planned iteration; the planner itself is unchanged (CPU, no GPU needed)."""
import pytest

from paper_2408_12596_b200 import poplar


def _profile():
    return {"effective_stage": 2, "n": 2, "devices": [
        {"device_id": 0, "mbs": 64, "probes_used": 5, "optimizer_time": 0.01,
         "samples": [(1, 0.010), (2, 0.018), (4, 0.034), (8, 0.066)]},
        {"device_id": 1, "mbs": 64, "probes_used": 5, "optimizer_time": 0.02,
         "samples": [(1, 0.020), (2, 0.036), (4, 0.068), (8, 0.132)]}]}


def test_recalibrate_scales_each_rank():
    prof = _profile()
    plan = {"stage": 2, "gas": 2, "devices": [{"predicted_time": 0.100}, {"predicted_time": 0.200}]}
    out = poplar.recalibrate(prof, plan, [{"compute": 0.110}, {"compute": 0.200}])
    r = 0.110 / 0.100
    assert out["devices"][0]["samples"] == [(b, t * r) for b, t in prof["devices"][0]["samples"]]
    assert out["devices"][1]["samples"] == prof["devices"][1]["samples"]
    assert out["devices"][0]["mbs"] == 64 and out["devices"][0]["optimizer_time"] == 0.01
    # the input profile is not modified
    assert prof["devices"][0]["samples"][0] == (1, 0.010)


def test_recalibrate_keeps_idle_rank():
    prof = _profile()
    plan = {"stage": 2, "gas": 1, "devices": [{"predicted_time": 0.0}, {"predicted_time": 0.2}]}
    out = poplar.recalibrate(prof, plan, [{"compute": 0.0}, {"compute": 0.1}], slow_only=False)
    assert out["devices"][0]["samples"] == prof["devices"][0]["samples"]
    assert out["devices"][1]["samples"][3][1] == pytest.approx(0.066)


def test_recalibrate_passes_compose():
    """bench.py repeats the correction (--recalibrate-passes): a second pass whose measured
    compute matches the corrected prediction leaves the profile unchanged, and two partial
    corrections compose to the product of their ratios."""
    prof = _profile()
    plan = {"stage": 2, "gas": 2, "devices": [{"predicted_time": 0.100}, {"predicted_time": 0.200}]}
    once = poplar.recalibrate(prof, plan, [{"compute": 0.105}, {"compute": 0.190}])
    plan2 = {"stage": 2, "gas": 2, "devices": [{"predicted_time": 0.105}, {"predicted_time": 0.190}]}
    twice = poplar.recalibrate(once, plan2, [{"compute": 0.105}, {"compute": 0.190}])
    assert twice["devices"] == once["devices"]
    third = poplar.recalibrate(once, plan2, [{"compute": 0.1155}, {"compute": 0.190}])
    for (b, t0), (_, t2) in zip(prof["devices"][0]["samples"], third["devices"][0]["samples"]):
        assert t2 == pytest.approx(t0 * 1.05 * 1.1)


@pytest.mark.parametrize("stage,gas", [(1, 3), (2, 4), (3, 6)])
def test_recalibrated_link_reproduces_the_measured_comm(stage, gas):
    """With the fitted link model the reference's additive comm cost (comm.cpp:101-120) of one
    iteration equals the measured exposed comm it was fitted to."""
    from paper_2408_12596_b200 import host, poplar
    from paper_2408_12596_b200.host import ClusterSpec, Device, ModelSpec
    psi = 6.738e9
    link = poplar.recalibrate_link((845e9, 26e-6), stage, gas, 0.108, psi)
    model = ModelSpec(psi, 4096, 32, 2.0, 16.0)
    cl = ClusterSpec([Device(1.0, 1.0, 0.0, 1.0)] * 4, [link[0]] * 4, link[1])
    cp = host.product().make_comm_profile(model, stage, cl)
    charged = (gas * cp.time_per_step if stage >= 2 else 0.0) + cp.sync_time
    assert charged == pytest.approx(0.108, rel=1e-12)


def test_recalibrate_only_slows():
    """A rank measured faster than predicted keeps its curve (its speed-up came from idling under
    the power cap); with slow_only=False it is credited."""
    prof = _profile()
    plan = {"stage": 3, "gas": 2, "devices": [{"predicted_time": 0.100}, {"predicted_time": 0.200}]}
    out = poplar.recalibrate(prof, plan, [{"compute": 0.090}, {"compute": 0.220}])
    assert out["devices"][0]["samples"] == prof["devices"][0]["samples"]
    assert out["devices"][1]["samples"][0][1] == pytest.approx(0.020 * 1.1)
    both = poplar.recalibrate(prof, plan, [{"compute": 0.090}, {"compute": 0.220}], slow_only=False)
    assert both["devices"][0]["samples"][0][1] == pytest.approx(0.010 * 0.9)
