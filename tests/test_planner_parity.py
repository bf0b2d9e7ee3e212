"""Host planner parity: the product (libzp.so) against the reference's own sources
(oracle/_ref/libzpref.so, compiled from /root/reference by oracle/Makefile).

Bar: bit-exact. Every double of every ProfileResult / AllocationPlan / IterationReport
field is compared with ==. Known-answer tests restate the reference's unit tests
(proj/tests/test_*.cpp) and the compiled-reference goldens of SURVEY.md Appendix B.
"""
import json
import math
import os
import random

import pytest

from paper_2408_12596_b200 import host
from paper_2408_12596_b200.host import ClusterSpec, Device, ModelSpec, CommProfile

import oracle

GiB = float(1 << 30)
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def prod():
    return host.product()


@pytest.fixture(scope="module")
def ref():
    if not oracle.available() and not oracle.build_reference():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return oracle.reference()


def mixed_cluster():
    # Shape of proj/tests/data/mixed_cluster.json: 2 fast + 2 slow, 16 GiB, 256 MiB/batch.
    fast = Device(16 * GiB, 256 * float(1 << 20), 0.02, 0.01)
    slow = Device(16 * GiB, 256 * float(1 << 20), 0.02, 0.02)
    return ClusterSpec([fast, fast, slow, slow], [12e9] * 4, 1e-4, 42), ModelSpec(5e8, 1024, 8)


def constant_profile(speeds, mbs):
    return {"effective_stage": 0,
            "devices": [{"device_id": i, "mbs": mbs, "samples": [(1, 1.0 / s)]} for i, s in enumerate(speeds)]}


def affine_profile(params):
    devs = []
    for i, (c0, c1, mbs) in enumerate(params):
        devs.append({"device_id": i, "mbs": mbs, "samples": [(b, c0 + c1 * float(b)) for b in range(1, mbs + 1)]})
    return {"effective_stage": 3, "devices": devs}


def comm_step(t, sync=0.0):
    return CommProfile(3, 0.0, 0.0, 0.0, t, sync)


# ---------------------------------------------------------------- known answers (product only)

def test_kat_appendix_b_fixture(prod):
    cl, m = mixed_cluster()
    golden = {0: (34, 0.23880634587026597, 0.4055730125369326, 1.6011035413786812),
              1: (50, 0.2387979326439084, 0.40556459931057504, 1.6225469331654148),
              2: (53, 0.23879694367734058, 0.4056636103440072, 1.6244903371501367),
              3: (56, 0.23879606290100389, 0.4890960629010038, 1.6261448181442764)}
    for st, (mbs, T, wall, obj) in golden.items():
        p = prod.profile_cluster(cl, m, st)
        assert [d["mbs"] for d in p["devices"]] == [mbs] * 4
        pl = prod.plan(64, p, st, m, cl)
        assert [d["b"] for d in pl["devices"]] == [21, 21, 11, 11]
        assert [d["gmbs"] for d in pl["devices"]] == [21, 21, 11, 11]
        assert [d["lbs"] for d in pl["devices"]] == [21, 21, 11, 11]
        assert pl["gas"] == 1
        assert pl["iteration_time"] == T
        assert pl["predicted_wall_time"] == wall
        assert pl["objective"] == obj
    p0 = prod.profile_cluster(cl, m, 0)
    assert p0["devices"][0]["samples"] == [(1, .03), (2, .04), (4, .06), (8, .1), (16, .18), (32, .34),
                                           (34, 0.36000000000000004)]
    c_fast = prod.build_curve(p0["devices"][0]["samples"], 34)
    c_slow = prod.build_curve(p0["devices"][2]["samples"], 34)
    assert c_fast["peak_speed"] == 94.44444444444443 and c_fast["peak_range"] == (18, 34)
    assert c_slow["peak_speed"] == 48.57142857142857 and c_slow["peak_range"] == (12, 34)


def test_kat_compare_speedups(prod):
    cl, m = mixed_cluster()
    for st, want in ((0, 1.2458411865934609), (3, 1.2039567611666326)):
        p = prod.profile_cluster(cl, m, st)
        pl = prod.plan(64, p, st, m, cl)
        comm = prod.make_comm_profile(m, st, cl)
        tail = max(d["optimizer_time"] for d in p["devices"])
        un = prod.make_uniform_plan(64, p, st, comm, tail)
        a = prod.simulate_run(cl, m, pl, st, 50)
        b = prod.simulate_run(cl, m, un, st, 50)
        assert a["throughput"] / b["throughput"] == want


def test_kat_spline(prod):
    assert prod.spline_eval([1, 2, 3, 4], [1, 8, 27, 64], [2.5])[0] == pytest.approx(15.25, rel=1e-12)
    assert prod.spline_eval([0, 1, 2], [0, 1, 2], [1.5])[0] == pytest.approx(1.5, rel=1e-12)
    assert prod.spline_eval([1, 3], [2, 6], [2.0])[0] == pytest.approx(4.0, rel=1e-12)
    assert prod.spline_eval([1, 2], [5, 7], [0.5, 3.0]) == [5.0, 7.0]
    _, segs = prod.spline_fit([0, 1, 2], [0, 1, 2])
    assert all(abs(s[2]) <= 1e-9 and abs(s[3]) <= 1e-9 for s in segs)
    # unsorted input is sorted internally
    assert prod.spline_eval([3, 1, 2], [9, 1, 4], [2.5]) == prod.spline_eval([1, 2, 3], [1, 4, 9], [2.5])
    for bad in ([1], [], [1, 1]):
        with pytest.raises(host.InvalidInputError):
            prod.spline_fit(bad, [1.0] * len(bad))


def test_kat_hardware_and_comm(prod):
    m = ModelSpec(1e9, 1024, 8)
    assert prod.resident_state_bytes(m, 0, 8) == 16e9
    assert prod.resident_state_bytes(m, 3, 8) == 2e9
    assert prod.resident_state_bytes(m, 1, 4) == 7e9
    assert prod.resident_state_bytes(m, 2, 4) == 5.5e9
    one = ClusterSpec([Device(64 * GiB, GiB, 0.1, 0.05)], [1e9])
    t = prod.run_step(one, 0, ModelSpec(1e8), 4, 0)
    assert t["forward_compute"] + t["backward_compute"] == pytest.approx(0.3, rel=1e-12)
    oom = ClusterSpec([Device(10e9, 1e9, 0.0, 0.01)], [1e9])
    assert prod.run_step(oom, 0, ModelSpec(0.5e9), 2, 0) is not None
    assert prod.run_step(oom, 0, ModelSpec(0.5e9), 3, 0) is None
    probe = prod.memory_probe(ClusterSpec([Device(16 * GiB, 0.5 * GiB, 0.0, 0.01)], [1e9]), 0,
                              ModelSpec(4 * GiB / 16), 0)
    assert probe == (4 * GiB, 4.5 * GiB, 16 * GiB)
    assert prod.ffn_volumes(1, 1) == (8, 16, 24)
    assert prod.ffn_volumes(1024, 8)[0] == 1 << 26
    with pytest.raises(host.InvalidInputError):
        prod.run_step(one, 0, ModelSpec(1e8), 0, 0)
    with pytest.raises(host.InvalidInputError):
        prod.run_step(one, 3, ModelSpec(1e8), 1, 0)


def test_kat_planner(prod):
    p = prod.plan_zero01(8, constant_profile([3.0, 1.0], 32))
    assert [d["gmbs"] for d in p["devices"]] == [6, 2]
    assert prod.allocate_remainder([6, 3], constant_profile([2.0, 1.0], 32), 1) == [7, 3]
    assert prod.allocate_remainder([2, 2, 2], constant_profile([1.0, 1.0, 1.0], 32), 3) == [3, 3, 3]
    p = prod.plan_zero01(10, constant_profile([2.0, 1.0], 32))
    assert [d["gmbs"] for d in p["devices"]] == [7, 3]
    assert p["iteration_time"] == pytest.approx(3.5, rel=1e-12)
    p = prod.plan_zero01(1, constant_profile([2.0, 1.0, 1.0], 8))
    assert [d["gmbs"] for d in p["devices"]] == [1, 0, 0]
    p = prod.plan_zero23(24, affine_profile([(0.1, 0.05, 8), (0.1, 0.1, 4)]), comm_step(0.2))
    assert p["gas"] == 2 and [d["b"] for d in p["devices"]] == [8, 4]
    p = prod.plan_zero23(8, affine_profile([(0.1, 0.05, 8)]), comm_step(0.25))
    assert p["gas"] == 1 and p["devices"][0]["b"] == 8 and p["devices"][0]["lbs"] == 8
    assert p["predicted_wall_time"] == pytest.approx(0.75, rel=1e-9)


def test_kat_profiler(prod):
    # mbs search finds the exact latent threshold (reference test_profiler.cpp:149-182 style)
    rnd = random.Random(7)
    m = ModelSpec(100000.0, 256, 4)
    resident = prod.resident_state_bytes(m, 0, 1)
    for _ in range(100):
        thr = rnd.randint(1, 4096)
        act = float(rnd.randint(1 << 18, 1 << 24))
        total = resident + act * thr + float(rnd.randint(0, int(act) - 1))
        cl = ClusterSpec([Device(total, act, 0.05, 0.01)], [1e9])
        est = prod.estimate_theoretical_mbs(cl, 0, m, 0)
        r = prod.search_mbs(cl, 0, m, 0, est if rnd.random() < 0.5 else thr + rnd.randint(0, 2048))
        assert r["mbs"] == thr
        assert r["probes_used"] <= 2 * math.ceil(math.log2(max(thr, 2))) + 4
    # infeasible at every stage
    big = ClusterSpec([Device(GiB, 256 * float(1 << 20), 0.02, 0.01)], [1e9])
    with pytest.raises(host.InfeasibleError):
        prod.profile_cluster(big, ModelSpec(5e9), None)


# ---------------------------------------------------------------- differential vs compiled reference

def assert_same(a, b):
    assert a == b, f"\nproduct  : {a}\nreference: {b}"


def full_pipeline(api, cl, m, gbs, st_req):
    out = {}
    try:
        prof = api.profile_cluster(cl, m, st_req)
    except host.ZeroplanError as e:
        return {"error": type(e).__name__}
    out["profile"] = prof
    st = prof["effective_stage"]
    pl = api.plan(gbs, prof, st, m, cl)
    out["plan"] = pl
    comm = api.make_comm_profile(m, st, cl)
    out["comm"] = (comm.time_per_step, comm.sync_time, comm.volume_forward, comm.volume_backward,
                   comm.volume_optimizer)
    tail = max(d["optimizer_time"] for d in prof["devices"])
    un = api.make_uniform_plan(gbs, prof, st, comm, tail)
    out["uniform"] = un
    out["sim"] = api.simulate_run(cl, m, pl, st, 5)
    out["sim_uniform"] = api.simulate_run(cl, m, un, st, 5)
    return out


def test_acceptance_fuzz_instances_bit_exact(prod, ref):
    """The reference acceptance suite's 500 fuzz instances (acceptance.cpp:72-110)."""
    for idx in range(500):
        cl, m, gbs, st = oracle.fuzz_instance(idx)
        assert_same(full_pipeline(prod, cl, m, gbs, st), full_pipeline(ref, cl, m, gbs, st))


def test_jitter_and_escalation_bit_exact(prod, ref):
    rnd = random.Random(11)
    for trial in range(120):
        n = rnd.randint(1, 8)
        devs = []
        for _ in range(n):
            devs.append(Device(rnd.uniform(2, 64) * GiB, rnd.uniform(16, 512) * float(1 << 20),
                               rnd.uniform(0.0, 0.3), rnd.uniform(0.001, 0.2), rnd.uniform(0.0, 0.05)))
        cl = ClusterSpec(devs, [10 ** rnd.uniform(8, 11) for _ in range(n)], rnd.uniform(0, 1e-3),
                         rnd.getrandbits(64), rnd.choice([0.0, 0.05, 0.2]))
        m = ModelSpec(rnd.uniform(1e7, 4e9), 1024, 8)
        gbs = rnd.randint(1, 2048)
        st = rnd.choice([None, 0, 1, 2, 3])
        assert_same(full_pipeline(prod, cl, m, gbs, st), full_pipeline(ref, cl, m, gbs, st))


def random_profile(rnd, n, stage):
    devs = []
    for i in range(n):
        mbs = rnd.randint(1, 300)
        bs = sorted(rnd.sample(range(1, mbs + 1), min(mbs, rnd.randint(1, 12))))
        c0, c1 = rnd.uniform(0.001, 0.5), rnd.uniform(0.0005, 0.1)
        # measured-looking times: affine plus multiplicative noise (non-monotone speeds)
        samples = [(b, (c0 + c1 * b) * rnd.uniform(0.8, 1.25)) for b in bs]
        devs.append({"device_id": i, "mbs": mbs, "samples": samples, "optimizer_time": rnd.uniform(0, 0.02),
                     "probes_used": len(bs)})
    return {"effective_stage": stage, "devices": devs}


def test_random_measured_profiles_bit_exact(prod, ref):
    """Profiles shaped like measured GPU curves (noisy, non-monotone speed)."""
    rnd = random.Random(1234)
    for trial in range(300):
        n = rnd.randint(1, 8)
        st = rnd.randint(0, 3)
        prof = random_profile(rnd, n, st)
        cl = ClusterSpec([Device(1e12, 1e6, 0.0, 1.0)] * n, [rnd.uniform(1e9, 9e11)] * n, rnd.uniform(0, 1e-4))
        m = ModelSpec(rnd.uniform(1e6, 7e9), 4096, 32)
        gbs = rnd.randint(1, 4096)
        for d in prof["devices"]:
            assert_same(prod.build_curve(d["samples"], d["mbs"], d["device_id"]),
                        ref.build_curve(d["samples"], d["mbs"], d["device_id"]))
        assert_same(prod.plan(gbs, prof, st, m, cl), ref.plan(gbs, prof, st, m, cl))
        comm = prod.make_comm_profile(m, st, cl)
        for s2 in range(4):
            assert_same(prod.make_uniform_plan(gbs, prof, s2, comm, 0.01),
                        ref.make_uniform_plan(gbs, prof, s2, comm, 0.01))


def test_spline_bit_exact(prod, ref):
    rnd = random.Random(101)
    for trial in range(200):
        cnt = rnd.randint(2, 25)
        xs, x = [], rnd.uniform(0.1, 4.0)
        for _ in range(cnt):
            xs.append(x)
            x += rnd.uniform(0.1, 4.0)
        ys = [rnd.uniform(-100, 100) for _ in xs]
        rnd.shuffle(xs)
        assert_same(prod.spline_fit(xs, ys), ref.spline_fit(xs, ys))
        q = [rnd.uniform(min(xs) - 1, max(xs) + 1) for _ in range(50)] + xs
        for deriv in range(3):
            assert_same(prod.spline_eval(xs, ys, q, deriv), ref.spline_eval(xs, ys, q, deriv))


def test_error_taxonomy_matches(prod, ref):
    cl, m = mixed_cluster()
    cases = [
        lambda api: api.profile_cluster(ClusterSpec([], []), m, None),
        lambda api: api.profile_cluster(ClusterSpec([Device(-1, 1, 0, 1)], [1.0]), m, None),
        lambda api: api.profile_cluster(cl, ModelSpec(0.0), None),
        lambda api: api.profile_cluster(ClusterSpec([Device(GiB, 2 * GiB, 0.0, 1.0)], [1.0]), ModelSpec(1e6), None),
        lambda api: api.plan_zero01(0, constant_profile([1.0], 4)),
        lambda api: api.build_curve([(5, 1.0)], 4),
        lambda api: api.build_curve([(1, 0.0)], 4),
        lambda api: api.build_curve([(1, 1.0), (1, 2.0)], 4),
        lambda api: api.search_mbs(cl, 0, m, 0, 0),
        lambda api: api.collective_time(-1.0, cl),
        lambda api: api.allocate_remainder([1], constant_profile([1.0], 4), -1),
    ]
    for f in cases:
        errs = []
        for api in (prod, ref):
            try:
                f(api)
                errs.append(None)
            except host.ZeroplanError as e:
                errs.append((type(e).__name__, str(e)))
        assert errs[0] == errs[1]


def test_committed_golden_vectors(prod):
    """Fixture generated from the compiled reference (tests/golden/make_planner_golden.py)."""
    path = os.path.join(HERE, "golden", "planner_golden.json")
    with open(path) as f:
        cases = json.load(f)
    assert len(cases) >= 50
    for c in cases:
        cl = ClusterSpec([Device(**d) for d in c["cluster"]["devices"]], c["cluster"]["link_bandwidths"],
                         c["cluster"]["link_latency"], c["cluster"]["seed"], c["cluster"]["jitter"])
        m = ModelSpec(**c["model"])
        got = full_pipeline(prod, cl, m, c["gbs"], c["stage_request"])
        assert json.loads(json.dumps(got)) == c["expect"]
