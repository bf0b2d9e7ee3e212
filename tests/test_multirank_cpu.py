"""World-size-2 host logic on CPU (gloo): every rank derives the same Poplar plan from the
all-gathered profile, the ranks' sample ranges partition the global batch, and the
per-rank timings combine into the reference's IterationReport identities."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_12596_b200 import host, poplar

        class FakeRt:  # the planner only needs the model shape and parameter count
            class model:
                d_model, n_layer = 768, 12
            param_count = 124_439_808

        # each rank contributes its own measured samples (different speed tiers)
        mine = {"device_id": rank, "mbs": 200 - 80 * rank, "probes_used": 9, "optimizer_time": 0.004,
                "samples": [(b, (0.01 + b * 0.0015 * (1 + rank))) for b in (1, 2, 4, 8, 16, 32, 64, 120 - 80 * rank + 80)]}
        mine["samples"] = [s for s in mine["samples"] if s[0] <= mine["mbs"]]
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        profile = {"effective_stage": 2, "devices": allp}
        plan = poplar.poplar_plan(FakeRt, profile, 1024, 2, world)
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        assert all(p == plans[0] for p in plans)
        first, count = poplar.rank_slice(plan, rank)
        ranges = [None] * world
        dist.all_gather_object(ranges, (first, count))
        covered = sorted(ranges)
        assert covered[0][0] == 0
        for (f0, c0), (f1, _) in zip(covered, covered[1:]):
            assert f0 + c0 == f1
        assert covered[-1][0] + covered[-1][1] == 1024
        # timings: fast rank waits inside the collectives
        t = {"compute": 1.0 + rank, "optimizer": 0.01, "wall": 2.1, "coll_times": [0.05 + 0.9 * (1 - rank), 0.02]}
        ts = [None] * world
        dist.all_gather_object(ts, t)
        rep = poplar.iteration_report(ts, 1024)
        assert rep["iteration_time"] == 2.1
        assert rep["comm_total"] == pytest.approx(0.07)
        assert rep["idle"][1] == pytest.approx(2.1 - (2.0 + 0.07 + 0.01))
        q.put((rank, "ok", plan["gas"], [d["b"] for d in plan["devices"]]))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def test_two_rank_plan_agreement():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
    assert res[0][2] == res[1][2] and res[0][3] == res[1][3]
