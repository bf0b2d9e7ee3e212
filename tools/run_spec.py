"""Run a reference experiment spec (proj/core/src/experiment.cpp format) on emulated B200 ranks:
Alg. 1 profile on the devices, Alg. 2 plan, then the measured iterations of the Poplar plan and
of the heterogeneity-blind uniform plan, printed as the reference's report objects
(`profile`, `plan`, `simulate` with measured values; `speedup_vs_baseline` = uniform T / Poplar T).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/run_spec.py SPEC.json \
        [--iterations K] [--model gpt2-small]

One rank per spec device (WORLD_SIZE must equal the number of devices); rank 0 prints the JSON.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2408_12596_b200 import poplar, spec as specmod  # noqa: E402
from paper_2408_12596_b200.models import MODELS  # noqa: E402
from paper_2408_12596_b200.runtime import Runtime, nccl_unique_id  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("spec")
    ap.add_argument("--iterations", type=int, default=0, help="cap the spec's iteration count")
    ap.add_argument("--model", default="")
    ap.add_argument("--out", default="", help="write the report here (default: stdout)")
    a = ap.parse_args()
    sp = specmod.parse_spec(a.spec)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != len(sp["cluster"]["devices"]):
        raise SystemExit(f"spec has {len(sp['cluster']['devices'])} devices, WORLD_SIZE is {world}")
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")

    def allgather(obj):
        if dist is None:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    sm, cap = specmod.emulation(sp)[rank]
    model_name = a.model or sp["b200"].get("model", "gpt2-small")
    model = MODELS[model_name]
    nid = allgather(nccl_unique_id() if rank == 0 and world > 1 else None)[0]
    rt = Runtime(model, rank=rank, world_size=world, device=local, nccl_id=nid, sm_budget=sm,
                 hbm_cap_bytes=cap, seed=sp["seed"])
    gbs = sp["gbs"]
    profile = rt.profile(sp["stage"])
    stage = profile["effective_stage"]
    plan = poplar.poplar_plan(rt, profile, gbs, stage, world)
    uniform = poplar.poplar_plan(rt, profile, gbs, stage, world, uniform=True)
    iters = min(sp["iterations"], a.iterations) if a.iterations else sp["iterations"]

    def run(p):
        first, count = poplar.rank_slice(p, rank)
        rt.load_tokens(first_sample=first, count=max(count, 1), iteration=0)
        rt.execute_iteration(p, stage)  # warm-up
        reps = []
        for _ in range(iters):
            t = rt.execute_iteration(p, stage)
            reps.append(poplar.iteration_report(allgather(t), gbs))
        return reps

    base = run(uniform)
    pop = run(plan)
    if rank == 0:
        base_sim = specmod.sim_report(base, rt.param_count)
        out = {"profile": specmod.profile_report(profile, sp), "plan": specmod.plan_report(plan),
               "simulate": specmod.sim_report(pop, rt.param_count, base_sim["mean"]["T"]),
               "baseline": {"plan": specmod.plan_report(uniform), "simulate": base_sim},
               "b200": {"model": model_name,
                        "emulation": [{"name": d["name"], "sm_budget": e[0], "hbm_cap": e[1]}
                                      for d, e in zip(sp["cluster"]["devices"], specmod.emulation(sp))],
                        "measured": True}}
        text = json.dumps(out, indent=2)
        if a.out:
            with open(a.out, "w") as f:
                f.write(text + "\n")
        else:
            print(text)
    rt.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
