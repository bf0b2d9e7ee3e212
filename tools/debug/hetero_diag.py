"""2-rank diagnostic: per-rank profile samples, the planner's predicted step time for the chosen
batch, and the measured per-micro-step compute time of the executed plan."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
from paper_2408_12596_b200.runtime import Runtime, MODELS, nccl_unique_id
from paper_2408_12596_b200 import poplar, host

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
nid = [nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(nid, 0)
tiers = [132, 66]
rt = Runtime(MODELS["gpt2-small"], rank=rank, world_size=world, device=rank, nccl_id=nid[0], sm_budget=tiers[rank % 2], seed=0)
gbs = 512 * world
prof = rt.profile(2)
plan = poplar.poplar_plan(rt, prof, gbs, 2, world)
first, count = poplar.rank_slice(plan, rank)
rt.load_tokens(first_sample=first, count=max(count, 1), iteration=0)
api = host.product()
for _ in range(2):
    rt.execute_iteration(plan, 2)
ts = [rt.execute_iteration(plan, 2) for _ in range(3)]
if rank == 0:
    for d in prof["devices"]:
        print("rank", d["device_id"], "mbs", d["mbs"], "samples", [(s[0], round(s[1] * 1e3, 2), round(s[0] / s[1], 1)) for s in d["samples"]])
        c = api.build_curve(d["samples"], d["mbs"]) if hasattr(api, "build_curve") else None
    print("plan", [(x["b"], x["lbs"], x["gmbs"], round(x["predicted_time"] * 1e3, 2)) for x in plan["devices"]], "gas", plan["gas"], "pred wall", plan["predicted_wall_time"])
out = [None] * world
dist.all_gather_object(out, [{k: t[k] for k in ("forward", "backward", "comm", "wall", "micro_steps")} for t in ts])
if rank == 0:
    for r, tl in enumerate(out):
        for t in tl:
            print("rank", r, "fwd+bwd per micro-step ms", round((t["forward"] + t["backward"]) / t["micro_steps"] * 1e3, 2), "comm", round(t["comm"] * 1e3, 2), "wall", round(t["wall"] * 1e3, 2))
dist.barrier()
rt.close()
