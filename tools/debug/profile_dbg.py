import sys, os, json
sys.path.insert(0, os.getcwd())
from paper_2408_12596_b200.runtime import Runtime, MODELS
from paper_2408_12596_b200 import poplar
rt = Runtime(MODELS["gpt2-small"], sm_budget=132, seed=0)
rt.load_tokens(count=512)
for rep in range(3):
    prof = rt.profile(2)
    d = prof["devices"][0]
    print("mbs", d["mbs"], "opt", d["optimizer_time"], "samples", [(s[0], round(s[1] * 1e3, 2), round(s[0] / s[1], 1)) for s in d["samples"]])
    plan = poplar.poplar_plan(rt, prof, 512, 2, 1)
    print("plan", [(x["b"], x["lbs"], x["gmbs"]) for x in plan["devices"]], plan["gas"], plan["predicted_wall_time"])
