"""Measured speed of one rank at each emulated SM tier, with and without green-context confinement.

    python tools/tier_ratio.py [--model gpt2-small] [--batch 16] [--stage 2]

For every budget: the SMs the rank was granted, probe-step compute (forward + backward) and the
AdamW pass, each the median of 5 steps after 2 warm-ups; printed as one JSON line per budget and
a summary of speed ratios against the full GPU. Green contexts (ZP_GREEN=1, default) confine every
kernel to the partition; ZP_GREEN=0 caps only the grids of the persistent GEMM / attention kernels.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def measure(model, budget, batch, stage, green):
    os.environ["ZP_GREEN"] = "1" if green else "0"
    from paper_2408_12596_b200.runtime import Runtime
    rt = Runtime(model, sm_budget=budget, seed=0)
    sms, is_green = rt.sm_info()
    comp, opt = [], []
    for i in range(7):
        t = rt.run_step(batch, stage, batch)
        if i >= 2:
            comp.append(t["forward_compute"] + t["backward_compute"])
            opt.append(t["optimizer_step"])
    rt.close()
    return {"budget": budget, "sms": sms, "green": is_green, "compute_s": statistics.median(comp),
            "optimizer_s": statistics.median(opt)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt2-small")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--stage", type=int, default=2)
    ap.add_argument("--budgets", default="148,132,104,74,66")
    a = ap.parse_args()
    from paper_2408_12596_b200.models import MODELS
    model = MODELS[a.model]
    out = []
    for green in (True, False):
        for b in [int(x) for x in a.budgets.split(",")]:
            r = measure(model, b, a.batch, a.stage, green)
            out.append(r)
            print(json.dumps(r), flush=True)
    for green in (True, False):
        rows = [r for r in out if r["green"] == green or (r["sms"] >= 148 and not green)]
        full = next((r for r in out if r["budget"] >= 148 and r["green"] is False), None)
        if not full:
            continue
        print(json.dumps({"green": green, "speed_vs_full": {r["budget"]: round(full["compute_s"] / r["compute_s"], 3)
                                                            for r in out if (r["green"] == green) or r["budget"] >= 148},
                          "adam_vs_full": {r["budget"]: round(full["optimizer_s"] / r["optimizer_s"], 3)
                                           for r in out if (r["green"] == green) or r["budget"] >= 148}}))


if __name__ == "__main__":
    main()
