"""Generate tests/golden/planner_golden.json from the compiled reference (oracle/_ref).

Run here (where /root/reference exists): python tests/golden/make_planner_golden.py
Each case stores the inputs and the reference's full pipeline output (profile, plan,
comm profile, uniform plan, simulated reports); doubles survive the JSON round trip
exactly (repr round-trip).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from test_planner_parity import full_pipeline, mixed_cluster  # noqa: E402


def main():
    assert oracle.build_reference(), "reference build failed"
    ref = oracle.reference()
    cases = []
    cl, m = mixed_cluster()
    insts = [(cl, m, 64, s) for s in (None, 0, 1, 2, 3)]
    for idx in range(0, 500, 8):
        insts.append(oracle.fuzz_instance(idx))
    for cl, m, gbs, st in insts:
        cases.append({
            "cluster": {"devices": [d.__dict__ for d in cl.devices], "link_bandwidths": cl.link_bandwidths,
                        "link_latency": cl.link_latency, "seed": cl.seed, "jitter": cl.jitter},
            "model": m.__dict__, "gbs": gbs, "stage_request": st,
            "expect": json.loads(json.dumps(full_pipeline(ref, cl, m, gbs, st))),
        })
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "planner_golden.json")
    with open(out, "w") as f:
        json.dump(cases, f)
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    main()
