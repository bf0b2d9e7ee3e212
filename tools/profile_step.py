"""One micro-step iteration (default GPT-2 small ZeRO-2) between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and single-kernel captures.

    python tools/profile_step.py [--b 32] [--sm 132] [--model gpt2-small] [--stage 2]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2408_12596_b200.models import MODELS  # noqa: E402
from paper_2408_12596_b200.runtime import Runtime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--sm", type=int, default=132)
    ap.add_argument("--model", default="gpt2-small")
    ap.add_argument("--stage", type=int, default=2)
    a = ap.parse_args()
    rt = Runtime(MODELS[a.model], sm_budget=a.sm, seed=0)
    rt.resident_bytes(a.stage)
    rt.load_tokens(count=a.b)
    plan = dict(stage=a.stage, gbs=a.b, gas=1, devices=[dict(device_id=0, b=a.b, gmbs=a.b, lbs=a.b, predicted_time=0.0)],
                iteration_time=0.0, idle=[0.0], under_utilization=[0.0], objective=0.0, weights=[1.0],
                predicted_wall_time=0.0)
    for _ in range(2):
        t = rt.execute_iteration(plan, a.stage)
    cudart = ctypes.CDLL("libcudart.so.12")
    cudart.cudaProfilerStart()
    t = rt.execute_iteration(plan, a.stage)
    rt.sync()
    cudart.cudaProfilerStop()
    print({k: (round(v * 1e3, 3) if isinstance(v, float) else v) for k, v in t.items() if k != "coll_times"})
    rt.close()


if __name__ == "__main__":
    main()
