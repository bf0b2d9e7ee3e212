"""HBM roofline of the peer-collective kernels with every rank emulated on ONE GPU (one cooperative
launch per call, zp_kernels.h peer group): the bytes a rank pulls over NVLink in production become
local HBM reads here, so the kernels are timed against the HBM peak. For ncu, each kernel is
launched `--reps` times after one warm-up.

    python tools/peer_bench.py [--n 4] [--len 33554432] [--reps 5]

Algorithmic bytes per call (all ranks):
  reduce-scatter  n * (n * len * 2 (bf16 shards read) + len * 4 (fp32 accumulator write))
  fused RS+AdamW  n * (n * len * 2 + len * (4 acc + 24 p/m/v read+write + 4 grad out) + n * len * 2 (push))
  all-gather      n * (n * len * 2 (shards read) + n * len * 2 (written))
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--len", type=int, default=1 << 25)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ctas", type=int, default=148 // 4)
    a = ap.parse_args()
    import torch
    from tests.test_peer_gpu import AdamP, Group, lib
    n, L = a.n, a.len
    g = Group(n, {"src": (n * L, torch.bfloat16), "p16": (n * L, torch.bfloat16), "p32": (L, torch.float32),
                  "m": (L, torch.float32), "v": (L, torch.float32), "acc": (L, torch.float32),
                  "gout": (L, torch.float32), "dst": (n * L, torch.bfloat16)})
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    adam = AdamP(1e-4, 0.9, 0.95, 1e-8, 0.0, 0.1, 0.05)
    calls = {
        "peer_rs_acc_k": (lambda e: lib().zp_peer_rs_accumulate(g.h, g.off("src"), L, g.off("acc"), 1, e, a.ctas, st),
                          n * (n * L * 2 + L * 4)),
        "peer_rs_adam_ag_k": (lambda e: lib().zp_peer_rs_adam_ag(g.h, g.off("src"), 0, L, g.off("acc"), g.off("p32"),
                                                                 g.off("m"), g.off("v"), g.off("p16"), g.off("gout"),
                                                                 C.byref(adam), e, a.ctas, st),
                              n * (n * L * 2 + L * 32 + n * L * 2)),
        "peer_ag_k": (lambda e: lib().zp_peer_all_gather(g.h, g.off("p32"), g.off("dst"), L, e, a.ctas, st),
                      n * (n * L * 2 * 2)),
    }
    out = {}
    for name, (fn, nbytes) in calls.items():
        assert fn(g.next_epoch()) == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            assert fn(g.next_epoch()) == 0
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) * 1e-3 / a.reps
        out[name] = {"ranks": n, "len_per_rank": L, "ms": sec * 1e3, "bytes": nbytes,
                     "GBps": nbytes / sec / 1e9}
        print(json.dumps({name: out[name]}), flush=True)
    g.close()


if __name__ == "__main__":
    main()
