"""NVLink roofline for the ZeRO collectives (RS/AG are NVLink-bound, report them
against measured link bandwidth). On the ZeRO-2 layout of a model (Psi bf16 parameters, equal
1/n shards), every rank times, with CUDA events on its runtime stream:

  peer_rs   - the pull reduce-scatter kernel (peer_rs_acc_k: each rank reads its shard of every
              peer's bf16 gradient over NVLink and sums in fp32)
  peer_ag   - the pull all-gather kernel (peer_ag_k)
  copy_pull - copy-engine pulls of every peer's shard (cudaMemcpyAsync on IPC-mapped memory;
              the ZeRO-3 prefetch path): the link bandwidth a DMA engine reaches
  nccl_rs / nccl_ag - NCCL reduce_scatter_tensor / all_gather_into_tensor (bf16) on the same sizes

and rank 0 prints one JSON line: per collective the per-call time (max over ranks) and the bytes
each rank pulls over NVLink per call, (n-1)/n * Psi * 2, divided by that time (GB/s per rank,
per direction; NCCL's "busbw" for RS/AG is the same quantity).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_bench.py \
        [--model gpt2-small] [--reps 20] [--out FILE]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2408_12596_b200.runtime import MODELS, Runtime, nccl_unique_id  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt2-small")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world < 2:
        raise SystemExit("run under torchrun with >= 2 ranks")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ids = [None] * world
    dist.all_gather_object(ids, nccl_unique_id() if rank == 0 else None)
    rt = Runtime(MODELS[a.model], rank=rank, world_size=world, device=local, nccl_id=ids[0], seed=0)
    res = {}
    if rt.peer_collectives():
        for which, name in ((0, "peer_rs"), (1, "peer_ag"), (2, "copy_pull")):
            sec, pulled = rt.bench_collective(which, a.reps)
            res[name] = (sec, pulled)
    # NCCL on the same element counts
    psi = rt.padded_params
    full = torch.randn(psi, device="cuda").to(torch.bfloat16)
    shard = torch.empty(psi // world, device="cuda", dtype=torch.bfloat16)
    pulled = (world - 1) * (psi // world) * 2
    for name, fn in (("nccl_rs", lambda: dist.reduce_scatter_tensor(shard, full)),
                     ("nccl_ag", lambda: dist.all_gather_into_tensor(full, shard))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = (e0.elapsed_time(e1) * 1e-3 / a.reps, pulled)
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        out = {"model": a.model, "params_padded": psi, "n_ranks": world, "reps": a.reps,
               "unit": "GB/s per rank per direction (bytes pulled from peers / time)",
               "nominal_nvlink_gbs_per_direction": 900.0, "collectives": {}}
        for name in res:
            t = max(r[name][0] for r in allres)
            b = res[name][1]
            out["collectives"][name] = {"ms": t * 1e3, "bytes_pulled": b, "gbs": b / t / 1e9,
                                        "frac_of_nominal": b / t / 1e9 / 900.0}
        text = json.dumps(out)
        if a.out:
            with open(a.out, "w") as f:
                f.write(text + "\n")
        print(text)
    rt.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
