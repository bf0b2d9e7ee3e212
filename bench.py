#!/usr/bin/env python
"""Heterogeneous-ZeRO (Poplar) training step on B200s — benchmark contract.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c5]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU)

Default workload: the largest BASELINE.json configuration that fits one B200 — C5, a
Llama-style 7B (L32 h4096 ffn11008 V32000, s=4096) at ZeRO-3 bf16, ranks cycling the SM tiers
148 / 104 / 74 SMs and HBM caps 180 / 128 GB (rank 0: 148 SMs, full HBM), global batch 32*N
samples (weak scaling). `--config c1..c4` select the other BASELINE configs (C2 = GPT-2 small
ZeRO-2 at 132 / 66 SMs, the round-1 headline).

Per run: measured alpha-beta link model (N > 1), Poplar Alg. 1 profiling on the devices (lockstep
probes), Alg. 2 plan from the bit-exact zeroplan planner (optionally recalibrated from measured
iterations), W warm-up iterations, then K timed iterations bracketed by barrier + device sync,
timed with CUDA events on the runtime stream, max over ranks. `value` = K * gbs / T (samples/s,
whole job). Inputs (tokens) are resident in HBM for `value`; `e2e` re-times the same iterations
through the C ABI with the tokens copied from pinned host memory and the loss read back every step.

Checks reported beside the numbers (the oracle as checker, never as the thing measured):
`plan_parity` — the compiled reference planner (oracle/_ref) re-plans the same measured profile
and every field must match bit for bit; `plan_fidelity` — the planner's predicted wall time against
the measured iteration (reference acceptance criterion 8, 2 %); `reference_prediction` — the
reference's own latent pipeline (profile_cluster -> plan -> simulate_iteration) on a cluster
fitted to the measured curves.

--impl reference times the reference's CPU implementation of the path on the host cores: the
reference has no tensor step (its device step is a closed-form latent model), so the CPU path in
the metric's unit is the float64 oracle port of the step (oracle/step.py); its planner (compiled
from the reference sources, oracle/_ref) is timed beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec (8×B200, emulated hetero) at 1/2/4/8 GPUs; sync idle %"
UNIT = "samples/s"

CONFIGS = {
    # name: model, ZeRO stage, SM tiers (cycled over ranks), HBM caps (GiB, cycled; 0 = full),
    # global batch per GPU (samples)
    "c1": dict(model="gpt-tiny", stage=1, tiers=[148, 74], caps=[0], gbs_per_gpu=32,
               label="C1: GPT-tiny L4 h256 V8192 s256, ZeRO-1, SM 148 vs 74"),
    "c2": dict(model="gpt2-small", stage=2, tiers=[132, 66], caps=[0], gbs_per_gpu=512,
               label="C2: GPT-2 small (124M) s1024, ZeRO-2, SM budgets 132 vs 66"),
    "c3": dict(model="gpt2-medium", stage=3, tiers=[148, 148, 74, 74], caps=[0, 80], gbs_per_gpu=256,
               label="C3: GPT-2 medium (355M) s1024, ZeRO-3, 2 SM tiers (148/74) x 2 HBM caps (180/80 GB)"),
    # 5 fast + 3 slow ranks at N=8 (tier list indexed by rank)
    "c4": dict(model="llama-1.3b", stage=3, tiers=[148, 148, 74, 148, 74, 148, 74, 148], caps=[0],
               gbs_per_gpu=128, label="C4: Llama-style 1.3B s2048, ZeRO-3 bf16, 5 fast (148 SM) + 3 slow (74 SM)"),
    # the memory tier (every 4th rank) holds 128 GB: 6 samples per micro-step instead of 8. A 96 GB
    # tier (3 samples) pinned every lockstep ZeRO-3 micro-step to 3 samples on the fast ranks, so
    # the 104-SM tier could only take 2 and idled 24 % by the planner's own prediction
    # (profiles/r2_bench_lines/g15_c5_n4.json, g20_c5_n4.json)
    # "full Poplar search over global batch" (BASELINE.json): Alg. 2 is evaluated on the measured
    # profile at every global batch of 24..40 samples per GPU; the run uses the batch with the best
    # predicted samples/s (the smallest within 0.1 % of it)
    "c5": dict(model="llama-7b", stage=3, tiers=[148, 104, 74, 148, 104, 74, 148, 74], caps=[0, 0, 0, 128],
               gbs_per_gpu=32, gbs_search=(24, 40, 2),
               label="C5: Llama-style 7B s4096, ZeRO-3 bf16, mixed SM tiers 148/104/74 + HBM caps 180/128 GB"),
}
DEFAULT_CONFIG = "c5"


def env_int(k, d):
    return int(os.environ.get(k, d))


# ---------------------------------------------------------------- clocks during the timed region
class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.out = os.path.join(ROOT, "gpurun_out", f".clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.out), exist_ok=True)
        try:
            self.f = open(self.out, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], 0.0, set()
        try:
            for line in open(self.out):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for nme, v in zip(names, parts[3:7]):
                    if v.lower() == "active":
                        reasons.add(nme)
            os.remove(self.out)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline (oracle port)
def _oracle_params(m, n_layer, rng):
    import numpy as np
    h, f = m.d_model, m.d_ff
    if m.arch == 1:
        P = {"wte": rng.normal(0, 0.02, (m.vocab, h)), "lnf_g": np.ones((1, h)),
             "lm_head": rng.normal(0, 0.02, (m.vocab, h))}
        for i in range(n_layer):
            P.update({f"h{i}.ln1_g": np.ones((1, h)), f"h{i}.w_qkv": rng.normal(0, 0.02, (3 * h, h)),
                      f"h{i}.w_o": rng.normal(0, 0.02, (h, h)), f"h{i}.ln2_g": np.ones((1, h)),
                      f"h{i}.w_gu": rng.normal(0, 0.02, (2 * f, h)), f"h{i}.w_down": rng.normal(0, 0.02, (h, f))})
        return P
    P = {"wte": rng.normal(0, 0.02, (m.vocab, h)), "wpe": rng.normal(0, 0.01, (m.seq_len, h)),
         "lnf_g": np.ones((1, h)), "lnf_b": np.zeros((1, h))}
    for i in range(n_layer):
        P.update({f"h{i}.ln1_g": np.ones((1, h)), f"h{i}.ln1_b": np.zeros((1, h)),
                  f"h{i}.w_qkv": rng.normal(0, 0.02, (3 * h, h)), f"h{i}.b_qkv": np.zeros((1, 3 * h)),
                  f"h{i}.w_o": rng.normal(0, 0.02, (h, h)), f"h{i}.b_o": np.zeros((1, h)),
                  f"h{i}.ln2_g": np.ones((1, h)), f"h{i}.ln2_b": np.zeros((1, h)),
                  f"h{i}.w_fc": rng.normal(0, 0.02, (f, h)), f"h{i}.b_fc": np.zeros((1, f)),
                  f"h{i}.w_proj": rng.normal(0, 0.02, (h, f)), f"h{i}.b_proj": np.zeros((1, h))})
    return P


def cpu_step_sample(model_name: str):
    """Times the float64 oracle step (forward + backward + AdamW) on one sample of the workload on
    all host cores. GPT-2 models run whole; for the Llama models the bounded sample (10-30 s of CPU
    work) is the model cut to one transformer layer (embedding + 1 layer + LM head at full width and
    vocabulary) on the first 1024 tokens of a sample, and the rate is extrapolated to the full
    sample by the FLOP ratio (6*N_matmul*s + 12*L*h*s^2).
    Returns (samples/s, cores, seconds, description)."""
    import dataclasses
    import numpy as np
    from oracle import step as so
    from paper_2408_12596_b200.models import MODELS
    m = MODELS[model_name]
    layers = m.n_layer if m.arch == 0 else 1
    seq = m.seq_len if m.arch == 0 else min(m.seq_len, 1024)
    cut = dataclasses.replace(m, n_layer=layers, seq_len=seq)
    rng = np.random.default_rng(0)
    P = _oracle_params(m, layers, rng)
    tok = rng.integers(0, m.vocab, (1, seq + 1))
    t0 = time.perf_counter()
    _, G = so.loss_and_grads(P, tok, layers, m.n_head, m.vocab, 1, arch=m.arch)
    for k in P:
        so.adamw(P[k], 0.0, 0.0, G[k], 1, 1e-4, 0.9, 0.95, 1e-8, 0.0)
    dt = time.perf_counter() - t0
    scale = cut.flops_per_sample() / m.flops_per_sample()
    desc = (f"1 sample x {model_name} fwd+bwd+AdamW, float64 numpy oracle port (oracle/step.py), {dt:.1f} s"
            + ("" if layers == m.n_layer else
               f"; model cut to {layers} of {m.n_layer} layers and {seq} of {m.seq_len} tokens (full width and "
               f"vocabulary), rate x {scale:.5f} by the FLOP ratio"))
    return scale / dt, os.cpu_count() or 1, dt, desc


def run_reference(args, cfg):
    """--impl reference: the reference's CPU path of the step (see module docstring)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    rate_sum, secs, n = 0.0, 0.0, 0
    cores, desc = os.cpu_count() or 1, ""
    deadline = time.perf_counter() + 150.0
    for k in range(max(1, args.steps)):
        sps, cores, dt, desc = cpu_step_sample(cfg["model"])
        rate_sum += 1.0 / sps
        secs += dt
        n += 1
        if time.perf_counter() > deadline:
            break
    value = n / rate_sum
    planner = reference_planner_ms()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": n, "warmup": 0, "ms_per_step": 1e3 / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["label"], "model": cfg["model"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{n} step(s): {desc}; the reference has no tensor step",
                             "reference_planner_ms": planner},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def reference_planner_ms():
    """The reference's own profile + plan (compiled from /root/reference sources, oracle/_ref) on
    a 2-device latent cluster; single-threaded as written. None if not built."""
    try:
        import oracle
        from paper_2408_12596_b200.host import ClusterSpec, Device, ModelSpec
        if not oracle.available():
            return None
        ref = oracle.reference()
        cl = ClusterSpec([Device(180e9, 0.8e9, 0.01, 0.0015), Device(180e9, 0.8e9, 0.01, 0.003)],
                         [770e9] * 2, 25e-6)
        m = ModelSpec(124.4e6, 768, 12)
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 0.5:
            p = ref.profile_cluster(cl, m, 2)
            ref.plan(1024, p, 2, m, cl)
            n += 1
        return 1e3 * (time.perf_counter() - t0) / n
    except Exception:
        return None


# ---------------------------------------------------------------- checks against the reference
def plans_equal(a: dict, b: dict) -> list:
    """Field-by-field bitwise comparison of two AllocationPlans; returns the differing fields."""
    diffs = []
    for k in ("stage", "gbs", "gas", "iteration_time", "objective", "predicted_wall_time", "idle",
              "under_utilization", "weights"):
        if a[k] != b[k]:
            diffs.append(k)
    for i, (x, y) in enumerate(zip(a["devices"], b["devices"])):
        for k in ("device_id", "b", "gmbs", "lbs", "predicted_time"):
            if x[k] != y[k]:
                diffs.append(f"devices[{i}].{k}")
    if len(a["devices"]) != len(b["devices"]):
        diffs.append("n")
    return diffs


def plan_parity(rt, profiles, gbs, stage, world, link):
    """Re-plan each measured profile (with the link model its plan used) with the reference planner
    compiled from its own sources (oracle/_ref, the checker) and compare with the product plan bit
    for bit."""
    import oracle
    from paper_2408_12596_b200 import poplar
    if not oracle.available():
        return {"checked": 0, "note": "oracle/_ref not built"}
    ref = oracle.reference()
    out = {"checked": 0, "identical": True, "diffs": []}
    for name, prof, plan, lk in profiles:
        theirs = poplar.poplar_plan(rt, prof, plan["gbs"], stage, world, link=lk, api=ref)
        d = plans_equal(plan, theirs)
        out["checked"] += 1
        if d:
            out["identical"] = False
            out["diffs"].append({name: d})
    return out


def search_gbs(rt, profile, stage, world, link, per_gpu):
    """Poplar's planner (Alg. 2, the product planner) evaluated over candidate global batches on
    the measured profile: the batch with the best predicted samples/s, the smallest within 0.1 %
    of the best. Deterministic in its inputs, so every rank picks the same batch."""
    from paper_2408_12596_b200 import poplar
    lo, hi, step = per_gpu
    table = []
    for g in range(lo * world, hi * world + 1, step * world):
        p = poplar.poplar_plan(rt, profile, g, stage, world, link=link)
        table.append((g, g / p["predicted_wall_time"]))
    best = max(t for _, t in table)
    return min(g for g, t in table if t >= 0.999 * best), table


def reference_prediction(rt, profile, probes, link, gbs, stage, world):
    """The reference's own latent pipeline (profile_cluster -> plan -> simulate_iteration,
    compiled from its sources) on a cluster fitted to the measured curves: per rank c0/c1 by least
    squares over the profile samples, act_mem_per_batch = the measured batch-1 footprint, total_mem
    placing the latent OOM threshold at the measured mbs, optimizer_time measured, link model
    measured (CPU path 1). Returns its predicted samples/s and sync idle %."""
    import numpy as np
    import oracle
    from paper_2408_12596_b200 import poplar
    from paper_2408_12596_b200.host import ClusterSpec, Device
    if not oracle.available():
        return None
    ref = oracle.reference()
    model, _ = poplar.planner_inputs(rt, world, *(link or ()))
    resident = ref.resident_state_bytes(model, stage, world)
    devs = []
    for d, pr in zip(profile["devices"], probes):
        b = np.array([s[0] for s in d["samples"]], dtype=np.float64)
        t = np.array([s[1] for s in d["samples"]], dtype=np.float64)
        if len(b) >= 2:
            c1, c0 = np.polyfit(b, t, 1)
        else:
            c1, c0 = t[0] / b[0], 0.0
        act = max(pr[1] - pr[0], 1.0)
        devs.append(Device(resident + act * (d["mbs"] + 0.5), act, max(float(c0), 0.0), max(float(c1), 1e-9),
                           d["optimizer_time"]))
    cl = ClusterSpec(devs, [link[0] if link else poplar.NVLINK_BPS] * world,
                     link[1] if link else poplar.NCCL_ALPHA)
    t0 = time.perf_counter()
    prof = ref.profile_cluster(cl, model, stage)
    plan = ref.plan(gbs, prof, prof["effective_stage"], model, cl)
    planner_ms = 1e3 * (time.perf_counter() - t0)
    rep = ref.simulate_iteration(cl, model, plan, prof["effective_stage"])
    T = rep["iteration_time"]
    return {"samples_per_s": rep["throughput"], "iteration_time_s": T,
            "sync_idle_pct": [100.0 * i / T for i in rep["idle"]],
            "plan_b": [d["b"] for d in plan["devices"]], "gas": plan["gas"],
            "fit": [{"c0": d.compute_fixed, "c1": d.compute_per_batch} for d in devs],
            "profile_plan_simulate_ms": planner_ms}


# ---------------------------------------------------------------- our arm
def rank_micro_steps(plan, r, stage):
    d = plan["devices"][r]
    if stage >= 2:
        return plan["gas"]
    return 0 if d["gmbs"] == 0 else -(-d["gmbs"] // d["b"])


def gemm_traffic(config: str):
    """DRAM traffic of one launch of the config's largest forward GEMM from a committed
    `ncu --set full` capture (profiles/gemm_traffic.json, keyed by config); None if not captured."""
    path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f).get(config)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--gbs", type=int, default=0, help="override global batch (samples)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-recalibrate", action="store_true",
                    help="plan from the Alg. 1 profile only (no measured-iteration correction)")
    ap.add_argument("--recalibrate-passes", type=int, default=3,
                    help="measured-iteration corrections before the timed run (each re-plans)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    dist = None
    if world > 1:
        import torch.distributed as dist  # plumbing only: rendezvous, barrier, max-over-ranks
        dist.init_process_group("gloo")
    from paper_2408_12596_b200 import _lib
    from paper_2408_12596_b200.models import MODELS
    from paper_2408_12596_b200.runtime import Runtime, nccl_unique_id, RankTiming
    from paper_2408_12596_b200 import poplar

    def allgather(obj):
        if dist is None:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def barrier():
        if dist is not None:
            dist.barrier()

    nid = nccl_unique_id() if rank == 0 and world > 1 else None
    nid = allgather(nid)[0] if world > 1 else None
    model = MODELS[cfg["model"]]
    tier = cfg["tiers"][rank % len(cfg["tiers"])]
    cap_gib = cfg["caps"][rank % len(cfg["caps"])]
    stage = cfg["stage"]
    gbs = args.gbs or cfg["gbs_per_gpu"] * world
    rt = Runtime(model, rank=rank, world_size=world, device=local, nccl_id=nid, sm_budget=tier,
                 hbm_cap_bytes=int(cap_gib * (1 << 30)), seed=0, lr=1e-4)

    # Measured alpha-beta link model of the stage's collectives (reference comm.cpp:88-99). One
    # rank launches no collectives: latency 0 and infinite bandwidth make collective_time 0 in the
    # reference's own formula (validate() only requires bandwidth > 0).
    link = rt.link_model(stage) if world > 1 else (float("inf"), 0.0)
    link_measured = link

    # Poplar: Alg. 1 on the devices, Alg. 2 on the host (bit-exact planner)
    t0 = time.perf_counter()
    profile = rt.profile(stage)
    t_profile = time.perf_counter() - t0
    stage = profile["effective_stage"]
    search = cfg.get("gbs_search") if not args.gbs else None
    search_table = None
    if search:
        gbs, search_table = search_gbs(rt, profile, stage, world, link, search)
    plan = poplar.poplar_plan(rt, profile, gbs, stage, world, link=link)
    first, count = poplar.rank_slice(plan, rank)
    rt.load_tokens(first_sample=first, count=max(count, 1), iteration=0)
    plan_initial, profile_initial = plan, profile
    # W warm-up iterations first: the recalibration below then measures thermally settled GPUs
    # (a power-capped GPU's speed drifts over its first minute of load)
    for _ in range(args.warmup):
        rt.execute_iteration(plan, stage)
    if world > 1 and not args.no_recalibrate:
        # one measured iteration corrects every rank's curve for the power-capped steady state,
        # then the same planner re-plans (poplar.recalibrate)
        # (repeated: each pass measures the current plan, so the residual of the previous
        # correction is corrected too; the compute of two iterations is averaged)
        for _ in range(max(1, args.recalibrate_passes)):
            rt.execute_iteration(plan, stage)
            t_cal = [rt.execute_iteration(plan, stage) for _ in range(2)]
            all_cal = allgather([{"compute": t["compute"], "coll_times": t["coll_times"], "wall": t["wall"],
                                  "optimizer": t["optimizer"]} for t in t_cal])
            profile = poplar.recalibrate(profile, plan,
                                         [{"compute": sum(c["compute"] for c in r) / len(r)} for r in all_cal])
            # the link model likewise: fitted to the comm the iteration exposed (mean of the two)
            floors = [poplar.iteration_report([r[k] for r in all_cal], gbs)["comm_total"] for k in range(2)]
            floor = sum(floors) / 2
            if stage in (1, 2) and rt.peer_collectives():
                # the fused sync kernel's span holds the AdamW pass too; the planner adds that as its
                # optimizer tail, so it leaves the comm floor
                floor -= max(d["optimizer_time"] for d in profile["devices"])
            link = poplar.recalibrate_link(link, stage, plan["gas"], floor, rt.param_count)
            if search:
                gbs, search_table = search_gbs(rt, profile, stage, world, link, search)
            plan = poplar.poplar_plan(rt, profile, gbs, stage, world, link=link)
            first, count = poplar.rank_slice(plan, rank)
            rt.load_tokens(first_sample=first, count=max(count, 1), iteration=0)

    def timed(k, plan_d, host_tokens=None):
        from paper_2408_12596_b200.host import plan_from_py
        cplan = plan_from_py(plan_d)
        tm = RankTiming()
        barrier()
        rt.sync()
        rt.mark(0)
        for _ in range(k):
            if host_tokens is not None:
                rt.load_tokens_ptr(host_tokens[0], host_tokens[1])
            rt.execute_iteration_c(cplan, stage, tm)
        rt.mark(1)
        local_t = rt.elapsed(0, 1)
        rt.sync()
        barrier()
        return max(allgather(local_t)), tm.to_py()

    # The predicted rates of neighbouring batches differ by about the planner's prediction error,
    # so the final choice is measured: one iteration of the plan at each of the three batches with
    # the best predicted samples/s (after one untimed iteration each), max over ranks
    measured_search = None
    if search_table and world > 1:
        top = [g for g, _ in sorted(search_table, key=lambda x: -x[1])[:3]]
        measured_search = {}
        for g in top:
            p_g = poplar.poplar_plan(rt, profile, g, stage, world, link=link)
            f_g, c_g = poplar.rank_slice(p_g, rank)
            rt.load_tokens(first_sample=f_g, count=max(c_g, 1), iteration=0)
            rt.execute_iteration(p_g, stage)
            T_g, _ = timed(1, p_g)
            measured_search[g] = g / T_g
        gbs = max(measured_search, key=measured_search.get)
        plan = poplar.poplar_plan(rt, profile, gbs, stage, world, link=link)
        first, count = poplar.rank_slice(plan, rank)
        rt.load_tokens(first_sample=first, count=max(count, 1), iteration=0)

    # heterogeneity-blind baseline at the same (final) global batch, from the Alg. 1 profile
    uniform = poplar.poplar_plan(rt, profile_initial, gbs, stage, world, uniform=True, link=link)
    rt.execute_iteration(plan, stage)  # the final plan once more before the timed region
    launches0 = _lib.lib.zp_launch_count()
    with ClockSampler(local) as clk:
        T, last_timing = timed(args.steps, plan)
    launches = _lib.lib.zp_launch_count() - launches0
    clocks = clk.summary()
    value = args.steps * gbs / T
    timings = allgather(last_timing)
    report = poplar.iteration_report(timings, gbs)

    # e2e: tokens from pinned host memory every step, loss read back every step
    e2e = None
    if not args.no_e2e:
        import torch
        s1 = model.seq_len + 1
        host = torch.randint(0, model.vocab, (max(count, 1), s1), dtype=torch.int32).pin_memory()
        ke = max(1, min(args.steps, 5))  # iterations are seconds long: five end-to-end ones suffice
        T_e2e, _ = timed(ke, plan, host_tokens=(host.data_ptr(), max(count, 1)))
        rt.load_tokens(first_sample=first, count=max(count, 1), iteration=0)
        h2d = sum(allgather(count * s1 * 4))
        d2h = 4 * sum(rank_micro_steps(plan, r, stage) for r in range(world))  # per-step loss read-back
        e2e = {"value": ke * gbs / T_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": ke}

    # Heterogeneity-blind baseline (equal split) on the same devices
    rt.load_tokens(first_sample=poplar.rank_slice(uniform, rank)[0],
                   count=max(poplar.rank_slice(uniform, rank)[1], 1), iteration=0)
    ku = max(2, args.steps // 4)
    rt.execute_iteration(uniform, stage)
    T_u, _ = timed(ku, uniform)
    uniform_value = ku * gbs / T_u

    # Roofline: per-launch event timing of the dense GEMMs over one more iteration
    rt.load_tokens(first_sample=first, count=max(count, 1), iteration=0)
    rt.gemm_timing(1)
    rt.execute_iteration(plan, stage)
    gflops, gsec, glaunch = rt.gemm_timing(2)
    rt.gemm_timing(0)
    g_all = allgather((gflops, gsec, glaunch, tier))

    # HBM-bound update kernel: fused accumulate + AdamW + bf16 cast over this rank's shard, timed
    # by its CUDA events in the last timed iteration. Bytes per element: p32/m/v read+write (24),
    # bf16 param write (2), gradient read (bf16 2 at Z2/3 + fp32 accumulator 4 when gas > 1; fp32 4
    # at Z0/1). At Z1/Z2 over NVLink the update is inside the fused sync kernel (timed as `sync`).
    shard = rt.padded_params if stage == 0 else rt.padded_params // world
    steps_r = rank_micro_steps(plan, rank, stage)
    fused = world > 1 and stage in (1, 2) and rt.peer_collectives()
    if fused:
        # fused RS + AdamW + AG: local HBM bytes = Adam state r/w (24) + p16 own write (2) + own
        # grad share read (2 bf16 / 4 fp32) + fp32 accumulator (Z2, gas > 1); NVLink bytes = the
        # peers' gradient shards pulled + the new bf16 shard pushed to every peer
        gb = 4 if stage == 1 else 2
        adam_bytes = shard * (26 + gb + (4 if stage == 2 and steps_r > 1 else 0))
        nvl_bytes = shard * (world - 1) * (gb + 2)
        adam_s = last_timing["sync"]
    else:
        # gradient read: the fp32 accumulator only when it holds every micro-step (ZeRO-0/1, one
        # rank, or ZeRO-3 over NVLink); else the last micro-step's bf16 shard (+ the accumulator)
        in_acc = stage <= 1 or world == 1 or (stage == 3 and rt.peer_collectives())
        gbytes = 4 if in_acc else (2 + (4 if steps_r > 1 else 0))
        adam_bytes = shard * (26 + gbytes)
        nvl_bytes = 0
        adam_s = last_timing["optimizer"]
    adam_all = allgather((adam_bytes, adam_s, nvl_bytes))

    # Memory probes of every rank (for the fitted reference cluster)
    probe = rt.memory_probe(stage)
    probes = allgather(probe)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sps, cores, dt, desc = cpu_step_sample(cfg["model"])
        cpu = {"value": sps, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": desc + "; the reference has no tensor step",
               "reference_planner_ms": reference_planner_ms()}

    if rank == 0:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
        fl, sec, nl, tr = g_all[0]
        achieved = fl / sec / 1e12 if sec > 0 else 0.0
        # Denominator: the burst bf16 figure (conservative: the GEMMs of the larger models run
        # above the 4-second sustained figure inside the step); the sustained fraction is
        # reported beside it
        peak = peaks["bf16_tflops"] * tr / 148.0
        peak_sust = peaks["bf16_tflops_sustained"] * tr / 148.0
        traffic = gemm_traffic(args.config)
        # checks against the reference (the oracle as checker; not timed, not on the product path)
        parity = plan_parity(rt, [("alg1", profile_initial, plan_initial, link_measured)] +
                             ([("recalibrated", profile, plan, link)] if plan is not plan_initial else []),
                             gbs, stage, world, link)
        measured_iter = T / args.steps
        # where the prediction and the measurement differ: the planner's wall time is
        # T(compute) + gas * comm_per_step + sync + optimizer tail (planner.cpp:335-359); measured
        # are the slowest rank's compute, the per-collective comm floor, the optimizer and the rest
        # of the iteration (accumulation passes, launch gaps: work the cost model has no term for)
        api_model, api_cluster = poplar.planner_inputs(rt, world, *(link or ()))
        from paper_2408_12596_b200 import host as _host
        cp = _host.product().make_comm_profile(api_model, stage, api_cluster)
        t_last = report["iteration_time"]
        m_comp = max(report["compute"])
        m_opt = max(t["optimizer"] for t in timings)
        fidelity = {"predicted_wall_time_s": plan["predicted_wall_time"], "measured_iteration_s": measured_iter,
                    "rel_err": (plan["predicted_wall_time"] - measured_iter) / measured_iter,
                    "gate": "reference acceptance criterion 8: |rel_err| <= 0.02 (acceptance.cpp:433-447)",
                    "predicted": {"compute_s": plan["iteration_time"],
                                  "comm_s": (plan["gas"] * cp.time_per_step if stage >= 2 else 0.0) + cp.sync_time,
                                  "optimizer_s": max(d["optimizer_time"] for d in profile["devices"])},
                    "measured_last_iteration": {"compute_s": m_comp, "comm_floor_s": report["comm_total"],
                                                "optimizer_s": m_opt,
                                                "unmodelled_s": t_last - m_comp - report["comm_total"] - m_opt},
                    "per_rank_compute_s": {"predicted": [d["predicted_time"] for d in plan["devices"]],
                                           "measured": report["compute"]},
                    "per_rank_collectives_s": {"gather": [t["ag_fwd"] + t["ag_bwd"] for t in timings],
                                               "reduce_scatter": [t["rs"] for t in timings],
                                               "sync": [t["sync"] for t in timings],
                                               "wall": [t["wall"] for t in timings]}}
        try:
            ref_pred = reference_prediction(rt, profile, probes, link, gbs, stage, world)
        except Exception as e:  # the reference pipeline may reject a fitted cluster
            ref_pred = {"error": str(e)}
        # the fused sync kernel's span on a fast rank includes its wait for the slowest one at the
        # entry barrier: the roofline uses the rank whose span is shortest (the last to arrive)
        a_bytes, a_s, a_nvl = min(adam_all, key=lambda x: x[1] if x[1] else float("inf")) if fused else adam_all[0]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg["label"], "model": cfg["model"], "params": rt.param_count,
                       "seq_len": model.seq_len, "head_dim": model.head_dim, "global_batch": gbs,
                       "gbs_search": ({"per_gpu_range": list(search), "chosen": gbs,
                                       "predicted_samples_per_s": {str(g): t for g, t in search_table},
                                       "measured_top3_samples_per_s": ({str(g): v for g, v in measured_search.items()}
                                                                       if measured_search else None)}
                                      if search_table else None),
                       "stage": stage,
                       "sm_budgets": [cfg["tiers"][r % len(cfg["tiers"])] for r in range(world)],
                       "hbm_caps_gib": [cfg["caps"][r % len(cfg["caps"])] or "full" for r in range(world)],
                       "plan": {"b": [d["b"] for d in plan["devices"]], "lbs": [d["lbs"] for d in plan["devices"]],
                                "gmbs": [d["gmbs"] for d in plan["devices"]], "gas": plan["gas"]},
                       "plan_alg1_only": {"b": [d["b"] for d in plan_initial["devices"]],
                                          "gmbs": [d["gmbs"] for d in plan_initial["devices"]],
                                          "gas": plan_initial["gas"]},
                       "recalibrated": plan is not plan_initial,
                       "recalibrate_passes": 0 if plan is plan_initial else max(1, args.recalibrate_passes),
                       "mbs": [d["mbs"] for d in profile["devices"]],
                       "link_model": ({"bandwidth_GBps": link_measured[0] / 1e9, "latency_us": link_measured[1] * 1e6,
                                       "source": "measured (zp_runtime_link_model, max over ranks)",
                                       "recalibrated_bandwidth_GBps": (link[0] / 1e9 if link is not link_measured
                                                                       else None),
                                       "recalibrated_note": "bandwidth solved from the measured exposed comm "
                                                            "(poplar.recalibrate_link); used by the final plan"}
                                      if world > 1 else "one rank: no collectives (latency 0, bandwidth inf)"),
                       "profile_seconds": t_profile, "parallelism": f"zero{stage}-dp{world}",
                       "collectives": (("nvlink-peer (pull RS/AG; fused RS+AdamW+AG at sync)" if stage in (1, 2) else "nvlink-peer (pull RS, copy-engine AG prefetch)" if stage == 3 else "nccl (all-reduce)") if rt.peer_collectives() else "nccl") if world > 1 else "none",
                       "l2": "inputs larger than L2 (per-step activations are tens of GB)"},
            "sync_idle_pct": report["sync_idle_pct"],
            "planner_idle_pct": [100.0 * i / plan["predicted_wall_time"] for i in plan["idle"]],
            "comm_floor_s": report["comm_total"],
            "plan_parity": parity,
            "plan_fidelity": fidelity,
            "reference_prediction": ref_pred,
            "uniform_split": {"value": uniform_value, "poplar_speedup": value / uniform_value,
                              "plan_b": [d["b"] for d in uniform["devices"]], "gas": uniform["gas"]},
            "roofline": {"kernel": "tcgen05 GEMM (dense linear layers, rank 0)", "bound": "tensor",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None,
                         "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                         "traffic_note": (traffic["note"] + f" Shape {traffic['shape']}.") if traffic else
                         "no ncu capture committed for this config",
                         "frac_vs_sustained": achieved / peak_sust if peak_sust else None,
                         "peak_note": f"MEASURED_PEAKS bf16_tflops (burst) {peaks['bf16_tflops']} x {tr}/148 SM budget; "
                                      f"sustained {peaks['bf16_tflops_sustained']} x {tr}/148 for frac_vs_sustained",
                         "launches": nl},
            "roofline_hbm": {"kernel": ("peer_rs_adam_ag_k (fused NVLink RS + AdamW + push AG), last-arriving rank" if fused else
                                        "adam_k (fused accumulate + AdamW + bf16 cast), rank 0"),
                             "bound": "nvlink" if fused else "hbm",
                             "nvlink": ({"achieved_GBps": a_nvl / a_s / 1e9, "peak_GBps": 770.0,
                                         "frac": a_nvl / a_s / 1e9 / 770.0,
                                         "peak_note": "measured peer copy per direction per GPU on this pool "
                                                      "(B200_PROFILING.md; 900 nominal); bytes = the peers' "
                                                      "gradient shards pulled + the new bf16 shard pushed"}
                                        if (fused and a_s) else None),
                             "achieved": a_bytes / a_s / 1e9 if a_s else None,
                             "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": (a_bytes / a_s / 1e9 / peaks["hbm_gbs"]) if a_s else None,
                             "bytes_per_launch": a_bytes,
                             "nvlink_GBps": (a_nvl / a_s / 1e9) if (a_s and a_nvl) else None},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    rt.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
