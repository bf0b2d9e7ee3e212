"""GPU step parity: the B200 GPT fwd/bwd + ZeRO reduce/update against the float64 oracle
(oracle/step.py, itself pinned to torch autograd by tests/test_oracle_step.py).

Tolerances (BASELINE.json north star): gradients and parameters within rel 2e-2 on the bf16
path (norm-wise per tensor); the AdamW update kernel within rel 1e-5 (fp32 path) given the
same gradient.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TINY = dict(n_layer=2, d_model=256, n_head=4, vocab=1000, seq_len=128, d_ff=1024)


def make_plan(stage, gbs, b, lbs, gas, n=1, per_rank=None):
    devs = per_rank or [dict(device_id=0, b=b, gmbs=(gas - 1) * b + lbs, lbs=lbs, predicted_time=0.0)]
    n = len(devs)
    return dict(stage=stage, gbs=gbs, gas=gas, devices=devs, iteration_time=0.0, idle=[0.0] * n,
                under_utilization=[0.0] * n, objective=0.0, weights=[1.0] * n, predicted_wall_time=0.0)


def runtime(cuda, seed=3, **kw):
    from paper_2408_12596_b200.runtime import Runtime, GPT
    rt = Runtime(GPT(**TINY), seed=seed, lr=1e-3, **kw)
    rt.keep_grads(True)
    return rt


def oracle_grads(rt, P16flat, tokens, B):
    from oracle import step as so
    P = {k: v.astype(np.float64) for k, v in rt.unflatten(P16flat).items()}
    return so.gpt_loss_and_grads(P, tokens, TINY["n_layer"], TINY["n_head"], TINY["vocab"], B)


def tokens_for(B, seed=0):
    rng = np.random.default_rng(seed)
    return rng.integers(0, TINY["vocab"], (B, TINY["seq_len"] + 1)).astype(np.int32)


@pytest.mark.parametrize("stage,b,lbs,gas", [(0, 4, 4, 1), (0, 3, 1, 2), (1, 2, 2, 2), (2, 4, 4, 1),
                                             (2, 3, 1, 2), (3, 4, 4, 1), (3, 2, 1, 3)])
def test_step_matches_fp64_oracle(cuda, stage, b, lbs, gas):
    from paper_2408_12596_b200.runtime import bf16_to_f32
    from oracle import step as so
    B = (gas - 1) * b + lbs
    rt = runtime(cuda)
    rt.resident_bytes(stage)  # configure the stage (initialises parameters)
    P16 = bf16_to_f32(rt.params_bf16())
    master0, _ = rt.state_flat(0)
    tok = tokens_for(B)
    rt.load_tokens(tok)
    t = rt.execute_iteration(make_plan(stage, B, b, lbs, gas), stage)
    loss, G = oracle_grads(rt, P16, tok, B)
    assert abs(t["loss_sum"] - loss) <= 1e-2 * abs(loss)
    g, _ = rt.state_flat(3)
    Gg = rt.unflatten(g)
    worst = max((so.rel_err(Gg[k], G[k]), k) for k in G if np.linalg.norm(G[k]) > 0)
    assert worst[0] < 2e-2, worst
    # AdamW update kernel (fp32 path): same gradient in, rel 1e-5 out.
    master1, _ = rt.state_flat(0)
    ref, _, _ = so.adamw(master0.astype(np.float64), 0.0, 0.0, g.astype(np.float64), 1, 1e-3, 0.9, 0.95, 1e-8, 0.0)
    assert so.rel_err(master1, ref) < 1e-5
    # parameters against the oracle's own gradient (bf16 path)
    ref2, _, _ = so.adamw(master0.astype(np.float64), 0.0, 0.0, _flat_like(rt, G, master0.size), 1, 1e-3,
                          0.9, 0.95, 1e-8, 0.0)
    assert so.rel_err(master1, ref2) < 2e-2
    rt.close()


def _flat_like(rt, G, n):
    flat = np.zeros(n, dtype=np.float64)
    for k, v in G.items():
        o, r, c = rt.tensor_info(k)
        flat[o:o + r * c] = v.ravel()
    return flat


def test_plans_are_equivalent(cuda):
    """Heterogeneous split invariance on one GPU: (b=8) == (b=3,3,2) == (Z2, b=5, lbs=3)."""
    from oracle import step as so
    B = 8
    tok = tokens_for(B, seed=5)
    grads = []
    for stage, b, lbs, gas in ((0, 8, 8, 1), (0, 3, 2, 3), (2, 5, 3, 2), (3, 3, 2, 3)):
        rt = runtime(cuda, seed=9)
        rt.resident_bytes(stage)
        rt.load_tokens(tok)
        rt.execute_iteration(make_plan(stage, B, b, lbs, gas), stage)
        grads.append(rt.state_flat(3)[0])
        rt.close()
    for g in grads[1:]:
        assert so.rel_err(g, grads[0]) < 1e-2


def test_memory_probe_and_oom(cuda):
    from paper_2408_12596_b200.runtime import Runtime, GPT
    rt = Runtime(GPT(**TINY), seed=1, hbm_cap_bytes=2 << 30)
    probe = rt.memory_probe(0)
    assert probe is not None
    before, after, total = probe
    assert total == 2 << 30
    act1 = rt.activation_bytes(1)
    assert after - before == pytest.approx(act1, rel=0.01)
    mbs = int((total - before) // (after - before))
    assert rt.run_step(mbs, 0, mbs) is not None
    assert rt.run_step(mbs + 2, 0, mbs + 2) is None  # OOM signalled, not raised
    rt.close()


def test_run_step_trace(cuda):
    rt = runtime(cuda)
    t = rt.run_step(4, 2, 4)
    assert t["forward_compute"] > 0 and t["backward_compute"] > 0 and t["optimizer_step"] > 0
    assert t["fwd_allgather"] == 0.0
    rt.close()


@pytest.mark.parametrize("layers,sm", [(1, 0), (2, 132), (12, 66)])
def test_step_gpt2_small_shapes(cuda, layers, sm):
    """GPT-2-small layer shapes (h=768, 12 heads, V=50257 padded to 50304, s=1024), SM budgets."""
    from paper_2408_12596_b200.runtime import Runtime, GPT, bf16_to_f32
    from oracle import step as so
    cfg = GPT(n_layer=layers, d_model=768, n_head=12, vocab=50257, seq_len=1024)
    rt = Runtime(cfg, seed=4, lr=1e-3, sm_budget=sm)
    rt.keep_grads(True)
    rt.resident_bytes(0)
    P = {k: v.astype(np.float64) for k, v in rt.unflatten(bf16_to_f32(rt.params_bf16())).items()}
    tok = np.random.default_rng(2).integers(0, cfg.vocab, (2, cfg.seq_len + 1)).astype(np.int32)
    rt.load_tokens(tok)
    t = rt.execute_iteration(make_plan(0, 2, 2, 2, 1), 0)
    loss, G = so.gpt_loss_and_grads(P, tok, layers, 12, cfg.vocab, 2)
    assert abs(t["loss_sum"] - loss) <= 1e-2 * abs(loss), (t["loss_sum"], loss)
    g = rt.unflatten(rt.get_state(3)[2])
    worst = max((so.rel_err(g[k], G[k]), k) for k in G if np.linalg.norm(G[k]) > 0)
    assert worst[0] < 2e-2, worst
    rt.close()


LLAMA = dict(n_layer=2, d_model=256, n_head=4, vocab=1000, seq_len=128, d_ff=512, arch=1)


@pytest.mark.parametrize("stage,b,lbs,gas,sm,heads", [(0, 3, 3, 1, 0, 4), (2, 2, 1, 2, 0, 4), (3, 3, 2, 2, 74, 4),
                                                       (3, 2, 2, 1, 0, 2), (2, 3, 1, 2, 104, 2)])
def test_llama_step_matches_fp64_oracle(cuda, stage, b, lbs, gas, sm, heads):
    """Llama family (RMSNorm, RoPE, SwiGLU, untied head) against oracle/step.py; heads 4 = head_dim
    64, heads 2 = head_dim 128 (the Llama-1.3B / 7B layout)."""
    from paper_2408_12596_b200.runtime import Runtime, GPT, bf16_to_f32
    from oracle import step as so
    B = (gas - 1) * b + lbs
    cfg = dict(LLAMA, n_head=heads)
    rt = Runtime(GPT(**cfg), seed=6, lr=1e-3, sm_budget=sm)
    rt.keep_grads(True)
    rt.resident_bytes(stage)
    P = {k: v.astype(np.float64) for k, v in rt.unflatten(bf16_to_f32(rt.params_bf16())).items()}
    tok = np.random.default_rng(8).integers(0, LLAMA["vocab"], (B, LLAMA["seq_len"] + 1)).astype(np.int32)
    rt.load_tokens(tok)
    t = rt.execute_iteration(make_plan(stage, B, b, lbs, gas), stage)
    loss, G = so.llama_loss_and_grads(P, tok, LLAMA["n_layer"], heads, LLAMA["vocab"], B)
    assert abs(t["loss_sum"] - loss) <= 1e-2 * abs(loss), (t["loss_sum"], loss)
    g = rt.unflatten(rt.state_flat(3)[0])
    worst = max((so.rel_err(g[k], G[k]), k) for k in G if np.linalg.norm(G[k]) > 0)
    assert worst[0] < 2e-2, worst
    rt.close()


@pytest.mark.parametrize("budget,expect", [(66, 64), (74, 72), (132, 128), (0, 148)])
def test_green_context_confinement(cuda, budget, expect):
    """An SM budget below the device's SM count becomes a green-context partition (a multiple of 8
    SMs, rounded down) that every kernel of the rank runs in; the step still matches the oracle."""
    import os
    if os.environ.get("ZP_GREEN", "1") == "0":
        pytest.skip("green contexts disabled")
    rt = runtime(cuda, sm_budget=budget)
    sms, green = rt.sm_info()
    assert sms == expect and green == (budget != 0)
    rt.resident_bytes(2)
    from paper_2408_12596_b200.runtime import bf16_to_f32
    from oracle import step as so
    P16 = bf16_to_f32(rt.params_bf16())
    tok = tokens_for(4)
    rt.load_tokens(tok)
    rt.execute_iteration(make_plan(2, 4, 4, 4, 1), 2)
    loss, G = oracle_grads(rt, P16, tok, 4)
    g, _ = rt.state_flat(3)
    Gg = rt.unflatten(g)
    assert max(so.rel_err(Gg[k], G[k]) for k in G if np.linalg.norm(G[k]) > 0) < 2e-2
    rt.close()
