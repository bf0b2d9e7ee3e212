"""Python handle on the B200 device back end (include/zp_runtime.h).

`Runtime` wraps one rank's zp_runtime: GPT-2-family model state in a capped HBM arena,
real ZeRO-0/1/2 micro-steps on the sm_100a kernels, NCCL collectives across ranks.
The profiler / planner / executor on top of it live in `poplar.py`.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .models import GPT, MODELS  # noqa: F401  (re-exported)
from .host import (Plan, Probe, Profile, StepTrace, plan_from_py, profile_to_py, ZeroplanError, _ERR, OK, OOM)

lib = _lib.lib


class GptConfig(C.Structure):
    _fields_ = [("n_layer", C.c_int32), ("d_model", C.c_int32), ("n_head", C.c_int32), ("d_ff", C.c_int32),
                ("vocab", C.c_int32), ("seq_len", C.c_int32), ("arch", C.c_int32)]


class RuntimeDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world_size", C.c_int32), ("device", C.c_int32),
                ("nccl_id", C.c_uint8 * 128), ("sm_budget", C.c_int32), ("hbm_cap_bytes", C.c_int64),
                ("model", GptConfig), ("seed", C.c_uint64), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float)]


class RankTiming(C.Structure):
    """zp_rank_timing (include/zp_runtime.h). The per-collective durations go to a caller-owned
    buffer; `n_collectives` always counts every collective, and `to_py` refuses a truncated list
    (the idle metric would silently undercount busy time)."""
    _fields_ = [("compute", C.c_double), ("forward", C.c_double), ("backward", C.c_double),
                ("comm", C.c_double), ("optimizer", C.c_double), ("wall", C.c_double),
                ("loss_sum", C.c_double), ("micro_steps", C.c_int64), ("n_collectives", C.c_int32),
                ("coll_capacity", C.c_int32), ("coll_times", C.POINTER(C.c_double)),
                ("coll_truncated", C.c_int32), ("pad_", C.c_int32),
                ("ag_fwd", C.c_double), ("ag_bwd", C.c_double), ("rs", C.c_double), ("sync", C.c_double)]

    def __init__(self, capacity: int = 1 << 16):
        super().__init__()
        self._buf = (C.c_double * capacity)()
        self.coll_times = C.cast(self._buf, C.POINTER(C.c_double))
        self.coll_capacity = capacity

    def to_py(self) -> dict:
        if self.coll_truncated or self.n_collectives > self.coll_capacity:
            raise ZeroplanError(f"{self.n_collectives} collectives exceed the timing buffer "
                                f"({self.coll_capacity}); pass a larger RankTiming(capacity)")
        return {"compute": self.compute, "forward": self.forward, "backward": self.backward,
                "comm": self.comm, "optimizer": self.optimizer, "wall": self.wall,
                "loss_sum": self.loss_sum, "micro_steps": self.micro_steps,
                "ag_fwd": self.ag_fwd, "ag_bwd": self.ag_bwd, "rs": self.rs, "sync": self.sync,
                "coll_times": list(self._buf[:self.n_collectives])}


_P = C.c_void_p
_SIGS = {
    "zp_runtime_last_error": ([], C.c_char_p),
    "zp_nccl_unique_id": ([C.POINTER(C.c_uint8)], C.c_int),
    "zp_runtime_create": ([C.POINTER(RuntimeDesc), C.POINTER(_P)], C.c_int),
    "zp_runtime_destroy": ([_P], C.c_int),
    "zp_runtime_param_count": ([_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "zp_runtime_activation_bytes": ([_P, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "zp_runtime_resident_bytes": ([_P, C.c_int32, C.POINTER(C.c_int64)], C.c_int),
    "zp_runtime_memory_probe": ([_P, C.c_int32, C.POINTER(Probe)], C.c_int),
    "zp_runtime_load_tokens": ([_P, _P, C.c_int64, C.c_int64, C.c_uint64, C.c_int32], C.c_int),
    "zp_runtime_run_step": ([_P, C.c_int64, C.c_int32, C.c_int64, C.POINTER(StepTrace)], C.c_int),
    "zp_runtime_execute_iteration": ([_P, C.POINTER(Plan), C.c_int32, C.POINTER(RankTiming)], C.c_int),
    "zp_runtime_get_state": ([_P, C.c_int32, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "zp_runtime_get_params_bf16": ([_P, _P], C.c_int),
    "zp_runtime_set_params": ([_P, _P], C.c_int),
    "zp_runtime_keep_grads": ([_P, C.c_int32], C.c_int),
    "zp_runtime_sm_info": ([_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
    "zp_runtime_peer_collectives": ([_P, C.POINTER(C.c_int32)], C.c_int),
    "zp_runtime_bench_collective": ([_P, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)],
                                    C.c_int),
    "zp_runtime_link_model": ([_P, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "zp_runtime_owned_ranges": ([_P, C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32)], C.c_int),
    "zp_runtime_tensor_info": ([_P, C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64)], C.c_int),
    "zp_runtime_sync": ([_P], C.c_int),
    "zp_runtime_profile": ([_P, C.c_int32, C.POINTER(Profile)], C.c_int),
    "zp_runtime_mark": ([_P, C.c_int32], C.c_int),
    "zp_runtime_elapsed": ([_P, C.c_int32, C.c_int32, C.POINTER(C.c_double)], C.c_int),
    "zp_runtime_gemm_stats": ([_P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.POINTER(C.c_int64)], C.c_int),
}
for _n, (_a, _r) in _SIGS.items():
    _f = getattr(lib, _n)
    _f.argtypes = _a
    _f.restype = _r


def _check(rc, allow_oom=False):
    if rc == OK:
        return True
    if rc == OOM and allow_oom:
        return False
    msg = lib.zp_runtime_last_error().decode()
    raise _ERR.get(rc, ZeroplanError)(msg or f"zp runtime error {rc}")


def gpt_config_c(m: GPT) -> GptConfig:
    return GptConfig(m.n_layer, m.d_model, m.n_head, m.d_ff, m.vocab, m.seq_len, m.arch)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib.zp_nccl_unique_id(buf))
    return bytes(buf)


class Runtime:
    def __init__(self, model: GPT, rank=0, world_size=1, device=0, nccl_id: Optional[bytes] = None,
                 sm_budget=0, hbm_cap_bytes=0, seed=0, lr=1e-4, betas=(0.9, 0.95), eps=1e-8,
                 weight_decay=0.0):
        self.model = model
        self.rank, self.world_size = rank, world_size
        d = RuntimeDesc()
        d.rank, d.world_size, d.device = rank, world_size, device
        if nccl_id is not None:
            for i, b in enumerate(nccl_id):
                d.nccl_id[i] = b
        d.sm_budget, d.hbm_cap_bytes = sm_budget, int(hbm_cap_bytes)
        d.model = gpt_config_c(model)
        d.seed = seed
        d.lr, d.beta1, d.beta2, d.eps, d.weight_decay = lr, betas[0], betas[1], eps, weight_decay
        self.desc = d
        h = _P()
        _check(lib.zp_runtime_create(C.byref(d), C.byref(h)))
        self.h = h
        pad, logical = C.c_int64(), C.c_int64()
        _check(lib.zp_runtime_param_count(self.h, C.byref(pad), C.byref(logical)))
        self.padded_params, self.param_count = pad.value, logical.value

    def close(self):
        if self.h:
            lib.zp_runtime_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- memory model
    def activation_bytes(self, batch: int) -> int:
        out = C.c_int64()
        _check(lib.zp_runtime_activation_bytes(self.h, batch, C.byref(out)))
        return out.value

    def resident_bytes(self, stage: int) -> int:
        out = C.c_int64()
        _check(lib.zp_runtime_resident_bytes(self.h, stage, C.byref(out)))
        return out.value

    def memory_probe(self, stage: int):
        p = Probe()
        ok = _check(lib.zp_runtime_memory_probe(self.h, stage, C.byref(p)), allow_oom=True)
        return (p.before_forward, p.after_forward, p.total) if ok else None

    # ---- data
    def load_tokens(self, tokens: Optional[np.ndarray] = None, first_sample=0, count=0, iteration=0):
        if tokens is not None:
            tokens = np.ascontiguousarray(tokens, dtype=np.int32)
            assert tokens.shape[1] == self.model.seq_len + 1
            _check(lib.zp_runtime_load_tokens(self.h, tokens.ctypes.data, first_sample, tokens.shape[0],
                                              iteration, 1))
        else:
            _check(lib.zp_runtime_load_tokens(self.h, None, first_sample, count, iteration, 0))

    def load_tokens_ptr(self, host_ptr: int, count: int):
        _check(lib.zp_runtime_load_tokens(self.h, host_ptr, 0, count, 0, 1))

    # ---- steps
    def run_step(self, batch: int, stage: int, global_batch: int = 0) -> Optional[dict]:
        t = StepTrace()
        ok = _check(lib.zp_runtime_run_step(self.h, batch, stage, global_batch, C.byref(t)), allow_oom=True)
        return {k: getattr(t, k) for k, _ in StepTrace._fields_} if ok else None

    def execute_iteration(self, plan: dict, stage: int) -> dict:
        t = RankTiming()
        _check(lib.zp_runtime_execute_iteration(self.h, C.byref(plan_from_py(plan)), stage, C.byref(t)))
        return t.to_py()

    def execute_iteration_c(self, cplan: Plan, stage: int, timing: RankTiming):
        _check(lib.zp_runtime_execute_iteration(self.h, C.byref(cplan), stage, C.byref(timing)))

    # ---- state
    def keep_grads(self, on=True):
        _check(lib.zp_runtime_keep_grads(self.h, 1 if on else 0))

    def sm_info(self):
        """(SMs the rank's kernels may use, True when a green context confines them)."""
        n, g = C.c_int32(), C.c_int32()
        _check(lib.zp_runtime_sm_info(self.h, C.byref(n), C.byref(g)))
        return n.value, bool(g.value)

    def peer_collectives(self) -> bool:
        """True when the ZeRO-1/2 collectives run over NVLink peer memory (peer.cu)."""
        on = C.c_int32(0)
        _check(lib.zp_runtime_peer_collectives(self.h, C.byref(on)))
        return bool(on.value)

    def bench_collective(self, which: int, reps: int = 10):
        """NVLink microbenchmark (all ranks call it together): which 0 pull reduce-scatter,
        1 pull all-gather, 2 copy-engine pulls. Returns (seconds per call, bytes pulled per call)."""
        sec, pulled = C.c_double(), C.c_int64()
        _check(lib.zp_runtime_bench_collective(self.h, which, reps, C.byref(sec), C.byref(pulled)))
        return sec.value, pulled.value

    def link_model(self, stage: int, reps: int = 10):
        """Measured (bandwidth B/s, latency s) of the stage's reduce-scatter path, collective over
        ranks (zp_runtime_link_model): the alpha-beta inputs of the planner's collective_time."""
        bw, lat = C.c_double(), C.c_double()
        _check(lib.zp_runtime_link_model(self.h, stage, reps, C.byref(bw), C.byref(lat)))
        return bw.value, lat.value

    def get_state(self, kind: int):
        """kind 0 master, 1 m, 2 v, 3 summed grad. Returns (begin, end, float32 array)."""
        out = np.zeros(self.padded_params, dtype=np.float32)
        b, e = C.c_int64(), C.c_int64()
        _check(lib.zp_runtime_get_state(self.h, kind, out.ctypes.data, C.byref(b), C.byref(e)))
        return b.value, e.value, out[: e.value - b.value].copy()

    def owned_ranges(self):
        """[(flat_begin, flat_end, shard_begin)] of the state this rank holds."""
        buf = (C.c_int64 * (3 * 1024))()
        cnt = C.c_int32()
        _check(lib.zp_runtime_owned_ranges(self.h, buf, 1024, C.byref(cnt)))
        return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(cnt.value)]

    def state_flat(self, kind: int):
        """State `kind` scattered into the flat layout: (values, mask of owned elements)."""
        _, _, shard = self.get_state(kind)
        flat = np.zeros(self.padded_params, dtype=np.float32)
        mask = np.zeros(self.padded_params, dtype=bool)
        for fb, fe, sb in self.owned_ranges():
            flat[fb:fe] = shard[sb:sb + (fe - fb)]
            mask[fb:fe] = True
        return flat, mask

    def params_bf16(self) -> np.ndarray:
        out = np.zeros(self.padded_params, dtype=np.uint16)
        _check(lib.zp_runtime_get_params_bf16(self.h, out.ctypes.data))
        return out

    def set_params(self, full: np.ndarray):
        full = np.ascontiguousarray(full, dtype=np.float32)
        assert full.size == self.padded_params
        _check(lib.zp_runtime_set_params(self.h, full.ctypes.data))

    def tensor_info(self, name: str):
        o, r, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.zp_runtime_tensor_info(self.h, name.encode(), C.byref(o), C.byref(r), C.byref(c)))
        return o.value, r.value, c.value

    def tensor_names(self):
        if self.model.arch == 1:
            names = ["wte"]
            for i in range(self.model.n_layer):
                names += [f"h{i}.{n}" for n in ("ln1_g", "w_qkv", "w_o", "ln2_g", "w_gu", "w_down")]
            return names + ["lnf_g", "lm_head"]
        names = ["wte", "wpe"]
        for i in range(self.model.n_layer):
            names += [f"h{i}.{n}" for n in ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b",
                                             "w_fc", "b_fc", "w_proj", "b_proj")]
        return names + ["lnf_g", "lnf_b"]

    def unflatten(self, flat: np.ndarray, begin: int = 0) -> dict:
        """Slices a flat-layout array (starting at flat index `begin`) into named tensors."""
        out = {}
        for n in self.tensor_names():
            o, r, c = self.tensor_info(n)
            o -= begin
            if o < 0 or o + r * c > flat.size:
                continue
            out[n] = flat[o:o + r * c].reshape(r, c)
        return out

    def sync(self):
        _check(lib.zp_runtime_sync(self.h))

    # ---- Poplar Alg. 1 on the devices (collective)
    def profile(self, stage_request: Optional[int] = None) -> dict:
        p = Profile()
        _check(lib.zp_runtime_profile(self.h, -1 if stage_request is None else stage_request, C.byref(p)))
        return profile_to_py(p)

    # ---- device timing
    def mark(self, slot: int):
        _check(lib.zp_runtime_mark(self.h, slot))

    def elapsed(self, a: int, b: int) -> float:
        out = C.c_double()
        _check(lib.zp_runtime_elapsed(self.h, a, b, C.byref(out)))
        return out.value

    def gemm_timing(self, mode: int):
        """1 = enable/reset, 0 = disable, 2 = collect -> (flops, seconds, launches)."""
        f, t, n = C.c_double(), C.c_double(), C.c_int64()
        _check(lib.zp_runtime_gemm_stats(self.h, mode, C.byref(f), C.byref(t), C.byref(n)))
        return f.value, t.value, n.value


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)
