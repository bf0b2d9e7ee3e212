"""ORACLE / TEST INFRASTRUCTURE — the checker, never the product.

* `reference()` loads oracle/_ref/libzpref.so: the reference's own zeroplan sources
  (/root/reference/proj/core/src, compiled in place by oracle/Makefile) behind the
  zp_host.h C ABI with prefix `zpref_`.
* `_ref/seam_b200` is the reference's own profiler / planner / simulator linked with the
  device-seam binding (integration/hardware_b200.cpp): the reference pipeline driving B200 ranks
  through its unchanged run_step / memory_probe signatures (tests/test_seam.py).
* `step.py` is the numpy fp64 oracle of the GPT training step (the reference has no
  tensors, so gradient/parameter parity is pinned by this restatement).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libzpref.so")
REF_SRC = "/root/reference/proj"


def build_reference(quiet: bool = True) -> bool:
    """Compile the reference sources into oracle/_ref (only where /root/reference exists)."""
    if not os.path.isdir(REF_SRC):
        return os.path.exists(REF_LIB)
    r = subprocess.run(["make", "-C", HERE], capture_output=quiet, text=True)
    return r.returncode == 0 and os.path.exists(REF_LIB)


def available() -> bool:
    return os.path.exists(REF_LIB)


_ref = None


def reference():
    global _ref
    if _ref is None:
        from paper_2408_12596_b200.host import HostAPI, Cluster, Model
        lib = C.CDLL(REF_LIB)
        _ref = HostAPI(lib, "zpref_")
        f = lib.zpref_fuzz_instance
        f.argtypes = [C.c_uint64, C.POINTER(Cluster), C.POINTER(Model), C.POINTER(C.c_int64),
                      C.POINTER(C.c_int32)]
        f.restype = C.c_int
        _ref.fuzz_fn = f
    return _ref


def fuzz_instance(index: int):
    """Acceptance-suite fuzz instance `index` (proj/tests/acceptance.cpp:72-110)."""
    from paper_2408_12596_b200.host import Cluster, Model, ClusterSpec, Device, ModelSpec
    ref = reference()
    c, m = Cluster(), Model()
    gbs, st = C.c_int64(), C.c_int32()
    ref.fuzz_fn(index, C.byref(c), C.byref(m), C.byref(gbs), C.byref(st))
    cluster = ClusterSpec(devices=[Device(c.devices[i].total_mem, c.devices[i].act_mem_per_batch,
                                          c.devices[i].compute_fixed, c.devices[i].compute_per_batch,
                                          c.devices[i].optimizer_time) for i in range(c.n)],
                          link_bandwidths=[c.link_bandwidths[i] for i in range(c.n)],
                          link_latency=c.link_latency, seed=c.seed, jitter=c.jitter)
    model = ModelSpec(m.param_count, m.hidden_size, m.num_layers, m.bytes_per_param,
                      m.optimizer_state_multiplier)
    return cluster, model, gbs.value, (None if st.value < 0 else st.value)
