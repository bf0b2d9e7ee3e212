"""Single-GPU parity of the NVLink peer-memory collectives (csrc/cuda/peer.cu) through the C ABI
(zp_kernels.h peer group): n "rank arenas" are n equal regions of one device allocation, and every
call runs all n rank instances in ONE cooperative launch, so instances that wait on one another
through the flag barriers are co-resident by construction (never separate launches that spin on
each other).

Checks (rows a16 / a17 / a18 and the fused sync kernel of SURVEY.md §8a):
* weighted reduce-scatter: the fp32 sum over ranks in rank order is bit-exact against the same
  fixed-order float32 sum computed by torch, with and without accumulation;
* fused reduce-scatter + AdamW + all-gather: the update within rel 1e-5 of float64 AdamW on the
  same gradient, the gradient bit-exact, and every rank's bf16 parameter buffer holding
  bf16(master) of every shard;
* all-gather: bit-exact copy of every rank's shard.
The multi-process tests (tests/test_multigpu_gpu.py) run the same kernels across real GPUs.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_lib = None


def lib():
    global _lib
    if _lib is None:
        from paper_2408_12596_b200 import _lib as L
        l = L.lib
        P, I64, I32, U32 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32
        l.zp_peer_group_create.argtypes = [I32, P, I64, C.POINTER(P)]
        l.zp_peer_group_destroy.argtypes = [P]
        l.zp_peer_rs_accumulate.argtypes = [P, I64, I64, I64, I32, U32, I32, P]
        l.zp_peer_rs_adam_ag.argtypes = [P, I64, I32, I64, I64, I64, I64, I64, I64, I64, P, U32, I32, P]
        l.zp_peer_all_gather.argtypes = [P, I64, I64, I64, U32, I32, P]
        _lib = l
    return _lib


class AdamP(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("lr", "beta1", "beta2", "eps", "weight_decay", "bc1", "bc2")]


def _align(x, a=256):
    return (x + a - 1) // a * a


class Group:
    """n arenas of `region` bytes carved from one device allocation; `layout` maps buffer names
    to (byte offset, element count, dtype), the same in every arena."""

    def __init__(self, n, layout):
        import torch
        self.n, self.layout = n, {}
        off = 0
        for name, (count, dtype) in layout.items():
            esz = torch.tensor([], dtype=dtype).element_size()
            self.layout[name] = (off, count, dtype)
            off = _align(off + count * esz)
        self.region = _align(off, 4096)
        self.buf = torch.zeros(n * self.region, dtype=torch.uint8, device="cuda")
        self.h = C.c_void_p()
        assert lib().zp_peer_group_create(n, C.c_void_p(self.buf.data_ptr()), self.region, C.byref(self.h)) == 0
        self.epoch = 0

    def off(self, name):
        return self.layout[name][0]

    def view(self, rank, name):
        import torch
        off, count, dtype = self.layout[name]
        nbytes = count * torch.tensor([], dtype=dtype).element_size()
        return self.buf[rank * self.region + off: rank * self.region + off + nbytes].view(dtype)

    def next_epoch(self):
        self.epoch += 1
        return self.epoch

    def close(self):
        lib().zp_peer_group_destroy(self.h)


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_pull_reduce_scatter_is_fixed_order_sum(cuda, n):
    import torch
    L = 8 * 4099  # odd number of 8-element vectors: exercises the tail loop
    total = n * L
    g = Group(n, {"src": (total, torch.bfloat16), "acc": (L, torch.float32)})
    torch.manual_seed(n)
    for j in range(n):
        g.view(j, "src").copy_(torch.randn(total, device="cuda").to(torch.bfloat16))
        g.view(j, "acc").copy_(torch.randn(L, device="cuda"))
    for overwrite in (1, 0):
        prev = [g.view(r, "acc").clone() for r in range(n)]
        assert lib().zp_peer_rs_accumulate(g.h, g.off("src"), L, g.off("acc"), overwrite, g.next_epoch(), 2,
                                           _stream()) == 0
        torch.cuda.synchronize()
        for r in range(n):
            ref = torch.zeros(L, device="cuda")
            for j in range(n):
                ref = ref + g.view(j, "src")[r * L:(r + 1) * L].float()
            if not overwrite:
                ref = ref + prev[r]
            assert torch.equal(g.view(r, "acc"), ref), (n, r, overwrite)
    g.close()


@pytest.mark.parametrize("n,src_f32", [(2, False), (4, False), (4, True), (8, False)])
def test_fused_reduce_scatter_adamw_all_gather(cuda, n, src_f32):
    import torch
    L = 8 * 1031
    total = n * L
    sdt = torch.float32 if src_f32 else torch.bfloat16
    g = Group(n, {"src": (total, sdt), "p16": (total, torch.bfloat16), "p32": (L, torch.float32),
                  "m": (L, torch.float32), "v": (L, torch.float32), "acc": (L, torch.float32),
                  "gout": (L, torch.float32)})
    torch.manual_seed(10 + n)
    for j in range(n):
        g.view(j, "src").copy_((1e-3 * torch.randn(total, device="cuda")).to(sdt))
        g.view(j, "p32").copy_(torch.randn(L, device="cuda") * 0.02)
        g.view(j, "acc").copy_(1e-3 * torch.randn(L, device="cuda"))
    lr, b1, b2, eps, wd = 1e-3, 0.9, 0.95, 1e-8, 0.1
    for t in (1, 2):
        ap = AdamP(lr, b1, b2, eps, wd, 1 - b1 ** t, 1 - b2 ** t)
        before = [tuple(g.view(r, k).double().cpu().numpy() for k in ("p32", "m", "v")) for r in range(n)]
        assert lib().zp_peer_rs_adam_ag(g.h, g.off("src"), int(src_f32), L, g.off("acc"), g.off("p32"), g.off("m"),
                                        g.off("v"), g.off("p16"), g.off("gout"), C.byref(ap), g.next_epoch(), 2,
                                        _stream()) == 0
        torch.cuda.synchronize()
        for r in range(n):
            ref = torch.zeros(L, device="cuda")
            for j in range(n):
                ref = ref + g.view(j, "src")[r * L:(r + 1) * L].float()
            ref = ref + g.view(r, "acc")
            assert torch.equal(g.view(r, "gout"), ref), (n, r, t)
            P0, M0, V0 = before[r]
            G = ref.double().cpu().numpy()
            M1 = b1 * M0 + (1 - b1) * G
            V1 = b2 * V0 + (1 - b2) * G * G
            P1 = P0 - lr * ((M1 / (1 - b1 ** t)) / (np.sqrt(V1 / (1 - b2 ** t)) + eps) + wd * P0)
            got = g.view(r, "p32").double().cpu().numpy()
            assert np.linalg.norm(got - P1) / np.linalg.norm(P1) < 1e-5
            m1 = g.view(r, "m").double().cpu().numpy()
            assert np.linalg.norm(m1 - M1) / np.linalg.norm(M1) < 1e-5
        # every rank's p16 holds bf16(master) of every shard (the push all-gather)
        full = torch.cat([g.view(r, "p32").to(torch.bfloat16) for r in range(n)])
        for j in range(n):
            assert torch.equal(g.view(j, "p16"), full), (n, j, t)
    g.close()


@pytest.mark.parametrize("n", [2, 4, 8])
def test_pull_all_gather_is_exact(cuda, n):
    import torch
    L = 8 * 2053
    g = Group(n, {"shard": (L, torch.bfloat16), "dst": (n * L, torch.bfloat16)})
    torch.manual_seed(20 + n)
    for j in range(n):
        g.view(j, "shard").copy_(torch.randn(L, device="cuda").to(torch.bfloat16))
    for _ in range(2):  # epoch reuse of the flag blocks
        for j in range(n):
            g.view(j, "dst").fill_(float("nan"))
        assert lib().zp_peer_all_gather(g.h, g.off("shard"), g.off("dst"), L, g.next_epoch(), 2, _stream()) == 0
        torch.cuda.synchronize()
        full = torch.cat([g.view(j, "shard") for j in range(n)])
        for r in range(n):
            assert torch.equal(g.view(r, "dst"), full), (n, r)
    g.close()


def test_peer_group_rejects_bad_arguments(cuda):
    import torch
    g = Group(2, {"src": (64, torch.bfloat16), "acc": (32, torch.float32)})
    # length not a multiple of 8 -> ZP_EINVAL (1), nothing launched
    assert lib().zp_peer_rs_accumulate(g.h, g.off("src"), 12, g.off("acc"), 1, 1, 2, None) == 1
    assert lib().zp_peer_rs_accumulate(g.h, g.off("src"), 8, -1, 1, 1, 2, None) == 1
    g.close()
