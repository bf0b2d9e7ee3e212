"""Single-GPU parity of the NVLink peer-memory collectives (csrc/cuda/peer.cu) through the C ABI
(zp_kernels.h peer group): n "rank arenas" are n regions of one device allocation, each rank's
kernel instance runs on its own stream (the flag barriers need all n instances co-resident).

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
        P = C.c_void_p
        l.zp_peer_group_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p), C.POINTER(P)]
        l.zp_peer_group_destroy.argtypes = [P]
        l.zp_peer_rs_accumulate.argtypes = [P, C.c_int32, C.c_int64, C.c_int64, P, C.c_int64, C.c_int32,
                                            C.c_uint32, C.c_int32, P]
        l.zp_peer_rs_adam_ag.argtypes = [P, C.c_int32, C.c_int64, C.c_int32, C.c_int64, P, P, P, P, C.c_int64, P,
                                         C.c_int64, P, C.c_uint32, C.c_int32, P]
        l.zp_peer_all_gather.argtypes = [P, C.c_int32, C.c_int64, P, C.c_int64, C.c_uint32, C.c_int32, P]
        _lib = l
    return _lib


class AdamP(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("lr", "beta1", "beta2", "eps", "weight_decay", "bc1", "bc2")]


class Group:
    """n arenas of `region` bytes carved from one device allocation."""

    def __init__(self, n, region):
        import torch
        self.n, self.region = n, region
        self.buf = torch.zeros(n * region, dtype=torch.uint8, device="cuda")
        bases = (C.c_void_p * n)(*[self.buf.data_ptr() + j * region for j in range(n)])
        self.h = C.c_void_p()
        assert lib().zp_peer_group_create(n, bases, C.byref(self.h)) == 0
        self.streams = [torch.cuda.Stream() for _ in range(n)]
        self.epoch = 0

    def view(self, rank, off, count, dtype):
        import torch
        nbytes = count * torch.tensor([], dtype=dtype).element_size()
        return self.buf[rank * self.region + off: rank * self.region + off + nbytes].view(dtype)

    def launch_all(self, fn):
        """fn(rank, stream, epoch) -> rc, for every rank, concurrently."""
        import torch
        torch.cuda.synchronize()
        self.epoch += 1
        for r in range(self.n):
            assert fn(r, C.c_void_p(self.streams[r].cuda_stream), self.epoch) == 0
        torch.cuda.synchronize()

    def close(self):
        lib().zp_peer_group_destroy(self.h)


def _ptr(t):
    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("n", [2, 4, 8])
def test_pull_reduce_scatter_is_fixed_order_sum(cuda, n):
    import torch
    L = 8 * 4099  # odd number of 8-element vectors: exercises the tail loop
    total = n * L
    g = Group(n, total * 2 + 4096)
    torch.manual_seed(n)
    for j in range(n):
        g.view(j, 0, total, torch.bfloat16).copy_(torch.randn(total, device="cuda").to(torch.bfloat16))
    accs = [torch.randn(L, device="cuda") for _ in range(n)]
    for overwrite in (1, 0):
        prev = [a.clone() for a in accs]
        g.launch_all(lambda r, s, e: lib().zp_peer_rs_accumulate(g.h, r, 0, r * L, _ptr(accs[r]), L, overwrite,
                                                                 e, 2, s))
        for r in range(n):
            ref = torch.zeros(L, device="cuda")
            for j in range(n):
                ref = ref + g.view(j, 0, total, torch.bfloat16)[r * L:(r + 1) * L].float()
            if not overwrite:
                ref = ref + prev[r]
            assert torch.equal(accs[r], ref), (n, r, overwrite)
    g.close()


@pytest.mark.parametrize("n,src_f32", [(2, False), (4, False), (4, True), (8, False)])
def test_fused_reduce_scatter_adamw_all_gather(cuda, n, src_f32):
    import torch
    L = 8 * 1031
    total = n * L
    esz = 4 if src_f32 else 2
    p16_off = (total * esz + 255) // 256 * 256
    g = Group(n, p16_off + total * 2 + 4096)
    torch.manual_seed(10 + n)
    sdt = torch.float32 if src_f32 else torch.bfloat16
    for j in range(n):
        g.view(j, 0, total, sdt).copy_((1e-3 * torch.randn(total, device="cuda")).to(sdt))
    p32 = [torch.randn(L, device="cuda") * 0.02 for _ in range(n)]
    m = [torch.zeros(L, device="cuda") for _ in range(n)]
    v = [torch.zeros(L, device="cuda") for _ in range(n)]
    acc = [1e-3 * torch.randn(L, device="cuda") for _ in range(n)]
    gout = [torch.empty(L, device="cuda") for _ in range(n)]
    lr, b1, b2, eps, wd = 1e-3, 0.9, 0.95, 1e-8, 0.1
    for t in (1, 2):
        ap = AdamP(lr, b1, b2, eps, wd, 1 - b1 ** t, 1 - b2 ** t)
        before = [(p.double().cpu().numpy(), mm.double().cpu().numpy(), vv.double().cpu().numpy())
                  for p, mm, vv in zip(p32, m, v)]
        g.launch_all(lambda r, s, e: lib().zp_peer_rs_adam_ag(
            g.h, r, 0, int(src_f32), r * L, _ptr(acc[r]), _ptr(p32[r]), _ptr(m[r]), _ptr(v[r]), p16_off,
            _ptr(gout[r]), L, C.byref(ap), e, 2, s))
        for r in range(n):
            ref = torch.zeros(L, device="cuda")
            for j in range(n):
                ref = ref + g.view(j, 0, total, sdt)[r * L:(r + 1) * L].float()
            ref = ref + acc[r]
            assert torch.equal(gout[r], ref), (n, r, t)
            P0, M0, V0 = before[r]
            G = ref.double().cpu().numpy()
            M1 = b1 * M0 + (1 - b1) * G
            V1 = b2 * V0 + (1 - b2) * G * G
            P1 = P0 - lr * ((M1 / (1 - b1 ** t)) / (np.sqrt(V1 / (1 - b2 ** t)) + eps) + wd * P0)
            got = p32[r].double().cpu().numpy()
            assert np.linalg.norm(got - P1) / np.linalg.norm(P1) < 1e-5
            assert np.linalg.norm(m[r].double().cpu().numpy() - M1) / np.linalg.norm(M1) < 1e-5
        # every rank's p16 holds bf16(master) of every shard (the push all-gather)
        full = torch.cat([p.to(torch.bfloat16) for p in p32])
        for j in range(n):
            assert torch.equal(g.view(j, p16_off, total, torch.bfloat16), full), (n, j, t)
    g.close()


@pytest.mark.parametrize("n", [2, 4, 8])
def test_pull_all_gather_is_exact(cuda, n):
    import torch
    L = 8 * 2053
    g = Group(n, L * 2 + 4096)
    torch.manual_seed(20 + n)
    for j in range(n):
        g.view(j, 0, L, torch.bfloat16).copy_(torch.randn(L, device="cuda").to(torch.bfloat16))
    dst = [torch.empty(n * L, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    for _ in range(2):  # epoch reuse of the flag blocks
        for d in dst:
            d.fill_(float("nan"))
        g.launch_all(lambda r, s, e: lib().zp_peer_all_gather(g.h, r, 0, _ptr(dst[r]), L, e, 2, s))
        full = torch.cat([g.view(j, 0, L, torch.bfloat16) for j in range(n)])
        for r in range(n):
            assert torch.equal(dst[r], full), (n, r)
    g.close()


def test_peer_group_rejects_bad_arguments(cuda):
    import torch
    g = Group(2, 4096)
    buf = torch.zeros(16, device="cuda")
    # length not a multiple of 8 -> ZP_EINVAL (1), nothing launched
    assert lib().zp_peer_rs_accumulate(g.h, 0, 0, 0, _ptr(buf), 12, 1, 1, 2, None) == 1
    assert lib().zp_peer_rs_accumulate(g.h, 5, 0, 0, _ptr(buf), 8, 1, 1, 2, None) == 1
    g.close()
