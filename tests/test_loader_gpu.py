"""Dynamic-batch loader: the synthetic token rows a rank synthesises on the device
for its contiguous sample range (zp_runtime_load_tokens with from_host = 0, the bench's and the
profiler's data) against a numpy restatement of the same function of (seed, iteration, sample,
position), bit-exact; a sample's row must not depend on which slice loads it; and a step run on
device-synthesised tokens equals the step run on the same tokens copied from the host."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


def mix64(z):  # splitmix64 finaliser on numpy uint64 arrays (wrapping arithmetic)
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(M64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def synth_ref(first, count, sp1, vocab, seed, it):
    """tok[i, t] = mix64(mix64(mix64(seed ^ K) ^ it) ^ (j << 20 | t)) % vocab, j = first + i
    (kernels.cu synth_tokens_k)."""
    with np.errstate(over="ignore"):
        base = mix64(mix64(np.uint64(seed) ^ np.uint64(0x7F4A7C15)) ^ np.uint64(it))
        j = np.arange(first, first + count, dtype=np.uint64)[:, None]
        t = np.arange(sp1, dtype=np.uint64)[None, :]
        h = mix64(base ^ ((j << np.uint64(20)) | t))
    return (h % np.uint64(vocab)).astype(np.int32)


def synth_dev(first, count, sp1, vocab, seed, it):
    import torch
    from paper_2408_12596_b200 import _lib
    out = torch.full((count * sp1,), -1, dtype=torch.int32, device="cuda")
    assert _lib.lib.zp_synth_tokens(out.data_ptr(), first, count, sp1, vocab, seed, it,
                                    torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    return out.view(count, sp1).cpu().numpy()


@pytest.mark.parametrize("first,count,sp1,vocab,seed,it", [(0, 6, 129, 1000, 7, 3), (1000, 3, 4097, 32000, 0, 0),
                                                           (5, 1, 257, 50257, 123456789, 41)])
def test_synth_tokens_match_numpy_restatement(cuda, first, count, sp1, vocab, seed, it):
    got = synth_dev(first, count, sp1, vocab, seed, it)
    assert np.array_equal(got, synth_ref(first, count, sp1, vocab, seed, it))
    assert got.min() >= 0 and got.max() < vocab


def test_sample_rows_do_not_depend_on_the_slice(cuda):
    full = synth_dev(0, 10, 129, 1000, 3, 2)
    for first, count in ((0, 4), (4, 3), (7, 3), (9, 1)):
        assert np.array_equal(synth_dev(first, count, 129, 1000, 3, 2), full[first:first + count])
    assert not np.array_equal(synth_dev(0, 10, 129, 1000, 3, 3), full)  # next iteration: new data


def test_step_on_device_tokens_equals_step_on_host_copy(cuda):
    from tests.test_step_gpu import TINY, make_plan, runtime
    first, B = 3, 4
    losses = []
    for from_host in (False, True):
        rt = runtime(cuda, seed=11)
        rt.resident_bytes(0)
        if from_host:
            rt.load_tokens(synth_ref(first, B, TINY["seq_len"] + 1, TINY["vocab"], 11, 5))
        else:
            rt.load_tokens(first_sample=first, count=B, iteration=5)
        losses.append(rt.execute_iteration(make_plan(0, B, B, B, 1), 0)["loss_sum"])
        rt.close()
    assert losses[0] == losses[1]
