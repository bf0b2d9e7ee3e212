import sys, os, torch
sys.path.insert(0, os.getcwd())
from tests.test_attention_gpu import ref_attention, relerr
from paper_2408_12596_b200 import _lib
L = _lib.lib
cuda = torch.device("cuda:0")
for (b, s, H, ctas) in [(1, 128, 1, 0), (2, 256, 2, 0), (2, 1024, 12, 0), (3, 512, 4, 37)]:
    h = H * 64; T = b * s
    g = torch.Generator(device="cpu").manual_seed(b * 1000 + s + H)
    qkv = torch.randn(T, 3 * h, generator=g).to(torch.bfloat16).to(cuda)
    for rep in range(2):
        out = torch.full((T, h), float('nan'), dtype=torch.bfloat16, device=cuda)
        lse = torch.full((b * H * s,), float('nan'), dtype=torch.float32, device=cuda)
        rc = L.zp_attention_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), b, s, H, ctas, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ro, rl = ref_attention(qkv, b, s, H)
        bad = (lse - rl).abs() > 1e-3
        print((b, s, H, ctas), rep, rc, "lse", relerr(lse, rl), "o", relerr(out, ro), "bad rows", int(bad.sum()), "nan", int(torch.isnan(lse).sum()))
        if bad.any():
            idx = bad.nonzero()[:8].flatten().tolist()
            print("   first bad", idx, lse[idx].tolist(), rl[idx].tolist())
