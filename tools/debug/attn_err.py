import sys, os, torch, ctypes
sys.path.insert(0, os.getcwd())
from paper_2408_12596_b200 import _lib
L = _lib.lib
cuda = torch.device("cuda:0")
b, s, H = 2, 256, 2
h = H * 64; T = b * s
qkv = torch.randn(T, 3 * h, device=cuda).to(torch.bfloat16)
out = torch.empty(T, h, dtype=torch.bfloat16, device=cuda)
lse = torch.empty(b * H * s, dtype=torch.float32, device=cuda)
st = torch.cuda.current_stream().cuda_stream
print("fwd", L.zp_attention_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), b, s, H, 0, st))
dout = torch.randn(T, h, device=cuda).to(torch.bfloat16)
dvec = torch.empty(b * H * s, dtype=torch.float32, device=cuda)
dq32 = torch.empty(T, h, dtype=torch.float32, device=cuda)
dqkv = torch.zeros(T, 3 * h, dtype=torch.bfloat16, device=cuda)
rc = L.zp_attention_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dvec.data_ptr(), dq32.data_ptr(), dqkv.data_ptr(), b, s, H, 0, st)
cudart = ctypes.CDLL("libcudart.so.12")
cudart.cudaGetErrorString.restype = ctypes.c_char_p
print("bwd rc", rc, cudart.cudaGetErrorString(cudart.cudaPeekAtLastError()), cudart.cudaGetErrorString(cudart.cudaDeviceSynchronize()))
