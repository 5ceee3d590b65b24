"""One tcgen05 GEMM launch (for ncu): python tools/gemm_one.py N K M BN EPI"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_18521_b200 import _capi
N, K, M, BN, EPI = map(int, sys.argv[1:6])
W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
for _ in range(2):
    _capi.call("ab_debug_gemm", C.c_void_p(W.data_ptr()), C.c_void_p(A.data_ptr()), C.c_void_p(out.data_ptr()), None, N, K, M, BN, EPI)
torch.cuda.synchronize()
