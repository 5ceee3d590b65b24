"""Per-CTA timeline of one tcgen05 GEMM launch (globaltimer marks, see gemm.cu trace_mark).

    python tools/gemm_trace.py N K M BN EPI
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_18521_b200 import _capi  # noqa: E402

N, K, M, BN, EPI = map(int, sys.argv[1:6])
W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
args = (C.c_void_p(W.data_ptr()), C.c_void_p(A.data_ptr()), C.c_void_p(out.data_ptr()), None, N, K, M, BN, EPI)
for _ in range(3):
    _capi.call("ab_debug_gemm", *args)
buf = (C.c_ulonglong * (160 * 16))()
_capi.call("ab_debug_gemm_trace", 1, None)
torch.cuda.synchronize()
_capi.call("ab_debug_trace_mark", 0)
_capi.call("ab_debug_gemm", *args)  # (synchronizes)
_capi.call("ab_debug_trace_mark", 1)
torch.cuda.synchronize()
_capi.call("ab_debug_gemm_trace", 0, buf)
mk = [buf[159 * 16], buf[159 * 16 + 1]]
t = [[buf[i * 16 + k] for k in range(16)] for i in range(160)]
t0 = min(r[0] for r in t[:159] if r[0])
t = t[:159]
ends = max(r[7] for r in t if r[7])
print(f"marker kernel before: {(mk[0] - t0) / 1e3:.2f} us, last CTA exit {(ends - t0) / 1e3:.2f} us, "
      f"marker after: {(mk[1] - t0) / 1e3:.2f} us (includes a host sync)")
names = ["entry", "setup", "tma0", "full0", "mma_end", "acc0", "epi_end", "exit", "part_wr", "prod0", "policy",
         "acquired", "fetched", "slot0", "epi_f0", "epi_lp"]
print(f"{'cta':>4} " + " ".join(f"{n:>8}" for n in names) + "   (us after the first CTA entry)")
for i, r in enumerate(t):
    if not r[0]:
        continue
    print(f"{i:4d} " + " ".join(f"{(x - t0) / 1e3:8.2f}" if x else f"{'-':>8}" for x in r[:16]))
