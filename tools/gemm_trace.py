"""MMA-thread timeline of GEMM CTA 0 (VPE_GEMM_TRACE=1)."""
import ctypes
import os
import sys

os.environ.setdefault("VPE_GEMM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops
from paper_2508_11584_b200._lib import lib

M, N, K = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (16400, 1536, 384))]
bn = int(sys.argv[4]) if len(sys.argv) > 4 else 256
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _ops.linear(a, w, out=out, bn=bn)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    _ops.linear(a, w, out=out, bn=bn)
e1.record()
torch.cuda.synchronize()
print("us per launch", e0.elapsed_time(e1) / 20 * 1e3)
buf = (ctypes.c_ulonglong * 4096)()
lib.vpe_debug_gemm_trace(ctypes.cast(buf, ctypes.c_void_p), 4096)
ev = [(buf[i], buf[i + 1]) for i in range(0, 4096, 2) if buf[i]]
t0 = ev[0][1]
print(" ".join(f"{c}@{t - t0}" for c, t in ev[:200]))
