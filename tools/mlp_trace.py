"""MMA-thread timeline of fused-MLP CTA 0 (VPE_MLP_TRACE=1)."""
import ctypes
import os
import sys

os.environ["VPE_MLP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops
from paper_2508_11584_b200._lib import lib

M, D, Hd = 16400, 384, 1536
dev = "cuda"
x = torch.randn(M, D, device=dev).to(torch.bfloat16)
w1 = (torch.randn(Hd, D, device=dev) * 0.05).to(torch.bfloat16)
w2 = (torch.randn(D, Hd, device=dev) * 0.03).to(torch.bfloat16)
b1, b2, ls2 = torch.zeros(Hd, device=dev), torch.zeros(D, device=dev), torch.ones(D, device=dev)
resid = torch.zeros(M, D, device=dev)
for _ in range(3):
    _ops.mlp(x, w1, b1, w2, b2, ls2, resid)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
lib.vpe_debug_mlp_trace(ctypes.cast(buf, ctypes.c_void_p), 4096)
ev = [(buf[i], buf[i + 1]) for i in range(0, 4096, 2) if buf[i]]
t0 = ev[0][1]
print(" ".join(f"{c}@{t - t0}" for c, t in ev[:160]))
