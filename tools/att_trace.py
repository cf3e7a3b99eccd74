"""Timeline of attention CTA 0 (diagnostics build: VPE_NVCC_EXTRA=-DVPE_TRACE_BUILD python
paper_2508_11584_b200/build.py -f; then VPE_ATT_TRACE=1). Events (code@clk):
  MMA slot x: 20 S issued, 21/22 P half 0/1 ready (PV half issued right after)
  softmax slot x (warp quad 0, half 0): 10 wait S, 11 got S, 12 max pass + token + P free done, 13 P written"""
import ctypes
import os
import sys

os.environ["VPE_ATT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops
from paper_2508_11584_b200._lib import lib

B, T, H = [int(x) for x in os.environ.get("ATT_SHAPE", "16,1025,6").split(",")]
D = H * 64
qkv = torch.randn(B * T, 3 * D, device="cuda").to(torch.bfloat16)
for _ in range(3):
    _ops.attention(qkv, B, T, D, H)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
lib.vpe_debug_att_trace(ctypes.cast(buf, ctypes.c_void_p), 4096)
ev = [(buf[i], buf[i + 1]) for i in range(0, 4096, 2)]
t0 = min(t for c, t in ev if c)
for name, lo, hi in (("mmaA", 0, 512), ("mmaB", 512, 1024), ("softA", 1024, 1536), ("softB", 1536, 2048)):
    rows = [(c, t - t0) for c, t in ev[lo:hi] if c]
    print(name, len(rows))
    print(" ".join(f"{c}@{t}" for c, t in rows[:400]))

if os.environ.get("VPE_ATT_DBG", "0") == "32":
    # per-warp pass start/end (codes 12/17) of softmax warps 3..18
    for sw in range(16):
        rows = [(c, t - t0) for c, t in ev[1024 + 64 * sw: 1024 + 64 * (sw + 1)] if c]
        print(f"warp{sw + 1}", " ".join(f"{c}@{t}" for c, t in rows[:40]))
    for x in range(2):
        rows = [(c, t - t0) for c, t in ev[512 * x: 512 * (x + 1)] if c]
        print(f"mmadone{'AB'[x]}", " ".join(f"{c}@{t}" for c, t in rows[:60]))
