"""Timeline of attention CTA 0 (VPE_ATT_TRACE=1): per event code the clock64 deltas."""
import ctypes
import os
import sys

os.environ["VPE_ATT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops
from paper_2508_11584_b200._lib import lib

B, T, H = 16, 1025, 6
D = H * 64
qkv = torch.randn(B * T, 3 * D, device="cuda").to(torch.bfloat16)
for _ in range(3):
    _ops.attention(qkv, B, T, D, H)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
lib.vpe_debug_att_trace(ctypes.cast(buf, ctypes.c_void_p), 4096)
ev = [(buf[i], buf[i + 1]) for i in range(0, 4096, 2)]
t0 = min(t for c, t in ev if c)
for name, lo, hi in (("mma", 0, 1024), ("softA", 1024, 1536), ("softB", 1536, 2048)):
    rows = [(c, t - t0) for c, t in ev[lo:hi] if c]
    print(name, len(rows))
    print(" ".join(f"{c}@{t}" for c, t in rows[:160]))
