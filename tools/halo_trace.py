"""Per-role timeline of halo-conv CTA 0 (VPE_GEMM_TRACE=1): MMA issuer (1 tempty ok, 2 A full,
3 MMAs issued), TMA producer (11 A slot free), epilogue warp 2 (21 accumulator full, 23 stores
done). Prints per-tile clocks relative to the first event.

  python tools/halo_trace.py B H C N   (default 16 256 64 32)"""
import ctypes
import os
import sys

os.environ.setdefault("VPE_GEMM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops
from paper_2508_11584_b200._lib import lib

B, H, C, N = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (16, 256, 64, 32))]
x = torch.randn(B, H, H, C, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, 9 * C, device="cuda") * 0.02).to(torch.bfloat16)
bias = torch.zeros(N, device="cuda")
out = torch.empty(B, H, H, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _ops.conv(x, w, C, 3, bias=bias, out=out)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
lib.vpe_debug_gemm_trace(ctypes.cast(buf, ctypes.c_void_p), 4096)
roles = {"mma": 0, "tma": 680, "epi": 1360}
ev = {}
for r, base in roles.items():
    ev[r] = [(buf[2 * (base + i)], buf[2 * (base + i) + 1]) for i in range(600) if buf[2 * (base + i)]]
t0 = min(e[0][1] for e in ev.values() if e)
for r, e in ev.items():
    print(r, " ".join(f"{c}@{t - t0}" for c, t in e[:90]))
m = [t for c, t in ev["mma"] if c == 1]
if len(m) > 2:
    d = [b - a for a, b in zip(m, m[1:])]
    print("mma tile period clk: median", sorted(d)[len(d) // 2], "n", len(m))
