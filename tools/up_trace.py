"""Per-role timeline of conv_up_kernel CTA 0 (diagnostics build: VPE_BUILD_TAG=trace
VPE_NVCC_EXTRA=-DVPE_TRACE_BUILD, run with VPE_LIB=libvpe_trace.so). Events: MMA 1 tempty ok,
2 halo full, 3 issued; TMA 11 source slot free; builder 21 halo slot free, 22 source full,
23 built; epilogue 31 accumulator full, 32 stored. Prints per-role per-tile period medians.

  python tools/up_trace.py [depth|conv]"""
import ctypes
import os
import sys

os.environ.setdefault("VPE_GEMM_TRACE", "1")
os.environ.setdefault("VPE_LIB", "libvpe_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops
from paper_2508_11584_b200._lib import lib

mode = sys.argv[1] if len(sys.argv) > 1 else "depth"
B, Hs, Cp, Ho = (16, 256, 32, 448) if mode == "depth" else (16, 128, 64, 256)
x = torch.randn(B, Hs, Hs, Cp, device="cuda").to(torch.bfloat16)
w = (torch.randn(32, 9 * Cp, device="cuda") * 0.05).to(torch.bfloat16)
bias = torch.zeros(32, device="cuda")
w3 = torch.randn(32, device="cuda") * 0.1 if mode == "depth" else None
wp = _ops.conv_up_pack(w)
for _ in range(3):
    _ops.conv_up(x, w, Ho, Ho, bias=bias, w3=w3, wpack=wp)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
lib.vpe_debug_gemm_trace(ctypes.cast(buf, ctypes.c_void_p), 4096)
roles = {"mma": 0, "tma": 510, "build": 1020, "epi": 1530}
ev = {r: [(buf[2 * (b + i)], buf[2 * (b + i) + 1]) for i in range(500) if buf[2 * (b + i)]] for r, b in roles.items()}
t0 = min(e[0][1] for e in ev.values() if e)
for r, e in ev.items():
    print(r, " ".join(f"{c}@{t - t0}" for c, t in e[:40]))
for r, e in ev.items():
    codes = sorted(set(c for c, _ in e))
    for c in codes:
        ts = [t for cc, t in e if cc == c]
        if len(ts) > 3:
            d = sorted(b - a for a, b in zip(ts, ts[1:]))
            print(f"{r} code {c}: n {len(ts)} period median {d[len(d) // 2]} clk")
