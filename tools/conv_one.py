"""Launch one 3x3 conv shape a few times (ncu target): python tools/conv_one.py B H C N."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops

B, H, C, N = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (16, 256, 64, 32))]
x = torch.randn(B, H, H, C, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, 9 * C, device="cuda") * 0.02).to(torch.bfloat16)
bias = torch.zeros(N, device="cuda")
out = torch.empty(B, H, H, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _ops.conv(x, w, C, 3, bias=bias, out=out)
torch.cuda.synchronize()
