"""Launch one kernel shape a few times (for ncu captures): attention / gemm."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops


def main():
    p = argparse.ArgumentParser()
    p.add_argument("what", choices=["attention", "gemm"])
    p.add_argument("--B", type=int, default=16)
    p.add_argument("--T", type=int, default=1025)
    p.add_argument("--H", type=int, default=6)
    p.add_argument("--M", type=int, default=16400)
    p.add_argument("--N", type=int, default=1536)
    p.add_argument("--K", type=int, default=384)
    p.add_argument("--act", type=int, default=1)
    p.add_argument("--bn", type=int, default=128)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--time", action="store_true")
    a = p.parse_args()
    dev = torch.device("cuda")
    if a.what == "attention":
        D = a.H * 64
        qkv = torch.randn(a.B * a.T, 3 * D, device=dev).to(torch.bfloat16)
        fn = lambda: _ops.attention(qkv, a.B, a.T, D, a.H)
    else:
        x = torch.randn(a.M, a.K, device=dev).to(torch.bfloat16)
        w = (torch.randn(a.N, a.K, device=dev) * 0.02).to(torch.bfloat16)
        bias = torch.zeros(a.N, device=dev)
        out = torch.empty(a.M, a.N, device=dev, dtype=torch.bfloat16)
        fn = lambda: _ops.linear(x, w, bias=bias, out=out, act=a.act, bn=a.bn)
    for _ in range(a.reps):
        fn()
    torch.cuda.synchronize()
    if a.time:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(a.what, "us", e0.elapsed_time(e1) / 50 * 1e3)


if __name__ == "__main__":
    main()
