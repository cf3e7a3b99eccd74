"""Kernel microbenchmarks (CUDA events on the launching stream): GEMM variants, attention, LN."""
import argparse
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops


def timeit(fn, reps=100, warm=10):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def timeit_graph(fn, reps=20, replays=5):
    """Device time per call with host overhead removed: `reps` calls captured in one CUDA graph."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(replays):
        g.replay()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (reps * replays) * 1e3  # us


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--only", default="")
    p.add_argument("--conv", action="store_true")
    p.add_argument("--bns", default="128,192,256,-128,-256")
    args = p.parse_args()
    dev = torch.device("cuda")
    res = []
    if args.only == "rln":  # residual GEMM + LayerNorm kernel vs the GEMM with LN in its epilogue
        M, D = 16400, 384
        for K in (384, 1536):
            a = torch.randn(M, K, device=dev).to(torch.bfloat16)
            w = (torch.randn(D, K, device=dev) * 0.05).to(torch.bfloat16)
            bias, ls = torch.zeros(D, device=dev), torch.ones(D, device=dev) * 0.1
            lw, lb = torch.ones(D, device=dev), torch.zeros(D, device=dev)
            resid = torch.randn(M, D, device=dev)
            t_g = timeit_graph(lambda: _ops.linear(a, w, bias=bias, scale=ls, out=resid, kind=_ops.EPI_RESID, bn=256))
            t_ln = timeit_graph(lambda: _ops.layernorm(resid, lw, lb))
            t_f = timeit_graph(lambda: _ops.linear_resid_ln(a, w, bias, ls, resid, lw, lb, 1e-6))
            print(json.dumps(dict(K=K, gemm_resid_us=t_g, layernorm_us=t_ln, fused_us=t_f)), flush=True)
        return
    if args.only == "seg":
        for (B, h, C, cp) in [(16, 32, 150, 160), (1, 32, 150, 160)]:
            lg = torch.randn(B, h * h, cp, device=dev)
            us = timeit_graph(lambda: _ops.upsample_argmax(lg, h, 14 * h, classes=C))
            print(json.dumps(dict(kernel="upsample_argmax", B=B, h=h, C=C, us=us)), flush=True)
        return
    gemms = [] if args.only == "attention" else None
    for (M, N, K) in [(16400, 1536, 384), (16400, 384, 1536), (16400, 1152, 384), (16400, 384, 384), (8192, 8192, 8192)] if gemms is None else gemms:
        a = torch.randn(M, K, device=dev).to(torch.bfloat16)
        w = (torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16)
        bias = torch.zeros(N, device=dev)
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        outf = torch.empty(M, N, device=dev, dtype=torch.float32)
        for bn in [int(x) for x in args.bns.split(",")]:
            for act in (0, 1):
                us = timeit_graph(lambda: _ops.linear(a, w, bias=bias, out=out, act=act, bn=bn))
                tf = 2 * M * N * K / us * 1e-6
                res.append(dict(M=M, N=N, K=K, bn=bn, act=act, us=us, tflops=tf))
                print(json.dumps(res[-1]), flush=True)
        if N == 384:  # the backbone's proj / FC2: LayerScale + fp32 residual reduce-add epilogue
            resid = torch.zeros(M, N, device=dev)
            for bn in [int(x) for x in args.bns.split(",")]:
                us = timeit_graph(lambda: _ops.linear(a, w, bias=bias, scale=bias, out=resid, kind=_ops.EPI_RESID, bn=bn))
                print(json.dumps(dict(M=M, N=N, K=K, bn=bn, kind="resid", us=us)), flush=True)
        us = timeit_graph(lambda: torch.matmul(a, w.t(), out=out))
        print(json.dumps(dict(M=M, N=N, K=K, impl="cublas", us=us, tflops=2 * M * N * K / us * 1e-6)), flush=True)
    if args.only == "gemm":
        return
    for (B, T, H) in [(16, 1025, 6), (1, 1025, 6), (8, 1370, 16), (1, 1370, 12)]:
        D = H * 64
        qkv = torch.randn(B * T, 3 * D, device=dev).to(torch.bfloat16)
        us = timeit(lambda: _ops.attention(qkv, B, T, D, H))
        fl = 4.0 * B * T * T * D
        print(json.dumps(dict(kernel="attention", B=B, T=T, H=H, us=us, tflops=fl / us * 1e-6)), flush=True)


if __name__ == "__main__":
    main()


def conv_bench():
    dev = torch.device("cuda")
    for (B, H, C, N) in [(16, 128, 64, 64), (16, 256, 64, 32), (16, 448, 32, 32), (16, 64, 64, 64), (16, 32, 384, 384)]:
        x = torch.randn(B, H, H, C, device=dev).to(torch.bfloat16)
        w = (torch.randn(N, 9 * C, device=dev) * 0.02).to(torch.bfloat16)
        bias = torch.zeros(N, device=dev)
        out = torch.empty(B, H, H, N, device=dev, dtype=torch.bfloat16)
        us = timeit_graph(lambda: _ops.conv(x, w, C, 3, bias=bias, out=out))
        fl = 2.0 * B * H * H * N * 9 * C
        print(json.dumps(dict(kernel="conv3x3", B=B, H=H, C=C, N=N, us=us, tflops=fl / us * 1e-6)), flush=True)


if __name__ == "__main__" and "--conv" in sys.argv:
    conv_bench()
