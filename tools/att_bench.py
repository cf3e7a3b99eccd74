"""Attention kernel timing + accuracy at the engine's shapes (graph-timed, CUDA events).
  VPE_ATT_POLY=k python tools/att_bench.py   (k selects the FMA-pipe exp2 share, csrc/attention.cu)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops
from microbench import timeit_graph


def main():
    dev = torch.device("cuda")
    for (B, T, H) in [(16, 1025, 6), (16, 1370, 12), (8, 1370, 16), (1, 1025, 6), (2, 257, 6)]:
        D = H * 64
        g = torch.Generator().manual_seed(T + B)
        qkv = torch.randn(B * T, 3 * D, generator=g).to(dev, torch.bfloat16)
        out = _ops.attention(qkv, B, T, D, H)
        out2 = _ops.attention(qkv, B, T, D, H)
        q, k, v = qkv.float().view(B, T, 3, H, 64).permute(2, 0, 3, 1, 4)
        ref = (torch.softmax(q @ k.transpose(-1, -2) / 8.0, -1) @ v).transpose(1, 2).reshape(B * T, D)
        err = ((out.float() - ref).norm() / ref.norm()).item()
        us = timeit_graph(lambda: _ops.attention(qkv, B, T, D, H))
        fl = 4.0 * B * T * T * D
        print(json.dumps(dict(kernel="attention", poly=os.environ.get("VPE_ATT_POLY", "3"), dbg=os.environ.get("VPE_ATT_DBG", "0"), B=B, T=T, H=H,
                              us=round(us, 2), tflops=round(fl / us * 1e-6, 1), rel_l2=err,
                              deterministic=bool(torch.equal(out, out2)))), flush=True)


if __name__ == "__main__":
    main()
