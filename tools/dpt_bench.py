"""DPT depth head alone at the bench config (S/14, 448, batch 16): CUDA-event time per forward,
and an ncu target (`ncu -k regex:conv_up ... python tools/dpt_bench.py`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200.config import model_config, tokens
from paper_2508_11584_b200.heads import DepthHead
from paper_2508_11584_b200.weights import make_weights


def main():
    B = int(os.environ.get("VPE_BATCH", "16"))
    model = os.environ.get("VPE_MODEL", "vits14")
    R = int(os.environ.get("VPE_RES", "448"))
    dev = torch.device("cuda:0")
    cfg = model_config(model)
    W = make_weights(model)
    taps = [torch.randn(B, tokens(R), cfg.backbone.dim, device=dev).to(torch.bfloat16) for _ in range(4)]
    head = DepthHead(W, cfg, R, B, dev)
    depth = torch.empty(B, R, R, device=dev)
    for _ in range(3):
        head.forward(taps, depth)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        head.forward(taps, depth)
    b.record()
    torch.cuda.synchronize()
    print(f"dpt head {model} B={B} R={R}: {a.elapsed_time(b) / reps * 1e3:.1f} us/forward")


if __name__ == "__main__":
    main()
