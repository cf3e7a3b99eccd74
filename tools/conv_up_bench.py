"""DPT head resize+conv shapes at B=16: fused conv_up_kernel vs bilinear + halo conv (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    B = int(os.environ.get("VPE_BATCH", "16"))
    dev = "cuda"
    for Hs, Cp, Ho in [(128, 64, 256), (256, 32, 448)]:
        x = torch.randn(B, Hs, Hs, Cp, device=dev).to(torch.bfloat16)
        w = (torch.randn(32, 9 * Cp, device=dev) * 0.05).to(torch.bfloat16)
        bias = torch.zeros(32, device=dev)
        out = torch.empty(B, Ho, Ho, 32, device=dev, dtype=torch.bfloat16)
        up = _ops.bilinear(x, Ho, Ho)
        wp = _ops.conv_up_pack(w)
        tf = t(lambda: _ops.conv_up(x, w, Ho, Ho, bias=bias, out=out, wpack=wp))
        tb = t(lambda: _ops.bilinear(x, Ho, Ho))
        tc = t(lambda: _ops.conv(up, w, Cp, 3, bias=bias, out=out))
        print(f"{Hs}->{Ho} C{Cp}: fused {tf:.1f} us | bilinear {tb:.1f} + conv {tc:.1f} = {tb + tc:.1f} us")
        if Cp == 32:  # the DPT head2 form: depth epilogue (what the engine runs)
            w3 = torch.randn(32, device=dev) * 0.1
            d = torch.empty(B, Ho, Ho, device=dev)
            td = t(lambda: _ops.conv_up(x, w, Ho, Ho, bias=bias, w3=w3, b3=0.1, out=d, wpack=wp))
            print(f"{Hs}->{Ho} C{Cp} depth epilogue: fused {td:.1f} us")


if __name__ == "__main__":
    main()
