"""Diagnostics: run the engine step N times on the same frame and report which outputs differ
bitwise from the first run (taps / depth / seg / det), with PDL on (VPE_PDL=1) or off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200.engine import VPEngine
from paper_2508_11584_b200.weights import make_frames

B = int(os.environ.get("VPE_BATCH", "2"))
eng = VPEngine("vits14", 448, B)
eng.pixels.copy_(make_frames(B, 448, 0).to(eng.device))


def grab():
    eng.submit()
    eng.synchronize()
    out = {"depth": eng.out["depth"]["depth"].clone()}
    return out


ref = grab()
bad = 0
for i in range(int(os.environ.get("REPS", "20"))):
    o = grab()
    for k, v in o.items():
        if not torch.equal(v, ref[k]):
            bad += 1
            print(f"run {i}: {k} differs, max {(v - ref[k]).abs().max().item():.3e}")
print("differing runs:", bad)
