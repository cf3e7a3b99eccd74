"""Run a few engine steps inside an NVTX range "prof" so ncu can capture exactly the steady-state
launches of one step:

  ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --batch 16
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200.engine import VPEngine


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--resolution", type=int, default=448)
    p.add_argument("--model", default="vits14")
    p.add_argument("--steps", type=int, default=1)
    p.add_argument("--graphs", type=int, default=1)
    a = p.parse_args()
    eng = VPEngine(a.model, a.resolution, a.batch, graphs=bool(a.graphs))
    for _ in range(3):
        eng.submit()
    eng.synchronize()
    torch.cuda.nvtx.range_push("prof")
    for _ in range(a.steps):
        eng.submit()
    eng.synchronize()
    torch.cuda.nvtx.range_pop()
    eng.close()


if __name__ == "__main__":
    main()
