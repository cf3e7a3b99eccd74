#!/bin/bash
# diagnostics: depth map with the row-staged vs gather bilinear kernels must be bit-identical
python - <<'PY'
import os, subprocess, torch
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2508_11584_b200.engine import VPEngine
from paper_2508_11584_b200.weights import make_frames
eng = VPEngine("vits14", 448, 2)
eng.pixels.copy_(make_frames(2, 448, 0).to(eng.device))
eng.submit(); eng.synchronize()
torch.save(eng.out["depth"]["depth"].cpu(), sys.argv[1])
'''
open("/tmp/_d.py", "w").write(code)
subprocess.run(["python", "/tmp/_d.py", "/tmp/d_rows.pt"], check=True)
env = dict(os.environ, **{os.environ.get("CMP_VAR", "VPE_BILINEAR_GATHER"): os.environ.get("CMP_VAL", "1")})
subprocess.run(["python", "/tmp/_d.py", "/tmp/d_gather.pt"], check=True, env=env)
a, b = torch.load("/tmp/d_rows.pt"), torch.load("/tmp/d_gather.pt")
print("bit-identical:", torch.equal(a, b), "max abs diff", (a - b).abs().max().item())
PY
