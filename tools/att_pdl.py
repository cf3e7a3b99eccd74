"""Diagnostics: QKV GEMM -> attention (PDL when VPE_OP_PDL=1 VPE_PDL=1), repeated; reports runs whose
attention output differs bitwise from the first."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200 import _ops

torch.manual_seed(0)
B, T, H = int(os.environ.get("B", "2")), 1025, 6
D = H * 64
x = torch.randn(B * T, D, device="cuda").to(torch.bfloat16)
w = (torch.randn(3 * D, D, device="cuda") * 0.05).to(torch.bfloat16)
qkv = torch.empty(B * T, 3 * D, device="cuda", dtype=torch.bfloat16)


def run():
    _ops.linear(x, w, out=qkv, bn=256)
    return _ops.attention(qkv, B, T, D, H)


if os.environ.get("GRAPH") == "1":
    out_holder = {}
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out_holder["o"] = run()
    eager = run

    def run():  # noqa: F811
        g.replay()
        return out_holder["o"]
ref = run().clone()
torch.cuda.synchronize()
bad = 0
for i in range(int(os.environ.get("REPS", "50"))):
    o = run()
    torch.cuda.synchronize()
    if not torch.equal(o, ref):
        bad += 1
        d = (o.float() - ref.float()).abs()
        if bad <= 3:
            rows = (d.amax(1) > 0).nonzero().flatten()
            print(f"run {i}: max {d.max().item():.3e}, rows {rows.numel()} first {rows[:8].tolist()}")
print("differing runs:", bad)
