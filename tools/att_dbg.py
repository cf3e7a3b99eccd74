import os, sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch
from paper_2508_11584_b200 import _ops
for (B, T, H) in [(1, 128, 2), (1, 257, 6), (3, 200, 4), (1, 1025, 6)] + ([(16, 1025, 6)] if os.environ.get("BIG") else []):
    D = H * 64
    g = torch.Generator().manual_seed(T + B)
    qkv = torch.randn(B * T, 3 * D, generator=g).to("cuda", torch.bfloat16)
    out = _ops.attention(qkv, B, T, D, H)
    torch.cuda.synchronize()
    q, k, v = qkv.float().view(B, T, 3, H, 64).permute(2, 0, 3, 1, 4)
    ref = (torch.softmax(q @ k.transpose(-1, -2) / 8.0, -1) @ v).transpose(1, 2).reshape(B * T, D)
    err = ((out.float() - ref).norm() / ref.norm()).item()
    # per 128-row q tile / per head error map to locate the damage
    e = (out.float() - ref).view(B, T, H, 64).norm(dim=-1) / ref.view(B, T, H, 64).norm(dim=-1)
    rows_bad = (e > 0.02).nonzero()
    print(json.dumps(dict(dbg=os.environ.get("VPE_ATT_DBG", "0"), B=B, T=T, H=H, rel=err, bad_rows=int(rows_bad.shape[0]),
                          first_bad=rows_bad[:5].tolist())), flush=True)
