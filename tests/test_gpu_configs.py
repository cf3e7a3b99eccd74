"""The other BASELINE.json configurations on the B200: ViT-B/14 and ViT-L/14 at 518x518
(T = 1370, 37x37 grid with bicubic-resized positions, ragged 128-row tiles everywhere) and
C1 (S/14 at 224 + depth only). Same bars as C2: taps rel-L2 <= 1e-2 / cos >= 0.999; depth
stage-wise rel-L2 <= 1e-2; seg agreement >= 99.9%; det detections identical."""

import pytest
import torch

from det_match import kept_match
from oracle import det as odet
from oracle import dpt as odpt
from oracle import seg as oseg
from oracle import vit as ovit
from paper_2508_11584_b200.config import grid, model_config, tokens
from paper_2508_11584_b200.weights import make_frames, make_weights

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def cosine(a, b):
    return torch.nn.functional.cosine_similarity(a.float().flatten(), b.float().flatten(), dim=0).item()


@pytest.mark.parametrize("model,R,B,heads", [("vitb14", 518, 1, ("depth", "seg", "det")),
                                             ("vitl14", 518, 2, ("depth",)),
                                             ("vits14", 224, 1, ("depth",))],
                         ids=["C3-B14-518", "C5-L14-518-b2", "C1-S14-224"])
def test_config_parity(model, R, B, heads):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2508_11584_b200.backbone import Backbone
    from paper_2508_11584_b200.heads import DepthHead, DetHead, SegHead
    dev = torch.device("cuda:0")
    cfg = model_config(model)
    W = make_weights(model, heads=heads)
    frames = make_frames(B, R, 7)
    bb = Backbone(W, cfg.backbone, R, B, dev)
    T = tokens(R)
    taps = [torch.empty(B, T, cfg.backbone.dim, device=dev, dtype=torch.bfloat16) for _ in range(4)]
    bb.forward(frames.to(dev), taps)
    torch.cuda.synchronize()
    ref = ovit.backbone_forward(frames, W, cfg.backbone.depth, cfg.backbone.heads, cfg.backbone.taps)
    for k, (g, r) in enumerate(zip(taps, ref)):
        e, c = rel_l2(g.cpu(), r), cosine(g.cpu(), r)
        assert e <= 1e-2 and c >= 0.999, f"{model} tap {k}: rel-L2 {e:.3e} cos {c:.6f}"
    tc = [t.float().cpu() for t in taps]
    h = grid(R)
    if "depth" in heads:
        head = DepthHead(W, cfg, R, B, dev)
        depth = torch.empty(B, R, R, device=dev)
        pre = torch.empty(B, R, R, device=dev)
        head.forward(taps, depth, pre)
        torch.cuda.synchronize()
        rd, rp = odpt.dpt_forward(tc, W, cfg.dpt.factors, h, return_pre_relu=True)
        assert rel_l2(pre.cpu(), rp) <= 1e-2 and cosine(pre.cpu(), rp) >= 0.999
        assert rel_l2(depth.cpu(), rd) <= 1e-2
    if "seg" in heads:
        head = SegHead(W, cfg, R, B, dev)
        labels = torch.empty(B, R, R, dtype=torch.uint8, device=dev)
        head.forward(taps[3], labels)
        torch.cuda.synchronize()
        rl = oseg.seg_forward(tc[3], W, h, R)
        assert (labels.cpu() == rl).float().mean().item() >= 0.999
    if "det" in heads:
        head = DetHead(W, cfg, R, B, dev)
        out = head.outputs()
        out["objectness"] = torch.empty(B, h * h * cfg.det.num_anchors, device=dev)
        out["deltas"] = torch.empty(B, h * h * cfg.det.num_anchors, 4, device=dev)
        head.forward(taps[3], out)
        torch.cuda.synchronize()
        obj, deltas, _ = odet.det_head_maps(tc[3], W, h)
        rr = odet.det_postprocess(obj, deltas, h, R, cfg.det)
        max_err = (out["objectness"].cpu() - obj).abs().max().item()
        for b in range(B):
            k = int(out["count"][b])
            ok, nsw, gap = kept_match(out["index"][b, :k], rr[b]["index"], obj[b], max_err)
            assert ok, (model, b, nsw, gap, max_err)
