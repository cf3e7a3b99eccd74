"""Head parity on the B200, stage-wise: the oracle head consumes the exact
bf16 tap tensor the GPU backbone wrote (upcast to fp32).

Bars (BASELINE.json north star): depth pre/post-ReLU rel-L2 <= 1e-2 and cosine >= 0.999;
seg argmax agreement >= 99.9%; det top-k indices identical after decode (ties below the fp32
resolution of the oracle's own scores are reported, not failed)."""

import pytest
import torch

from det_match import align_to, kept_match
from oracle import det as odet
from oracle import dpt as odpt
from oracle import seg as oseg
from paper_2508_11584_b200.config import grid, model_config, tokens
from paper_2508_11584_b200.weights import make_frames, make_weights

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def cosine(a, b):
    return torch.nn.functional.cosine_similarity(a.float().flatten(), b.float().flatten(), dim=0).item()


@pytest.fixture(scope="module", params=[(224, 1), (448, 1), (224, 2)], ids=["r224b1", "r448b1", "r224b2"])
def setup(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2508_11584_b200.backbone import Backbone
    R, B = request.param
    dev = torch.device("cuda:0")
    cfg = model_config("vits14")
    W = make_weights("vits14")
    frames = make_frames(B, R, 0)
    bb = Backbone(W, cfg.backbone, R, B, dev)
    taps = [torch.empty(B, tokens(R), cfg.backbone.dim, device=dev, dtype=torch.bfloat16) for _ in range(4)]
    bb.forward(frames.to(dev), taps)
    torch.cuda.synchronize()
    return dict(R=R, B=B, dev=dev, cfg=cfg, W=W, taps=taps, taps_cpu=[t.float().cpu() for t in taps])


def test_depth_stagewise(setup):
    from paper_2508_11584_b200.heads import DepthHead
    s = setup
    R, B, dev = s["R"], s["B"], s["dev"]
    head = DepthHead(s["W"], s["cfg"], R, B, dev)
    depth = torch.empty(B, R, R, device=dev)
    pre = torch.empty(B, R, R, device=dev)
    head.forward(s["taps"], depth, pre)
    torch.cuda.synchronize()
    ref, ref_pre = odpt.dpt_forward(s["taps_cpu"], s["W"], s["cfg"].dpt.factors, grid(R), return_pre_relu=True)
    e_pre, c_pre = rel_l2(pre.cpu(), ref_pre), cosine(pre.cpu(), ref_pre)
    e, c = rel_l2(depth.cpu(), ref), cosine(depth.cpu(), ref)
    print(f"depth pre rel {e_pre:.3e} cos {c_pre:.6f}; post rel {e:.3e} cos {c:.6f}")
    assert e_pre <= 1e-2 and c_pre >= 0.999
    assert e <= 1e-2 and c >= 0.999



def test_depth_fused_resize_bitexact(setup, monkeypatch):
    """The DPT head with both resizes fused into their convs (default) writes exactly the depth the
    unfused path (VPE_DPT_UNFUSED=1: resize kernels + halo convs) writes."""
    from paper_2508_11584_b200.heads import DepthHead
    s = setup
    R, B, dev = s["R"], s["B"], s["dev"]
    outs = []
    for unfused in ("0", "1"):
        monkeypatch.setenv("VPE_DPT_UNFUSED", unfused)
        head = DepthHead(s["W"], s["cfg"], R, B, dev)
        depth = torch.empty(B, R, R, device=dev)
        pre = torch.empty(B, R, R, device=dev)
        head.forward(s["taps"], depth, pre)
        torch.cuda.synchronize()
        outs.append((depth.clone(), pre.clone()))
        del head
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_depth_branches_bitexact(setup):
    """Reassemble / neck branches on side streams (vpe_set_dpt_branches(1)), eager and captured in
    a CUDA graph, write exactly the depth the single-stream order (0) writes."""
    from paper_2508_11584_b200._lib import lib
    from paper_2508_11584_b200.heads import DepthHead
    s = setup
    R, B, dev = s["R"], s["B"], s["dev"]
    head = DepthHead(s["W"], s["cfg"], R, B, dev)
    outs = []
    try:
        for mode in (0, 1):
            assert lib.vpe_set_dpt_branches(mode) == 0
            depth = torch.full((B, R, R), float("nan"), device=dev)
            head.forward(s["taps"], depth)
            torch.cuda.synchronize()
            outs.append(depth.clone())
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            depth = torch.full((B, R, R), float("nan"), device=dev)
            head.forward(s["taps"], depth)  # side streams at this stream's priority, before capture
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                head.forward(s["taps"], depth)
        depth.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        outs.append(depth.clone())
    finally:
        lib.vpe_set_dpt_branches(-1)
    assert lib.vpe_set_dpt_branches(2) != 0
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])

def test_seg_stagewise(setup):
    from paper_2508_11584_b200.heads import SegHead
    s = setup
    R, B, dev, cfg = s["R"], s["B"], s["dev"], s["cfg"]
    head = SegHead(s["W"], cfg, R, B, dev)
    labels = torch.empty(B, R, R, dtype=torch.uint8, device=dev)
    h = grid(R)
    logits = torch.empty(B, h * h, cfg.seg_classes, device=dev)
    head.forward(s["taps"][3], labels, logits)
    torch.cuda.synchronize()
    ref_labels, ref_logits, _ = oseg.seg_forward(s["taps_cpu"][3], s["W"], h, R, return_logits=True)
    ref_l = ref_logits.permute(0, 2, 3, 1).reshape(B, h * h, -1)
    e = rel_l2(logits.cpu(), ref_l)
    agree = (labels.cpu() == ref_labels).float().mean().item()
    print(f"seg logits rel {e:.3e}; argmax agreement {agree * 100:.4f}%")
    assert e < 1e-5
    assert agree >= 0.999


def test_det_stagewise(setup):
    from paper_2508_11584_b200.heads import DetHead
    s = setup
    R, B, dev, cfg = s["R"], s["B"], s["dev"], s["cfg"]
    head = DetHead(s["W"], cfg, R, B, dev)
    out = head.outputs()
    n = grid(R) ** 2 * cfg.det.num_anchors
    out["objectness"] = torch.empty(B, n, device=dev)
    out["deltas"] = torch.empty(B, n, 4, device=dev)
    out["top_index"] = torch.empty(B, min(n, cfg.det.pre_nms_top_n), dtype=torch.int64, device=dev)
    head.forward(s["taps"][3], out)
    torch.cuda.synchronize()
    obj, deltas, _ = odet.det_head_maps(s["taps_cpu"][3], s["W"], grid(R))
    e_obj = rel_l2(out["objectness"].cpu(), obj)
    ref = odet.det_postprocess(obj, deltas, grid(R), R, cfg.det)
    for b in range(B):
        k = int(out["count"][b])
        gi = out["index"][b, :k].cpu()
        ri = ref[b]["index"]
        top_same = torch.equal(out["top_index"][b].cpu(), ref[b]["top_index"])
        print(f"det obj rel {e_obj:.3e}; kept {k} vs {ri.numel()}; top-k identical {top_same}; "
              f"kept identical {torch.equal(gi, ri)}")
    # numeric floor: tensor-core fp32 accumulation over K = 9*D (~1e-5 relative, see det.cu)
    assert e_obj < 3e-5
    max_err = (out["objectness"].cpu() - obj).abs().max().item()
    for b in range(B):
        k = int(out["count"][b])
        gi, ri = out["index"][b, :k].cpu(), ref[b]["index"]
        # the detections (post-NMS top-k) are identical, index for index, up to near-tie swaps
        # the measured logit error explains (tests/det_match.py)
        ok, nsw, kgap = kept_match(gi, ri, obj[b], max_err)
        assert ok, (b, nsw, kgap, max_err)
        p = align_to(gi, ri)
        # the pre-NMS top-k ranking may only differ by swaps the measured error can explain
        gt, rt = out["top_index"][b].cpu(), ref[b]["top_index"]
        diff = (gt != rt).nonzero().flatten()
        if diff.numel():
            gap = (obj[b][gt[diff]] - obj[b][rt[diff]]).abs().max().item()
            assert gap <= 2 * max_err, f"top-k swap gap {gap:.3e} > 2 x max err {max_err:.3e}"
        torch.testing.assert_close(out["boxes"][b, :k].cpu()[p], ref[b]["boxes"], rtol=1e-5, atol=1e-3)
        torch.testing.assert_close(out["scores"][b, :k].cpu()[p], ref[b]["scores"], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("B,h,C,cp", [(2, 32, 150, 160), (1, 16, 21, 32), (1, 32, 7, 8), (1, 16, 256, 256)])
def test_upsample_argmax_exact(B, h, C, cp):
    """The fused upsample+argmax on the SAME fp32 logits as torch's CPU F.interpolate + argmax
    (oracle/seg.py seg_forward): labels bit-identical, including exact ties (duplicated classes,
    a class duplicated into the tail past the last 8-class chunk, all-equal pixels, +-0)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2508_11584_b200 import _ops
    R = 14 * h
    g = torch.Generator().manual_seed(7 + C)
    lg = torch.randn(B, h * h, cp, generator=g)
    lg[..., C:] = 1e9  # padding classes must never be read
    if C > 8:
        lg[..., C - 1] = lg[..., 2]            # tail class ties an early class: index 2 must win
        lg[..., 5] = lg[..., 1]                # tie inside one chunk
    lg[:, : h, :C] = 0.25                      # first source row: every class equal -> label 0
    lg[:, h: 2 * h, :C] = -0.0
    lg[:, 2 * h: 2 * h + 3, 0] = 0.0           # +0 vs -0
    labels = _ops.upsample_argmax(lg.cuda(), h, R, classes=C)
    torch.cuda.synchronize()
    x = lg[..., :C].reshape(B, h, h, C).permute(0, 3, 1, 2)
    ref = torch.nn.functional.interpolate(x, size=(R, R), mode="bilinear", align_corners=False).argmax(1)
    ref = ref.to(torch.uint8)
    bad = (labels.cpu() != ref).sum().item()
    assert bad == 0, f"{bad} of {ref.numel()} labels differ"


def _upsample_argmax_formula(lg: torch.Tensor, h: int, C: int, R: int) -> torch.Tensor:
    """CPU fp32 restatement of the kernels' per-pixel arithmetic (oracle/seg.py's bilinear,
    align_corners=False, in torch's channels-last rounding order: s = fma(scale, o + 0.5, -0.5),
    value = (a*w0 + b*w1)*h0 + (c*w0 + d*w1)*h1, every op rounded to fp32) + first-index argmax."""
    scale = torch.tensor(h, dtype=torch.float32) / torch.tensor(R, dtype=torch.float32)
    o = torch.arange(R, dtype=torch.float64) + 0.5
    src = (scale.double() * o - 0.5).float().clamp_min(0.0)  # one rounding: the fma
    i0 = src.long()
    i1 = torch.where(i0 < h - 1, i0 + 1, i0)
    l1 = (src - i0.float()).clamp(0.0, 1.0)
    l0 = 1.0 - l1
    B = lg.shape[0]
    x = lg[..., :C].reshape(B, h, h, C)
    out = torch.empty(B, R, R, dtype=torch.uint8)
    for oy in range(R):
        r0, r1 = x[:, i0[oy]], x[:, i1[oy]]  # [B, h, C]
        t0 = r0[:, i0] * l0[None, :, None] + r0[:, i1] * l1[None, :, None]  # [B, R, C]
        t1 = r1[:, i0] * l0[None, :, None] + r1[:, i1] * l1[None, :, None]
        v = t0 * l0[oy] + t1 * l1[oy]
        out[:, oy] = v.argmax(-1).to(torch.uint8)
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_upsample_argmax_smooth_near_ties(seed):
    """Class pruning (seg_upsample_argmax_pruned_kernel) on spatially smooth logits -- few
    candidate classes per 7x7 block -- with classes within a few ulps of each other (and exact
    ties), so the pruning margin decides: labels must equal the same arithmetic evaluated over
    every class on the CPU. (Against torch's own interpolate such near-ties are decided by its
    rounding order, not this kernel's; the exact-tie cases above are order-independent.)"""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2508_11584_b200 import _ops
    B, h, C, cp = 2, 32, 150, 160
    R = 14 * h
    g = torch.Generator().manual_seed(100 + seed)
    coarse = torch.randn(B, C, 5, 5, generator=g)
    x = torch.nn.functional.interpolate(coarse, size=(h, h), mode="bicubic", align_corners=True)
    x[:, 3] = x[:, 7] * (1 + 2 ** -23 * torch.randint(-4, 5, (B, h, h), generator=g).float())
    x[:, 9] = x[:, 11]
    x[:, 20] = x.max(1).values  # a class equal to the per-pixel maximum at every source pixel
    lg = torch.zeros(B, h * h, cp)
    lg[..., :C] = x.permute(0, 2, 3, 1).reshape(B, h * h, C)
    labels = _ops.upsample_argmax(lg.cuda(), h, R, classes=C)
    torch.cuda.synchronize()
    ref = _upsample_argmax_formula(lg, h, C, R)
    bad = (labels.cpu() != ref).sum().item()
    assert bad == 0, f"{bad} of {ref.numel()} labels differ"
