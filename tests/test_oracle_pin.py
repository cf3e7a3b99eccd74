"""Pin the CPU oracle restatements against the pinned third-party
implementations they restate (transformers 5.5.0, torchvision 0.26.0).

The reference ships no NN code, so these pins — plus the frozen
golden fixtures — are what make the oracle trustworthy.
"""

import pytest
import torch

from oracle import det as odet
from oracle import dpt as odpt
from oracle import seg as oseg
from oracle import vit as ovit
from paper_2508_11584_b200.config import model_config
from paper_2508_11584_b200.weights import make_frames, make_weights

R = 224
H = R // 14


@pytest.fixture(scope="module")
def small():
    torch.manual_seed(0)
    cfg = model_config("vits14")
    W = make_weights("vits14")
    frames = make_frames(1, R, 0)
    taps = ovit.backbone_forward(frames, W, cfg.backbone.depth, cfg.backbone.heads, cfg.backbone.taps)
    return cfg, W, frames, taps


def test_backbone_matches_transformers(small):
    from transformers import Dinov2Backbone, Dinov2Config
    cfg, W, frames, taps = small
    bb = cfg.backbone
    hf = Dinov2Backbone(Dinov2Config(image_size=518, hidden_size=bb.dim, num_hidden_layers=bb.depth,
                                     num_attention_heads=bb.heads, out_indices=list(bb.taps),
                                     reshape_hidden_states=False, attn_implementation="eager"))
    sd = {k: v for k, v in W.items() if not k.startswith(("neck.", "head.", "seg.", "det."))}
    missing, unexpected = hf.load_state_dict(sd, strict=True), None
    hf.eval()
    with torch.no_grad():
        fm = hf(ovit.preprocess(frames)).feature_maps
    assert len(fm) == 4
    for a, b in zip(taps, fm):
        assert a.shape == b.shape
        torch.testing.assert_close(a, b, rtol=1e-4, atol=1e-4)


def test_dpt_matches_transformers(small):
    from transformers import DepthAnythingConfig, DepthAnythingForDepthEstimation
    cfg, W, frames, taps = small
    bb = cfg.backbone
    dac = DepthAnythingConfig(backbone_config=dict(model_type="dinov2", image_size=518, hidden_size=bb.dim,
                                                   num_hidden_layers=bb.depth, num_attention_heads=bb.heads,
                                                   out_indices=list(bb.taps), reshape_hidden_states=False),
                              reassemble_hidden_size=bb.dim, neck_hidden_sizes=list(cfg.dpt.neck),
                              fusion_hidden_size=cfg.dpt.fusion)
    hf = DepthAnythingForDepthEstimation(dac)
    sd = {}
    for k, v in W.items():
        if k.startswith(("neck.", "head.")):
            sd[k] = v
        elif not k.startswith(("seg.", "det.")):
            sd["backbone." + k] = v
    hf.load_state_dict(sd, strict=True)
    hf.eval()
    with torch.no_grad():
        ref = hf(ovit.preprocess(frames)).predicted_depth
    ours, pre = odpt.dpt_forward(taps, W, cfg.dpt.factors, H, return_pre_relu=True)
    torch.testing.assert_close(ours, ref, rtol=1e-4, atol=1e-5)
    assert (ours > 0).float().mean() > 0.5  # recipe keeps the map non-degenerate


def test_seg_restatement(small):
    cfg, W, frames, taps = small
    labels, logits, up = oseg.seg_forward(taps[-1], W, H, R, return_logits=True)
    # independent path: nn modules
    bn = torch.nn.BatchNorm2d(cfg.backbone.dim).eval()
    bn.load_state_dict({"weight": W["seg.bn.weight"], "bias": W["seg.bn.bias"],
                        "running_mean": W["seg.bn.running_mean"], "running_var": W["seg.bn.running_var"],
                        "num_batches_tracked": torch.tensor(0)})
    conv = torch.nn.Conv2d(cfg.backbone.dim, cfg.seg_classes, 1)
    conv.load_state_dict({"weight": W["seg.classifier.weight"], "bias": W["seg.classifier.bias"]})
    x = taps[-1][:, 1:].reshape(1, H, H, -1).permute(0, 3, 1, 2)
    with torch.no_grad():
        ref = conv(bn(x))
    torch.testing.assert_close(logits, ref, rtol=1e-5, atol=1e-5)
    assert labels.shape == (1, R, R) and labels.dtype == torch.uint8
    assert int(labels.max()) < cfg.seg_classes


def test_det_matches_torchvision(small):
    from torchvision.models.detection.anchor_utils import AnchorGenerator
    from torchvision.models.detection._utils import BoxCoder
    from torchvision.models.detection.image_list import ImageList
    from torchvision.models.detection.rpn import RPNHead
    from torchvision.ops import boxes as box_ops
    cfg, W, frames, taps = small
    dc = cfg.det
    # head maps vs RPNHead
    head = RPNHead(cfg.backbone.dim, dc.num_anchors)
    head.load_state_dict({"conv.0.0.weight": W["det.conv.weight"], "conv.0.0.bias": W["det.conv.bias"],
                          "cls_logits.weight": W["det.cls_logits.weight"], "cls_logits.bias": W["det.cls_logits.bias"],
                          "bbox_pred.weight": W["det.bbox_pred.weight"], "bbox_pred.bias": W["det.bbox_pred.bias"]})
    x = taps[-1][:, 1:].reshape(1, H, H, -1).permute(0, 3, 1, 2)
    with torch.no_grad():
        lg, rg = head([x])
    obj, deltas, _ = odet.det_head_maps(taps[-1], W, H)
    from torchvision.models.detection.rpn import concat_box_prediction_layers
    tv_obj, tv_reg = concat_box_prediction_layers(lg, rg)
    torch.testing.assert_close(obj.reshape(-1), tv_obj.reshape(-1), rtol=1e-5, atol=1e-6)
    torch.testing.assert_close(deltas.reshape(-1, 4), tv_reg, rtol=1e-5, atol=1e-6)
    # anchors vs AnchorGenerator
    ag = AnchorGenerator(sizes=(dc.sizes,), aspect_ratios=(dc.ratios,))
    il = ImageList(torch.zeros(1, 3, R, R), [(R, R)])
    tv_anchors = ag(il, [x])[0]
    ours = odet.grid_anchors(H, H, R // H, dc.sizes, dc.ratios)
    torch.testing.assert_close(ours, tv_anchors)
    # decode vs BoxCoder
    bc = BoxCoder(weights=dc.weights)
    torch.testing.assert_close(odet.decode(deltas[0], ours), bc.decode_single(deltas[0], tv_anchors))
    # nms vs torchvision nms on the actual candidate set
    res = odet.det_postprocess(obj, deltas, H, R, dc)[0]
    top_i = res["top_index"]
    boxes = bc.decode_single(deltas[0][top_i], tv_anchors[top_i])
    boxes = box_ops.clip_boxes_to_image(boxes, (R, R))
    scores = torch.sigmoid(res["top_logit"])
    keep = box_ops.remove_small_boxes(boxes, dc.min_size)
    tv_keep = box_ops.nms(boxes[keep], scores[keep], dc.nms_thresh)[: dc.post_nms_top_n]
    torch.testing.assert_close(top_i[keep[tv_keep]], res["index"])
    assert 0 < res["index"].numel() <= dc.post_nms_top_n
