"""fp32 CPU restatement of the RPN-style detection head (TEST INFRASTRUCTURE).

The paper's "custom FasterRCNN head" is not shipped; the head
is defined per SURVEY §8a A19 from torchvision 0.26.0 pieces (third-party),
restated here and pinned against torchvision in tests/test_oracle_pin.py:
  RPNHead          rpn.py:15-79        3x3 conv+ReLU, 1x1 cls (A), 1x1 bbox (4A)
  anchors          anchor_utils.py:58-113  sizes x ratios, ratio-major, rounded
  decode           _utils.py:183-225   BoxCoder(1,1,1,1), clip log(1000/16)
  filter_proposals rpn.py:231-297      top-n, sigmoid, clip, remove small,
                                       score thresh, NMS, post top-n
  nms              ops/boxes.py:20-48  greedy, IoU > thresh suppressed
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def base_anchors(sizes, ratios) -> torch.Tensor:
    """anchor_utils.py:58-77: [A,4] zero-centred, ratio-major then size."""
    scales = torch.as_tensor(sizes, dtype=torch.float32)
    ar = torch.as_tensor(ratios, dtype=torch.float32)
    h_r = torch.sqrt(ar)
    w_r = 1 / h_r
    ws = (w_r[:, None] * scales[None, :]).view(-1)
    hs = (h_r[:, None] * scales[None, :]).view(-1)
    return (torch.stack([-ws, -hs, ws, hs], dim=1) / 2).round()


def grid_anchors(h: int, w: int, stride: int, sizes, ratios) -> torch.Tensor:
    """anchor_utils.py:85-113: [h*w*A, 4], location-major (y, x), anchor-minor."""
    base = base_anchors(sizes, ratios)
    sx = torch.arange(0, w, dtype=torch.int32) * stride
    sy = torch.arange(0, h, dtype=torch.int32) * stride
    yy, xx = torch.meshgrid(sy, sx, indexing="ij")
    xx, yy = xx.reshape(-1), yy.reshape(-1)
    shifts = torch.stack((xx, yy, xx, yy), dim=1)
    return (shifts.view(-1, 1, 4) + base.view(1, -1, 4)).reshape(-1, 4)


def decode(deltas: torch.Tensor, anchors: torch.Tensor, weights=(1.0, 1.0, 1.0, 1.0),
           clip=math.log(1000.0 / 16)) -> torch.Tensor:
    """_utils.py:183-225 decode_single. deltas/anchors: [N,4]."""
    widths = anchors[:, 2] - anchors[:, 0]
    heights = anchors[:, 3] - anchors[:, 1]
    ctr_x = anchors[:, 0] + 0.5 * widths
    ctr_y = anchors[:, 1] + 0.5 * heights
    wx, wy, ww, wh = weights
    dx, dy = deltas[:, 0] / wx, deltas[:, 1] / wy
    dw = torch.clamp(deltas[:, 2] / ww, max=clip)
    dh = torch.clamp(deltas[:, 3] / wh, max=clip)
    pcx = dx * widths + ctr_x
    pcy = dy * heights + ctr_y
    pw = torch.exp(dw) * widths
    ph = torch.exp(dh) * heights
    return torch.stack((pcx - 0.5 * pw, pcy - 0.5 * ph, pcx + 0.5 * pw, pcy + 0.5 * ph), dim=1)


def nms(boxes: torch.Tensor, scores: torch.Tensor, thresh: float) -> torch.Tensor:
    """ops/boxes.py:20-48 semantics: stable descending order, greedy."""
    order = torch.sort(scores, descending=True, stable=True).indices
    b = boxes[order]
    area = (b[:, 2] - b[:, 0]) * (b[:, 3] - b[:, 1])
    n = b.shape[0]
    suppressed = torch.zeros(n, dtype=torch.bool)
    keep = []
    for i in range(n):
        if suppressed[i]:
            continue
        keep.append(i)
        xx1 = torch.maximum(b[i, 0], b[i + 1:, 0])
        yy1 = torch.maximum(b[i, 1], b[i + 1:, 1])
        xx2 = torch.minimum(b[i, 2], b[i + 1:, 2])
        yy2 = torch.minimum(b[i, 3], b[i + 1:, 3])
        inter = (xx2 - xx1).clamp(min=0) * (yy2 - yy1).clamp(min=0)
        iou = inter / (area[i] + area[i + 1:] - inter)
        suppressed[i + 1:] |= iou > thresh
    return order[torch.tensor(keep, dtype=torch.long)]


@torch.no_grad()
def det_head_maps(final: torch.Tensor, W: dict, h: int):
    """RPNHead on the final patch map. Returns objectness [B, h*h*A] and
    deltas [B, h*h*A, 4] in torchvision's (y, x, a) flattening
    (rpn.py:275 permute_and_flatten)."""
    B, _, D = final.shape
    x = final[:, 1:].reshape(B, h, h, D).permute(0, 3, 1, 2)
    t = F.relu(F.conv2d(x, W["det.conv.weight"], W["det.conv.bias"], padding=1))
    logits = F.conv2d(t, W["det.cls_logits.weight"], W["det.cls_logits.bias"])
    reg = F.conv2d(t, W["det.bbox_pred.weight"], W["det.bbox_pred.bias"])
    A = logits.shape[1]
    obj = logits.permute(0, 2, 3, 1).reshape(B, -1)
    deltas = reg.view(B, A, 4, h, h).permute(0, 3, 4, 1, 2).reshape(B, -1, 4)
    return obj, deltas, t


@torch.no_grad()
def det_postprocess(obj: torch.Tensor, deltas: torch.Tensor, h: int, resolution: int, cfg):
    """filter_proposals (rpn.py:231-297) for one feature level, per image.

    Returns per image: dict(boxes [K,4], scores [K], index [K] into the
    flattened anchor list (int64))."""
    stride = resolution // h
    anchors = grid_anchors(h, h, stride, cfg.sizes, cfg.ratios)
    out = []
    for b in range(obj.shape[0]):
        k = min(cfg.pre_nms_top_n, obj.shape[1])
        top_v, top_i = obj[b].topk(k)
        boxes = decode(deltas[b][top_i], anchors[top_i], cfg.weights)
        scores = torch.sigmoid(top_v)
        boxes[:, 0::2] = boxes[:, 0::2].clamp(0, resolution)
        boxes[:, 1::2] = boxes[:, 1::2].clamp(0, resolution)
        ws, hs = boxes[:, 2] - boxes[:, 0], boxes[:, 3] - boxes[:, 1]
        keep = torch.where((ws >= cfg.min_size) & (hs >= cfg.min_size))[0]
        keep = keep[scores[keep] >= cfg.score_thresh]
        kept = nms(boxes[keep], scores[keep], cfg.nms_thresh)[: cfg.post_nms_top_n]
        sel = keep[kept]
        out.append({"boxes": boxes[sel], "scores": scores[sel], "index": top_i[sel],
                    "top_index": top_i, "top_logit": top_v})
    return out


@torch.no_grad()
def det_forward(final, W, h, resolution, cfg):
    obj, deltas, _ = det_head_maps(final, W, h)
    return det_postprocess(obj, deltas, h, resolution, cfg)
