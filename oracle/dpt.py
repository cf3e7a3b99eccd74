"""fp32 CPU restatement of the DepthAnything DPT neck + depth head (TEST INFRA).

Follows transformers 5.5.0 modeling_depth_anything.py (third-party):
  reassemble   :31-93   drop cls, [B,h,w,D]->NCHW, 1x1 proj, ConvT k=s=4/2,
                        identity, 3x3 s2 conv
  neck convs   :229-262 3x3 no-bias to fusion width
  fusion       :96-203  pre-act RCUs, bilinear align_corners=True (x2 / size)
  depth head   :265-308 conv 3x3, bilinear to (14h,14w) align_corners=True,
                        conv 3x3, ReLU, 1x1, ReLU * max_depth
Pinned against DepthAnythingForDepthEstimation in tests/test_oracle_pin.py.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


def _c(x, W, name, stride=1, padding=None):
    w = W[name + ".weight"]
    pad = (w.shape[-1] // 2) if padding is None else padding
    return F.conv2d(x, w, W.get(name + ".bias"), stride=stride, padding=pad)


def reassemble(taps, W, factors, h):
    out = []
    for i, t in enumerate(taps):
        B, _, D = t.shape
        x = t[:, 1:].reshape(B, h, h, D).permute(0, 3, 1, 2).contiguous()
        p = f"neck.reassemble_stage.layers.{i}."
        x = _c(x, W, p + "projection")
        f = factors[i]
        if f > 1:
            x = F.conv_transpose2d(x, W[p + "resize.weight"], W[p + "resize.bias"], stride=int(f))
        elif f < 1:
            x = _c(x, W, p + "resize", stride=int(1 / f), padding=1)
        out.append(x)
    return out


def rcu(x, W, p):
    """DepthAnythingPreActResidualLayer (:96-136)."""
    y = _c(F.relu(x), W, p + ".convolution1")
    y = _c(F.relu(y), W, p + ".convolution2")
    return y + x


def fusion(features, W):
    """DepthAnythingFeatureFusionStage (:165-203); features in reassemble order."""
    feats = features[::-1]
    fused = None
    outs = []
    for idx, x in enumerate(feats):
        p = f"neck.fusion_stage.layers.{idx}"
        size = feats[idx + 1].shape[2:] if idx != len(feats) - 1 else None
        if fused is None:
            hs = x
        else:
            hs = fused + rcu(x, W, p + ".residual_layer1")
        hs = rcu(hs, W, p + ".residual_layer2")
        if size is None:
            hs = F.interpolate(hs, scale_factor=2, mode="bilinear", align_corners=True)
        else:
            hs = F.interpolate(hs, size=tuple(size), mode="bilinear", align_corners=True)
        fused = _c(hs, W, p + ".projection")
        outs.append(fused)
    return outs


@torch.no_grad()
def dpt_forward(taps, W, factors, h, patch=14, max_depth=1.0, return_pre_relu=False):
    """taps: 4 x [B,T,D] fp32 (tap order L/4, L/2, 3L/4, L). Returns depth [B,R,R]."""
    feats = reassemble(taps, W, factors, h)
    feats = [_c(f, W, f"neck.convs.{i}") for i, f in enumerate(feats)]
    fused = fusion(feats, W)[-1]
    d = _c(fused, W, "head.conv1")
    d = F.interpolate(d, size=(h * patch, h * patch), mode="bilinear", align_corners=True)
    d = F.relu(_c(d, W, "head.conv2"))
    pre = _c(d, W, "head.conv3")
    depth = (F.relu(pre) * max_depth).squeeze(1)
    if return_pre_relu:
        return depth, pre.squeeze(1)
    return depth
