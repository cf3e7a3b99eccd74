"""fp32 CPU restatement of the DINOv2 "linear" segmentation head (TEST INFRA).

No third-party implementation exists in the image; the
head is defined by the paper ("linear layer for semantic segmentation
[DINOv2]") and restated exactly as SURVEY §8a A18 specifies:
BatchNorm2d(D) in eval mode + Conv2d(D, C, 1) on the final patch map,
bilinear upsample to (R, R) with align_corners=False, argmax over classes.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


@torch.no_grad()
def seg_logits(final: torch.Tensor, W: dict, h: int, eps: float = 1e-5) -> torch.Tensor:
    """final: [B,T,D] -> low-res logits [B,C,h,h] fp32."""
    B, _, D = final.shape
    x = final[:, 1:].reshape(B, h, h, D).permute(0, 3, 1, 2)
    x = F.batch_norm(x, W["seg.bn.running_mean"], W["seg.bn.running_var"],
                     W["seg.bn.weight"], W["seg.bn.bias"], training=False, eps=eps)
    return F.conv2d(x, W["seg.classifier.weight"], W["seg.classifier.bias"])


@torch.no_grad()
def seg_forward(final: torch.Tensor, W: dict, h: int, resolution: int, eps: float = 1e-5,
                return_logits: bool = False):
    logits = seg_logits(final, W, h, eps)
    up = F.interpolate(logits, size=(resolution, resolution), mode="bilinear", align_corners=False)
    labels = up.argmax(1).to(torch.uint8)
    if return_logits:
        return labels, logits, up
    return labels
