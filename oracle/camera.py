"""fp32 CPU restatement of the camera ingest transform (TEST INFRASTRUCTURE).

SURVEY §8f row 2 ("pre-processing
transformations that normalize inputs for the foundation model"). The reference ships the
NormalizeAffine / CastDType / Reshape adapters but no resize, so the resize semantics are
defined here and mirrored by csrc/misc.cu camera_im2col_kernel:

  u8 HWC frame [H, W, 3]
  -> centre crop to S = min(H, W) (offsets (H-S)//2, (W-S)//2)
  -> torch F.interpolate(size=(R, R), mode="bilinear", align_corners=False, antialias=False)
  -> ImageNet normalisation (u/255 - mean) / std            (oracle/vit.py preprocess)
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

from .vit import MEAN, STD


def camera_preprocess(frames_hwc_u8: torch.Tensor, R: int) -> torch.Tensor:
    """[B, H, W, 3] u8 -> normalised fp32 [B, 3, R, R]."""
    B, H, W, _ = frames_hwc_u8.shape
    S = min(H, W)
    oy, ox = (H - S) // 2, (W - S) // 2
    x = frames_hwc_u8[:, oy:oy + S, ox:ox + S, :].permute(0, 3, 1, 2).float()
    x = F.interpolate(x, size=(R, R), mode="bilinear", align_corners=False, antialias=False)
    return (x / 255.0 - MEAN) / STD


def patch_rows(x: torch.Tensor, kp: int = 640) -> torch.Tensor:
    """[B, 3, R, R] -> im2col rows [B*(R/14)^2, kp] with k = c*196 + ky*14 + kx (zero padded)."""
    B, C, R, _ = x.shape
    h = R // 14
    p = x.reshape(B, C, h, 14, h, 14).permute(0, 2, 4, 1, 3, 5).reshape(B * h * h, C * 196)
    return F.pad(p, (0, kp - C * 196))
