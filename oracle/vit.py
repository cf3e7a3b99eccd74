"""fp32 CPU restatement of the DINOv2 backbone forward (TEST INFRASTRUCTURE).

Follows transformers 5.5.0 (third-party; the reference ships no NN code,
SURVEY §0.5 / §8c):
  preprocess      ImageNet mean/std on u8/255
  patch embed     modeling_dinov2.py:139-149  (Conv2d k=s=14)
  cls + pos       modeling_dinov2.py:97-116   (cat then add)
  pos interp      modeling_dinov2.py:57-95    (bicubic, align_corners=False)
  block           modeling_dinov2.py:348-386  (pre-LN, LayerScale, residual)
  self-attention  modeling_dinov2.py:153-178, 196-229 (scale 1/sqrt(64))
  MLP             modeling_dinov2.py:312-328  (exact-erf GELU)
  taps            modeling_dinov2.py:605-618  (final LN applied per tap)
Pinned against ``Dinov2Backbone`` in tests/test_oracle_pin.py.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F

MEAN = torch.tensor([0.485, 0.456, 0.406]).view(1, 3, 1, 1)
STD = torch.tensor([0.229, 0.224, 0.225]).view(1, 3, 1, 1)


def preprocess(frames_u8: torch.Tensor) -> torch.Tensor:
    return (frames_u8.float() / 255.0 - MEAN) / STD


def interpolate_pos(pos: torch.Tensor, h: int, w: int) -> torch.Tensor:
    """modeling_dinov2.py:57-95. pos: [1, 1+G*G, D] -> [1, 1+h*w, D]."""
    n = pos.shape[1] - 1
    g = int(math.sqrt(n))
    if g == h and g == w:
        return pos
    cls_pos, patch_pos = pos[:, :1], pos[:, 1:]
    d = pos.shape[-1]
    patch_pos = patch_pos.reshape(1, g, g, d).permute(0, 3, 1, 2)
    patch_pos = F.interpolate(patch_pos.float(), size=(h, w), mode="bicubic", align_corners=False)
    patch_pos = patch_pos.permute(0, 2, 3, 1).reshape(1, -1, d)
    return torch.cat([cls_pos, patch_pos], dim=1)


def layer_norm(x, w, b, eps):
    return F.layer_norm(x, (x.shape[-1],), w, b, eps)


def block(h: torch.Tensor, W: dict, i: int, heads: int, eps: float) -> torch.Tensor:
    """One Dinov2Layer (modeling_dinov2.py:348-386)."""
    p = f"encoder.layer.{i}."
    B, T, D = h.shape
    hd = D // heads
    x = layer_norm(h, W[p + "norm1.weight"], W[p + "norm1.bias"], eps)
    a = p + "attention.attention."
    q = F.linear(x, W[a + "query.weight"], W[a + "query.bias"]).view(B, T, heads, hd).transpose(1, 2)
    k = F.linear(x, W[a + "key.weight"], W[a + "key.bias"]).view(B, T, heads, hd).transpose(1, 2)
    v = F.linear(x, W[a + "value.weight"], W[a + "value.bias"]).view(B, T, heads, hd).transpose(1, 2)
    s = torch.matmul(q, k.transpose(-1, -2)) * (hd ** -0.5)
    ctx = torch.matmul(torch.softmax(s, dim=-1), v).transpose(1, 2).reshape(B, T, D)
    o = F.linear(ctx, W[p + "attention.output.dense.weight"], W[p + "attention.output.dense.bias"])
    h = h + o * W[p + "layer_scale1.lambda1"]
    x = layer_norm(h, W[p + "norm2.weight"], W[p + "norm2.bias"], eps)
    m = F.gelu(F.linear(x, W[p + "mlp.fc1.weight"], W[p + "mlp.fc1.bias"]))
    m = F.linear(m, W[p + "mlp.fc2.weight"], W[p + "mlp.fc2.bias"])
    return h + m * W[p + "layer_scale2.lambda1"]


def embed(frames_u8: torch.Tensor, W: dict) -> torch.Tensor:
    """preprocess + patch conv + cls + interpolated pos -> [B, T, D] fp32. A floating-point input
    is taken as already normalised (camera ingest: oracle/camera.py camera_preprocess)."""
    x = frames_u8 if frames_u8.is_floating_point() else preprocess(frames_u8)
    B, _, R, _ = x.shape
    e = F.conv2d(x, W["embeddings.patch_embeddings.projection.weight"],
                 W["embeddings.patch_embeddings.projection.bias"], stride=14)
    h = e.shape[-1]
    e = e.flatten(2).transpose(1, 2)
    cls = W["embeddings.cls_token"].expand(B, -1, -1)
    t = torch.cat([cls, e], dim=1)
    return t + interpolate_pos(W["embeddings.position_embeddings"], h, h)


@torch.no_grad()
def backbone_forward(frames_u8: torch.Tensor, W: dict, depth: int, heads: int,
                     taps: tuple[int, ...], eps: float = 1e-6,
                     return_hidden: bool = False):
    """Returns the tap features (each final-LN'd, [B,T,D] fp32) in tap order."""
    h = embed(frames_u8, W)
    outs, hidden = [], [h]
    for i in range(depth):
        h = block(h, W, i, heads, eps)
        hidden.append(h)
        if (i + 1) in taps:
            outs.append(layer_norm(h, W["layernorm.weight"], W["layernorm.bias"], eps))
    if return_hidden:
        return outs, hidden
    return outs
