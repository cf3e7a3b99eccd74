"""Seeded random-init weights for the backbone and the three heads.

There is no network in this environment, so every run uses random-init
weights of the real architectures. The recipe is fixed here so
the GPU path and the CPU oracle always see identical fp32 parameters:

* backbone (generator seed ``seed``): HF DINOv2 init
  (``transformers/models/dinov2/modeling_dinov2.py:406-422``): trunc-normal
  std 0.02 for Linear / Conv / cls / pos. On top of that every affine term
  the fused epilogues consume is perturbed so parity tests exercise it:
  biases N(0, 0.02), LayerNorm gamma 1+N(0, 0.1) / beta N(0, 0.02),
  LayerScale U(0.5, 1.5).
* DPT depth head (seed+1): PyTorch default ``reset_parameters`` (uniform
  +-1/sqrt(fan_in)) for every Conv / ConvTranspose; ``head.conv3.bias`` is
  shifted by +0.1 so the post-ReLU depth map is not identically zero at
  random init.
* linear seg head (seed+2): BatchNorm2d eval stats mean N(0, 0.1),
  var U(0.5, 1.5), gamma N(1, 0.1), beta N(0, 0.1); 1x1 conv default init.
* RPN-style det head (seed+3): normal std 0.01, zero bias
  (``torchvision/models/detection/rpn.py:36-40``).

Names follow the HF / torchvision state-dict keys so the tensors load
directly into ``Dinov2Backbone`` / ``DepthAnythingForDepthEstimation`` for
pinning the oracle.
"""

from __future__ import annotations

import math

import torch

from .config import PATCH, POS_GRID, ModelConfig, model_config


def _tn(g: torch.Generator, *shape, std=0.02) -> torch.Tensor:
    t = torch.empty(*shape)
    torch.nn.init.trunc_normal_(t, mean=0.0, std=std, a=-2.0, b=2.0, generator=g)
    return t


def _n(g, *shape, mean=0.0, std=1.0) -> torch.Tensor:
    return torch.randn(*shape, generator=g) * std + mean


def _u(g, *shape, lo=0.0, hi=1.0) -> torch.Tensor:
    return torch.rand(*shape, generator=g) * (hi - lo) + lo


def backbone_weights(cfg: ModelConfig, seed: int = 0) -> dict[str, torch.Tensor]:
    bb = cfg.backbone
    D, Hd = bb.dim, bb.hidden
    g = torch.Generator().manual_seed(seed)
    W: dict[str, torch.Tensor] = {}
    p = "embeddings."
    W[p + "cls_token"] = _tn(g, 1, 1, D)
    W[p + "mask_token"] = torch.zeros(1, D)
    W[p + "position_embeddings"] = _tn(g, 1, POS_GRID * POS_GRID + 1, D)
    W[p + "patch_embeddings.projection.weight"] = _tn(g, D, 3, PATCH, PATCH)
    W[p + "patch_embeddings.projection.bias"] = _n(g, D, std=0.02)
    for i in range(bb.depth):
        p = f"encoder.layer.{i}."
        for ln in ("norm1", "norm2"):
            W[p + ln + ".weight"] = _n(g, D, mean=1.0, std=0.1)
            W[p + ln + ".bias"] = _n(g, D, std=0.02)
        for name in ("query", "key", "value"):
            W[p + f"attention.attention.{name}.weight"] = _tn(g, D, D)
            W[p + f"attention.attention.{name}.bias"] = _n(g, D, std=0.02)
        W[p + "attention.output.dense.weight"] = _tn(g, D, D)
        W[p + "attention.output.dense.bias"] = _n(g, D, std=0.02)
        W[p + "layer_scale1.lambda1"] = _u(g, D, lo=0.5, hi=1.5)
        W[p + "mlp.fc1.weight"] = _tn(g, Hd, D)
        W[p + "mlp.fc1.bias"] = _n(g, Hd, std=0.02)
        W[p + "mlp.fc2.weight"] = _tn(g, D, Hd)
        W[p + "mlp.fc2.bias"] = _n(g, D, std=0.02)
        W[p + "layer_scale2.lambda1"] = _u(g, D, lo=0.5, hi=1.5)
    W["layernorm.weight"] = _n(g, D, mean=1.0, std=0.1)
    W["layernorm.bias"] = _n(g, D, std=0.02)
    return W


def dpt_weights(cfg: ModelConfig, seed: int = 1) -> dict[str, torch.Tensor]:
    D = cfg.backbone.dim
    dp = cfg.dpt
    F = dp.fusion
    g = torch.Generator().manual_seed(seed)
    W: dict[str, torch.Tensor] = {}

    def conv(name, cout, cin, k, bias=True):
        bound = 1.0 / math.sqrt(cin * k * k)
        W[name + ".weight"] = _u(g, cout, cin, k, k, lo=-bound, hi=bound)
        if bias:
            W[name + ".bias"] = _u(g, cout, lo=-bound, hi=bound)

    def convT(name, cin, cout, k):
        # ConvTranspose2d weight is [in, out, k, k]; torch's fan_in uses dim 1.
        bound = 1.0 / math.sqrt(cout * k * k)
        W[name + ".weight"] = _u(g, cin, cout, k, k, lo=-bound, hi=bound)
        W[name + ".bias"] = _u(g, cout, lo=-bound, hi=bound)

    for i, (ch, f) in enumerate(zip(dp.neck, dp.factors)):
        p = f"neck.reassemble_stage.layers.{i}."
        conv(p + "projection", ch, D, 1)
        if f > 1:
            convT(p + "resize", ch, ch, int(f))
        elif f < 1:
            conv(p + "resize", ch, ch, 3)
    for i, ch in enumerate(dp.neck):
        conv(f"neck.convs.{i}", F, ch, 3, bias=False)
    for i in range(4):
        p = f"neck.fusion_stage.layers.{i}."
        conv(p + "projection", F, F, 1)
        for r in ("residual_layer1", "residual_layer2"):
            conv(p + r + ".convolution1", F, F, 3)
            conv(p + r + ".convolution2", F, F, 3)
    conv("head.conv1", F // 2, F, 3)
    conv("head.conv2", dp.head_hidden, F // 2, 3)
    conv("head.conv3", 1, dp.head_hidden, 1)
    W["head.conv3.bias"] = W["head.conv3.bias"] + 0.1
    return W


def seg_weights(cfg: ModelConfig, seed: int = 2) -> dict[str, torch.Tensor]:
    D, C = cfg.backbone.dim, cfg.seg_classes
    g = torch.Generator().manual_seed(seed)
    W = {
        "seg.bn.running_mean": _n(g, D, std=0.1),
        "seg.bn.running_var": _u(g, D, lo=0.5, hi=1.5),
        "seg.bn.weight": _n(g, D, mean=1.0, std=0.1),
        "seg.bn.bias": _n(g, D, std=0.1),
    }
    bound = 1.0 / math.sqrt(D)
    W["seg.classifier.weight"] = _u(g, C, D, 1, 1, lo=-bound, hi=bound)
    W["seg.classifier.bias"] = _u(g, C, lo=-bound, hi=bound)
    return W


def det_weights(cfg: ModelConfig, seed: int = 3) -> dict[str, torch.Tensor]:
    D, A = cfg.backbone.dim, cfg.det.num_anchors
    g = torch.Generator().manual_seed(seed)
    return {
        "det.conv.weight": _n(g, D, D, 3, 3, std=0.01),
        "det.conv.bias": torch.zeros(D),
        "det.cls_logits.weight": _n(g, A, D, 1, 1, std=0.01),
        "det.cls_logits.bias": torch.zeros(A),
        "det.bbox_pred.weight": _n(g, 4 * A, D, 1, 1, std=0.01),
        "det.bbox_pred.bias": torch.zeros(4 * A),
    }


def make_weights(name: str = "vits14", seed: int = 0, seg_classes: int = 150,
                 heads: tuple[str, ...] = ("depth", "seg", "det")) -> dict[str, torch.Tensor]:
    """Full canonical fp32 state dict (CPU) for backbone + requested heads."""
    cfg = model_config(name, seg_classes)
    W = backbone_weights(cfg, seed)
    if "depth" in heads:
        W.update(dpt_weights(cfg, seed + 1))
    if "seg" in heads:
        W.update(seg_weights(cfg, seed + 2))
    if "det" in heads:
        W.update(det_weights(cfg, seed + 3))
    return W


def make_frames(batch: int, resolution: int, stream_id: int = 0) -> torch.Tensor:
    """Seeded synthetic u8 RGB frames [B,3,R,R]."""
    g = torch.Generator().manual_seed(1000 + stream_id)
    return torch.randint(0, 256, (batch, 3, resolution, resolution), dtype=torch.uint8, generator=g)
