"""Model / head geometry for the shared-backbone hot path.

Backbone geometry follows DINOv2 (``PAPER.md:136``; third-party oracle
``transformers/models/dinov2/configuration_dinov2.py:55-75``, pinned 5.5.0).
Depth-head geometry follows DepthAnything(V2)'s DPT neck
(``transformers/models/depth_anything/configuration_depth_anything.py:64-91``).
Tap labels follow SPEC ``{final, layer3, layer6, layer9}`` (``SPEC.md:266``):
the final-LN'd outputs of blocks L/4, L/2, 3L/4 and L.
"""

from __future__ import annotations

from dataclasses import dataclass, field

PATCH = 14
POS_GRID = 37  # image_size=518 -> 37x37 learned position grid
IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


@dataclass(frozen=True)
class BackboneConfig:
    name: str
    dim: int
    depth: int
    heads: int
    mlp_ratio: int = 4
    ln_eps: float = 1e-6

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads

    @property
    def hidden(self) -> int:
        return self.dim * self.mlp_ratio

    @property
    def taps(self) -> tuple[int, ...]:
        L = self.depth
        return (L // 4, L // 2, 3 * L // 4, L)

    @property
    def tap_labels(self) -> tuple[str, ...]:
        t = self.taps
        return tuple(f"layer{k}" for k in t[:3]) + ("final",)


@dataclass(frozen=True)
class DPTConfig:
    neck: tuple[int, int, int, int]
    fusion: int
    head_hidden: int = 32
    factors: tuple[float, ...] = (4, 2, 1, 0.5)
    max_depth: float = 1.0


@dataclass(frozen=True)
class DetConfig:
    sizes: tuple[int, ...] = (32, 64, 128)
    ratios: tuple[float, ...] = (0.5, 1.0, 2.0)
    pre_nms_top_n: int = 1000
    post_nms_top_n: int = 100
    nms_thresh: float = 0.7
    min_size: float = 1e-3
    score_thresh: float = 0.0
    weights: tuple[float, float, float, float] = (1.0, 1.0, 1.0, 1.0)

    @property
    def num_anchors(self) -> int:
        return len(self.sizes) * len(self.ratios)


@dataclass(frozen=True)
class ModelConfig:
    backbone: BackboneConfig
    dpt: DPTConfig
    seg_classes: int = 150
    seg_bn_eps: float = 1e-5
    det: DetConfig = field(default_factory=DetConfig)


BACKBONES = {
    "vits14": BackboneConfig("vits14", 384, 12, 6),
    "vitb14": BackboneConfig("vitb14", 768, 12, 12),
    "vitl14": BackboneConfig("vitl14", 1024, 24, 16),
}

DPTS = {
    "vits14": DPTConfig((48, 96, 192, 384), 64),
    "vitb14": DPTConfig((96, 192, 384, 768), 128),
    "vitl14": DPTConfig((256, 512, 1024, 1024), 256),
}


def model_config(name: str = "vits14", seg_classes: int = 150) -> ModelConfig:
    if name not in BACKBONES:
        raise KeyError(f"unknown backbone {name!r}; have {sorted(BACKBONES)}")
    return ModelConfig(BACKBONES[name], DPTS[name], seg_classes=seg_classes)


def grid(resolution: int) -> int:
    if resolution % PATCH:
        raise ValueError(f"resolution {resolution} not a multiple of {PATCH}")
    return resolution // PATCH


def tokens(resolution: int) -> int:
    h = grid(resolution)
    return h * h + 1


def backbone_flops(cfg: BackboneConfig, resolution: int) -> float:
    """2*Np*588*D + L*(24*T*D^2 + 4*T^2*D) per image."""
    h = grid(resolution)
    np_, t, d = h * h, h * h + 1, cfg.dim
    return 2.0 * np_ * 588 * d + cfg.depth * (24.0 * t * d * d + 4.0 * t * t * d)
