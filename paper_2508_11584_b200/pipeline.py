"""Pipeline pieces of the reference SPEC that sit on the hot path:
``RateGate`` / ``gate_admit`` / ``set_rate`` (per-head frequency control), the ``Transform``
adapters, and the ``ComputeBackend`` descriptors the registry references.

``gate_admit`` is the SPEC's deadline scheduler with one-period catch-up clamp:
admit iff now >= next_deadline; on admit next_deadline := max(next_deadline + period,
now - period). ``set_rate`` re-bases the deadline to now. A frame-ratio mode
(``every_n``) expresses BASELINE config C3's 1:1 / 1:2 / 1:4 head frequencies.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from fractions import Fraction

import torch

from .errors import ConfigError, NotFound, ShapeError

UNLIMITED = None


@dataclass
class RateGate:
    """rate_hz None = Unlimited; every_n = admit one frame in n (frame-ratio mode)."""

    rate_hz: float | Fraction | None = UNLIMITED
    next_deadline: int = 0
    every_n: int | None = None
    _count: int = 0

    @property
    def period_ns(self) -> int | None:
        if self.rate_hz is None:
            return None
        return int(round(1e9 / float(self.rate_hz)))


def make_gate(rate_hz=None, every_n: int | None = None, now_ns: int = 0) -> RateGate:
    if rate_hz is not None and float(rate_hz) <= 0:
        raise ConfigError(f"rate must be positive, got {rate_hz}")
    if every_n is not None and every_n < 1:
        raise ConfigError(f"every_n must be >= 1, got {every_n}")
    return RateGate(rate_hz=rate_hz, next_deadline=now_ns, every_n=every_n)


def gate_admit(g: RateGate, now: int) -> bool:
    """SPEC.md:276-284 (deadline mode) or every-n-th frame (frame-ratio mode)."""
    if g.every_n is not None:
        ok = (g._count % g.every_n) == 0
        g._count += 1
        return ok
    if g.rate_hz is None:
        return True
    if now >= g.next_deadline:
        p = g.period_ns
        g.next_deadline = max(g.next_deadline + p, now - p)
        return True
    return False


def set_rate(gates: dict, head: str, new_rate, now: int, every_n: int | None = None) -> None:
    """unknown head -> NotFound, non-positive -> ConfigError, re-base to now."""
    if head not in gates:
        raise NotFound(f"unknown head {head!r}")
    if new_rate is not None and float(new_rate) <= 0:
        raise ConfigError(f"rate must be positive, got {new_rate}")
    g = gates[head]
    g.rate_hz = new_rate
    g.every_n = every_n
    g._count = 0
    g.next_deadline = now


# ---- transforms ----------------------------------------------------
class TransformKind(Enum):
    RESHAPE = "reshape"
    NORMALIZE_AFFINE = "normalize_affine"
    CAST_DTYPE = "cast_dtype"
    CROP_PAD = "crop_pad"
    IDENTITY = "identity"


@dataclass(frozen=True)
class Transform:
    name: str
    kind: TransformKind
    scale: tuple[float, ...] = ()
    offset: tuple[float, ...] = ()
    dims: tuple[int, ...] = ()
    dtype: torch.dtype | None = None


def apply_transform(t: Transform, x: torch.Tensor) -> torch.Tensor:
    """Pure, deterministic adapters. On the hot path the ImageNet NormalizeAffine + CastDType
    U8->F32 pair is fused into the patch-embedding kernel (misc.cu patch_im2col_kernel)."""
    if t.kind is TransformKind.IDENTITY:
        return x
    if t.kind is TransformKind.RESHAPE:
        n = 1
        for d in t.dims:
            n *= d
        if n != x.numel():
            raise ShapeError(f"reshape {tuple(x.shape)} -> {t.dims} changes element count")
        return x.reshape(t.dims)
    if t.kind is TransformKind.CAST_DTYPE:
        if t.dtype is None:
            raise ShapeError("cast needs a dtype")
        if not t.dtype.is_floating_point:
            info = torch.iinfo(t.dtype)
            return x.clamp(info.min, info.max).to(t.dtype)  # saturating cast
        return x.to(t.dtype)
    if t.kind is TransformKind.NORMALIZE_AFFINE:
        c = x.shape[-3] if x.dim() >= 3 else 1
        s = torch.tensor(t.scale or (1.0,) * c, dtype=torch.float32, device=x.device).view(-1, 1, 1)
        o = torch.tensor(t.offset or (0.0,) * c, dtype=torch.float32, device=x.device).view(-1, 1, 1)
        return x.float() * s + o
    if t.kind is TransformKind.CROP_PAD:
        out = torch.zeros(t.dims, dtype=x.dtype, device=x.device)
        sl = tuple(slice(0, min(a, b)) for a, b in zip(x.shape, t.dims))
        out[sl] = x[sl]
        return out
    raise ShapeError(f"unknown transform {t.kind}")


IMAGENET_NORMALIZE = Transform(
    "imagenet", TransformKind.NORMALIZE_AFFINE,
    scale=tuple(1.0 / (255.0 * s) for s in (0.229, 0.224, 0.225)),
    offset=tuple(-m / s for m, s in zip((0.485, 0.456, 0.406), (0.229, 0.224, 0.225))))


# ---- compute backends: descriptors the registry cards carry ---------------
@dataclass(frozen=True)
class ComputeBackend:
    kind: str                     # "b200_vit" | "b200_dpt" | "b200_linseg" | "b200_det"
    params: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return {"kind": self.kind, "params": dict(sorted(self.params.items()))}


BACKEND_KINDS = ("b200_vit", "b200_dpt", "b200_linseg", "b200_det")
