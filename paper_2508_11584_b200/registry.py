"""Model registry — SPEC's ``registry`` module: ``ModelCard``, ``register``,
``get`` (by version or ``@latest``), ``validate_deployment``.

Cards are canonical sorted-key JSON bodies with a SHA-256 checksum stored as
``<root>/<name>/<version>/card`` + ``checksum`` (write-to-temp-then-rename). The ``backend``
descriptor names the sm_100a backend that serves the card ("b200_vit", "b200_dpt",
"b200_linseg", "b200_det") — the stand-in for the paper's TensorRT engines.
"""

from __future__ import annotations

import hashlib
import json
import os
import tempfile
from dataclasses import dataclass, field

from .arena import DType, TensorSpec
from .errors import AlreadyExists, ConfigError, CorruptCard, NotFound


@dataclass(frozen=True)
class ModelCard:
    name: str
    version: int
    kind: str                      # "foundation" | "head"
    input_specs: tuple[TensorSpec, ...]
    output_specs: tuple[TensorSpec, ...]
    backend: dict = field(default_factory=dict)
    default_rate: float | None = None
    subscriptions: tuple[str, ...] = ()   # head: labels consumed from the foundation

    def body(self) -> dict:
        return {"name": self.name, "version": self.version, "kind": self.kind,
                "input_specs": [s.to_dict() for s in self.input_specs],
                "output_specs": [s.to_dict() for s in self.output_specs],
                "backend": self.backend, "default_rate": self.default_rate,
                "subscriptions": list(self.subscriptions)}

    def canonical(self) -> bytes:
        return json.dumps(self.body(), sort_keys=True, separators=(",", ":")).encode()

    @property
    def checksum(self) -> str:
        return hashlib.sha256(self.canonical()).hexdigest()

    @classmethod
    def from_body(cls, d: dict) -> "ModelCard":
        return cls(name=d["name"], version=int(d["version"]), kind=d["kind"],
                   input_specs=tuple(TensorSpec.from_dict(s) for s in d["input_specs"]),
                   output_specs=tuple(TensorSpec.from_dict(s) for s in d["output_specs"]),
                   backend=d.get("backend", {}), default_rate=d.get("default_rate"),
                   subscriptions=tuple(d.get("subscriptions", ())))


class Registry:
    def __init__(self, root: str):
        self.root = root
        os.makedirs(root, exist_ok=True)

    def _dir(self, name, version):
        return os.path.join(self.root, name, str(version))

    def versions(self, name: str) -> list[int]:
        d = os.path.join(self.root, name)
        if not os.path.isdir(d):
            return []
        return sorted(int(v) for v in os.listdir(d) if v.isdigit())

    def register(self, card: ModelCard) -> int:
        if card.kind not in ("foundation", "head"):
            raise ConfigError(f"card kind must be foundation|head, got {card.kind!r}")
        d = self._dir(card.name, card.version)
        if os.path.exists(d):
            raise AlreadyExists(f"{card.name} v{card.version} already registered")
        parent = os.path.join(self.root, card.name)
        os.makedirs(parent, exist_ok=True)
        tmp = tempfile.mkdtemp(dir=parent)
        with open(os.path.join(tmp, "card"), "wb") as f:
            f.write(card.canonical())
        with open(os.path.join(tmp, "checksum"), "w") as f:
            f.write(card.checksum)
        os.rename(tmp, d)
        return card.version

    def get(self, ref: str, version: int | None = None) -> ModelCard:
        name, _, tag = ref.partition("@")
        if version is None:
            vs = self.versions(name)
            if not vs:
                raise NotFound(f"no card named {name!r}")
            version = vs[-1] if tag in ("", "latest") else int(tag)
        d = self._dir(name, version)
        if not os.path.isdir(d):
            raise NotFound(f"{name} v{version} not registered")
        body = open(os.path.join(d, "card"), "rb").read()
        want = open(os.path.join(d, "checksum")).read().strip()
        if hashlib.sha256(body).hexdigest() != want:
            raise CorruptCard(f"{name} v{version}: checksum mismatch")
        return ModelCard.from_body(json.loads(body))


@dataclass(frozen=True)
class Mismatch:
    head: str
    label: str
    problem: str


def validate_deployment(fm: ModelCard, heads: list[ModelCard]) -> list[Mismatch]:
    """Per head, every subscribed label must exist in the foundation outputs with the same
    dtype and dims. Returns the mismatch report (empty = valid)."""
    outs = {s.label: s for s in fm.output_specs}
    report = []
    for h in heads:
        for spec in h.input_specs:
            have = outs.get(spec.label)
            if have is None:
                report.append(Mismatch(h.name, spec.label, "missing label"))
            elif have.dtype != spec.dtype:
                report.append(Mismatch(h.name, spec.label, f"dtype {spec.dtype.value} != {have.dtype.value}"))
            elif have.dims != spec.dims:
                report.append(Mismatch(h.name, spec.label, f"dims {spec.dims} != {have.dims}"))
    return report


def demo_cards(model_cfg, resolution: int, batch: int = 1, rates: dict | None = None) -> tuple[ModelCard, list[ModelCard]]:
    """The paper's example deployment: FM with 4 labelled outputs, depth head on
    all four, seg and det heads on ``final``. ``rates`` sets the cards' default_rate per head
    name ("depth_dpt", "seg_linear", "det_rpn")."""
    from .config import tokens
    bb = model_cfg.backbone
    T = tokens(resolution)
    rates = rates or {}
    feat = tuple(TensorSpec(l, DType.BF16, (batch, T, bb.dim)) for l in bb.tap_labels)
    img = (TensorSpec("image", DType.U8, (batch, 3, resolution, resolution)),)
    fm = ModelCard(f"dinov2_{bb.name}", 1, "foundation", img, feat,
                   {"kind": "b200_vit", "model": bb.name, "dim": bb.dim, "depth": bb.depth, "resolution": resolution})
    R = resolution
    post = model_cfg.det.post_nms_top_n
    depth = ModelCard("depth_dpt", 1, "head", feat, (TensorSpec("depth", DType.F32, (batch, R, R)),),
                      {"kind": "b200_dpt"}, rates.get("depth_dpt"), bb.tap_labels)
    seg = ModelCard("seg_linear", 1, "head", feat[-1:], (TensorSpec("labels", DType.U8, (batch, R, R)),),
                    {"kind": "b200_linseg", "classes": model_cfg.seg_classes}, rates.get("seg_linear"), ("final",))
    det = ModelCard("det_rpn", 1, "head", feat[-1:],
                    (TensorSpec("boxes", DType.F32, (batch, post, 4)), TensorSpec("scores", DType.F32, (batch, post)),
                     TensorSpec("index", DType.I64, (batch, post)), TensorSpec("count", DType.I32, (batch,))),
                    {"kind": "b200_det"}, rates.get("det_rpn"), ("final",))
    return fm, [depth, seg, det]
