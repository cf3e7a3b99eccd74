"""SPEC known-answer examples for the per-head frequency control (PAPER.md
Appendix D), the transforms and the model registry."""

import os

import pytest
import torch

from paper_2508_11584_b200.arena import DType, TensorSpec
from paper_2508_11584_b200.errors import AlreadyExists, ConfigError, CorruptCard, NotFound, ShapeError
from paper_2508_11584_b200.pipeline import (IMAGENET_NORMALIZE, Transform, TransformKind, apply_transform, gate_admit,
                                            make_gate, set_rate)
from paper_2508_11584_b200.registry import ModelCard, Registry, demo_cards, validate_deployment

MS = 1_000_000


def count_admits(gate, period_ns, duration_ns, start=0):
    n, t = 0, start
    while t < start + duration_ns:
        n += gate_admit(gate, t)
        t += period_ns
    return n


@pytest.mark.parametrize("rate,stream_hz,expect", [(5, 100, 50), (10, 30, 100), (15, 30, 150), (30, 30, 300)])
def test_rate_gate_appendix_d(rate, stream_hz, expect):
    """PAPER.md:262-272 / SPEC.md:282-284: admits over 10 s within +-1 of rate x 10."""
    g = make_gate(rate_hz=rate, now_ns=0)
    n = count_admits(g, int(1e9 / stream_hz), 10_000 * MS)
    assert abs(n - expect) <= 1, n


def test_unlimited_and_frame_ratio():
    g = make_gate(None)
    assert count_admits(g, 10 * MS, 1000 * MS) == 100
    g2 = make_gate(every_n=4)
    assert sum(gate_admit(g2, i) for i in range(40)) == 10


def test_set_rate_semantics():
    gates = {"depth": make_gate(30, now_ns=0)}
    n1 = count_admits(gates["depth"], int(1e9 / 30), 10_000 * MS)
    set_rate(gates, "depth", 5, now=10_000 * MS)
    n2 = count_admits(gates["depth"], int(1e9 / 30), 10_000 * MS, start=10_000 * MS)
    assert abs(n1 - 300) <= 1 and abs(n2 - 50) <= 2
    with pytest.raises(NotFound):
        set_rate(gates, "seg", 5, now=0)
    with pytest.raises(ConfigError):
        set_rate(gates, "depth", 0, now=0)


def test_transforms():
    x = torch.arange(6, dtype=torch.float32).reshape(2, 3)
    assert torch.equal(apply_transform(Transform("r", TransformKind.RESHAPE, dims=(6,)), x), x.reshape(6))
    with pytest.raises(ShapeError):
        apply_transform(Transform("r", TransformKind.RESHAPE, dims=(4,)), x)
    u8 = torch.full((3, 2, 2), 255, dtype=torch.uint8)
    assert float(apply_transform(Transform("c", TransformKind.CAST_DTYPE, dtype=torch.float32), u8).max()) == 255.0
    ident = Transform("n", TransformKind.NORMALIZE_AFFINE, scale=(1.0, 1.0, 1.0), offset=(0.0, 0.0, 0.0))
    assert torch.equal(apply_transform(ident, u8.float()), u8.float())
    # the hot path's fused normalisation equals the oracle's (u8/255 - mean)/std
    from oracle.vit import preprocess
    img = torch.randint(0, 256, (1, 3, 4, 4), dtype=torch.uint8)
    torch.testing.assert_close(apply_transform(IMAGENET_NORMALIZE, img[0]), preprocess(img)[0], rtol=1e-5, atol=1e-5)


def test_registry_roundtrip_and_validation(tmp_path):
    from paper_2508_11584_b200.config import model_config
    reg = Registry(str(tmp_path))
    fm, heads = demo_cards(model_config("vits14"), 448)
    reg.register(fm)
    for h in heads:
        reg.register(h)
    assert reg.get(fm.name + "@latest").canonical() == fm.canonical()
    with pytest.raises(AlreadyExists):
        reg.register(fm)
    assert validate_deployment(fm, heads) == []
    bad = ModelCard("bad", 1, "head", (TensorSpec("layer99", DType.BF16, (1, 1025, 384)),), (), {"kind": "b200_det"})
    rep = validate_deployment(fm, [bad])
    assert rep and rep[0].problem == "missing label"
    wrong = ModelCard("wrong", 1, "head", (TensorSpec("final", DType.F32, (1, 1025, 384)),), (), {})
    assert "dtype" in validate_deployment(fm, [wrong])[0].problem
    # tamper -> CorruptCard
    p = os.path.join(str(tmp_path), fm.name, "1", "card")
    with open(p, "ab") as f:
        f.write(b" ")
    with pytest.raises(CorruptCard):
        reg.get(fm.name, 1)
    with pytest.raises(NotFound):
        reg.get("nope")
