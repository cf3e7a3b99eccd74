"""Camera ingest: u8 HWC frames -> crop -> bilinear resize -> normalise ->
patch embedding, fused into one kernel (csrc/misc.cu camera_im2col_kernel) and checked against
oracle/camera.py."""
import pytest
import torch
import torch.nn.functional as F

from oracle import camera as ocam
from oracle import vit as ovit


def rel_l2(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm()).item()


def test_oracle_identity_resize_matches_chw_preprocess():
    """H = W = R: the crop/resize is the identity and the transform reduces to the CHW path."""
    g = torch.Generator().manual_seed(5)
    hwc = torch.randint(0, 256, (2, 224, 224, 3), dtype=torch.uint8, generator=g)
    chw = hwc.permute(0, 3, 1, 2).contiguous()
    assert torch.allclose(ocam.camera_preprocess(hwc, 224), ovit.preprocess(chw), atol=1e-6)


def test_oracle_crop_is_centred():
    hwc = torch.zeros(1, 100, 140, 3, dtype=torch.uint8)
    hwc[:, :, 20:120] = 255  # the centred 100x100 square
    x = ocam.camera_preprocess(hwc, 28)
    white = (1.0 - ovit.MEAN) / ovit.STD
    assert torch.allclose(x, white.expand_as(x), atol=1e-5)


def test_patch_rows_layout():
    x = torch.arange(2 * 3 * 28 * 28, dtype=torch.float32).reshape(2, 3, 28, 28)
    rows = ocam.patch_rows(x)
    assert rows.shape == (2 * 4, 640)
    # row 1 = image 0, patch (0, 1); k = c*196 + ky*14 + kx
    assert rows[1, 196 + 2 * 14 + 3] == x[0, 1, 2, 14 + 3]
    assert (rows[:, 588:] == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("B,H,W,R", [(2, 1080, 1920, 448), (1, 480, 640, 224), (1, 518, 518, 518),
                                     (2, 101, 333, 224), (1, 720, 1280, 518)])
def test_camera_im2col_kernel(ops, device, B, H, W, R):
    g = torch.Generator().manual_seed(H + W)
    hwc = torch.randint(0, 256, (B, H, W, 3), dtype=torch.uint8, generator=g)
    out = ops.camera_im2col(hwc.to(device), R)
    torch.cuda.synchronize()
    ref = ocam.patch_rows(ocam.camera_preprocess(hwc, R))
    assert out.shape == ref.shape
    # bf16 rounding of the normalised values is the only difference
    assert (out.float().cpu() - ref).abs().max().item() < 0.02
    assert rel_l2(out, ref) < 4e-3


@pytest.mark.gpu
def test_backbone_camera_forward(device):
    from paper_2508_11584_b200.backbone import Backbone
    from paper_2508_11584_b200.config import model_config, tokens
    from paper_2508_11584_b200.weights import make_weights
    cfg = model_config("vits14")
    W = make_weights("vits14", heads=())
    R, B = 224, 2
    g = torch.Generator().manual_seed(11)
    hwc = torch.randint(0, 256, (B, 480, 640, 3), dtype=torch.uint8, generator=g)
    bb = Backbone(W, cfg.backbone, R, B, device)
    T, D = tokens(R), cfg.backbone.dim
    taps = [torch.empty(B, T, D, device=device, dtype=torch.bfloat16) for _ in range(4)]
    bb.forward_camera(hwc.to(device), taps)
    torch.cuda.synchronize()
    x = ocam.camera_preprocess(hwc, R)
    ref = ovit.backbone_forward(x, W, cfg.backbone.depth, cfg.backbone.heads, cfg.backbone.taps)
    for t, r in zip(taps, ref):
        assert rel_l2(t, r) < 1e-2
        assert F.cosine_similarity(t.float().cpu().flatten(), r.flatten(), dim=0).item() > 0.999
    bb.close()
