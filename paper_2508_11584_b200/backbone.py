"""Backbone backend ("b200_vit"): packs canonical DINOv2 weights into the device layouts the
sm_100a kernels consume and drives ``vpe_vit_forward`` (include/vpe.h).

Device layouts (HBM, packed once at init):
  patch_w  bf16 [D, 640]  conv weight flattened (c, ky, kx), K zero-padded 588 -> 640 (TMA 16B rows)
  qkv_w    bf16 [3D, D]   query | key | value rows -> one fused QKV GEMM per block
  proj/fc  bf16 [N, K]    K-major, straight from nn.Linear
  vectors  fp32           biases, LayerNorm affine, LayerScale, cls+pos[0], pos [T, D]
The position grid (37x37 learned, image_size=518) is bicubic-resized once per resolution at
init (modeling_dinov2.py:57-95), on the device.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.nn.functional as F

from . import _lib
from ._lib import check, lib
from .config import PATCH, BackboneConfig, grid, tokens

KPATCH = 640


def _interp_pos(pos: torch.Tensor, h: int) -> torch.Tensor:
    n = pos.shape[1] - 1
    g = int(round(n ** 0.5))
    if g == h:
        return pos[0]
    cls_pos, patch = pos[:, :1], pos[:, 1:]
    d = pos.shape[-1]
    patch = patch.reshape(1, g, g, d).permute(0, 3, 1, 2).float()
    patch = F.interpolate(patch, size=(h, h), mode="bicubic", align_corners=False)
    patch = patch.permute(0, 2, 3, 1).reshape(1, -1, d)
    return torch.cat([cls_pos, patch], dim=1)[0]


class Backbone:
    """DINOv2 ViT forward writing the 4 tap features into caller-provided (ring) buffers."""

    def __init__(self, W: dict, cfg: BackboneConfig, resolution: int, batch: int,
                 device: torch.device | str = "cuda"):
        self.cfg, self.resolution, self.batch = cfg, resolution, batch
        self.device = torch.device(device)
        self.h = grid(resolution)
        self.T = tokens(resolution)
        D, L = cfg.dim, cfg.depth
        dev = self.device
        keep = []

        def f32(t):
            t = t.detach().to(dev, torch.float32).contiguous()
            keep.append(t)
            return t.data_ptr()

        def bf16(t):
            t = t.detach().to(dev, torch.float32).to(torch.bfloat16).contiguous()
            keep.append(t)
            return t.data_ptr()

        wc = _lib.VitWeightsC()
        pw = W["embeddings.patch_embeddings.projection.weight"].reshape(D, 3 * PATCH * PATCH)
        wc.patch_w = bf16(F.pad(pw, (0, KPATCH - pw.shape[1])))
        wc.patch_b = f32(W["embeddings.patch_embeddings.projection.bias"])
        pos = _interp_pos(W["embeddings.position_embeddings"].to(dev, torch.float32), self.h)
        wc.cls_pos0 = f32(W["embeddings.cls_token"].reshape(D).to(dev) + pos[0])
        wc.pos = f32(pos)
        wc.norm_w = f32(W["layernorm.weight"])
        wc.norm_b = f32(W["layernorm.bias"])
        for i in range(L):
            p = f"encoder.layer.{i}."
            a = p + "attention.attention."
            wc.ln1_w[i] = f32(W[p + "norm1.weight"])
            wc.ln1_b[i] = f32(W[p + "norm1.bias"])
            wc.qkv_w[i] = bf16(torch.cat([W[a + "query.weight"], W[a + "key.weight"], W[a + "value.weight"]], 0))
            wc.qkv_b[i] = f32(torch.cat([W[a + "query.bias"], W[a + "key.bias"], W[a + "value.bias"]], 0))
            wc.proj_w[i] = bf16(W[p + "attention.output.dense.weight"])
            wc.proj_b[i] = f32(W[p + "attention.output.dense.bias"])
            wc.ls1[i] = f32(W[p + "layer_scale1.lambda1"])
            wc.ln2_w[i] = f32(W[p + "norm2.weight"])
            wc.ln2_b[i] = f32(W[p + "norm2.bias"])
            wc.fc1_w[i] = bf16(W[p + "mlp.fc1.weight"])
            wc.fc1_b[i] = f32(W[p + "mlp.fc1.bias"])
            wc.fc2_w[i] = bf16(W[p + "mlp.fc2.weight"])
            wc.fc2_b[i] = f32(W[p + "mlp.fc2.bias"])
            wc.ls2[i] = f32(W[p + "layer_scale2.lambda1"])
        cc = _lib.VitConfigC(dim=D, depth=L, heads=cfg.heads, mlp_hidden=cfg.hidden, resolution=resolution,
                             batch=batch, ln_eps=cfg.ln_eps)
        for k, t in enumerate(cfg.taps):
            cc.taps[k] = t
        h = C.c_void_p()
        torch.cuda.synchronize(dev)
        check(lib.vpe_vit_create(C.byref(cc), C.byref(wc), C.byref(h)), "vpe_vit_create")
        self._h = h
        self._keep = keep
        self._wc = wc

    def tap_shape(self) -> tuple[int, int, int]:
        return (self.batch, self.T, self.cfg.dim)

    def forward(self, pixels_u8: torch.Tensor, taps, stream: int | None = None) -> None:
        """pixels_u8: device u8 [B,3,R,R]; taps: 4 device bf16 tensors or raw pointers [B,T,D]."""
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        ptrs = (C.c_void_p * 4)(*[t if isinstance(t, int) else t.data_ptr() for t in taps])
        check(lib.vpe_vit_forward(self._h, C.c_void_p(pixels_u8.data_ptr()), ptrs, C.c_void_p(stream)),
              "vpe_vit_forward")

    def forward_camera(self, frames_hwc_u8: torch.Tensor, taps, stream: int | None = None) -> None:
        """frames_hwc_u8: device u8 [B, H, W, 3] camera frames (any H, W): centre crop, bilinear
        resize to R, normalisation and patch embedding in one kernel (vpe_vit_forward_camera)."""
        if frames_hwc_u8.dim() != 4 or frames_hwc_u8.shape[-1] != 3 or frames_hwc_u8.dtype != torch.uint8:
            raise ValueError(f"expected u8 [B,H,W,3], got {tuple(frames_hwc_u8.shape)} {frames_hwc_u8.dtype}")
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        ptrs = (C.c_void_p * 4)(*[t if isinstance(t, int) else t.data_ptr() for t in taps])
        H, Wd = frames_hwc_u8.shape[1], frames_hwc_u8.shape[2]
        check(lib.vpe_vit_forward_camera(self._h, C.c_void_p(frames_hwc_u8.data_ptr()), H, Wd, ptrs,
                                         C.c_void_p(stream)), "vpe_vit_forward_camera")

    def residual(self) -> torch.Tensor:
        p = C.c_void_p()
        check(lib.vpe_vit_residual(self._h, C.byref(p)))
        return _wrap_f32(p.value, (self.batch * self.T, self.cfg.dim), self.device)

    def close(self):
        if getattr(self, "_h", None):
            lib.vpe_vit_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_f32(ptr: int, shape, device) -> torch.Tensor:
    """Copy a libvpe-owned fp32 device buffer into a torch tensor (debug path only)."""
    n = 1
    for s in shape:
        n *= s
    out = torch.empty(shape, dtype=torch.float32, device=device)
    check(lib.vpe_memcpy_async(C.c_void_p(out.data_ptr()), C.c_void_p(ptr), n * 4,
                               C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))
    return out
