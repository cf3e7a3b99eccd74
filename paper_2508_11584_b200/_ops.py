"""Single-kernel entry points over the C ABI (vpe_op_*), used by parity tests and microbenchmarks."""

from __future__ import annotations

import ctypes as C

import torch

from ._lib import check, lib

EPI_BF16, EPI_RESID, EPI_F32 = 0, 1, 3
ACT_NONE, ACT_GELU, ACT_RELU = 0, 1, 2


def _s(stream):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream if stream is None else stream)


def _p(t):
    return C.c_void_p(None if t is None else t.data_ptr())


def linear(a: torch.Tensor, w: torch.Tensor, bias=None, scale=None, out=None, kind=EPI_BF16, act=ACT_NONE,
           bn=64, k_in=None, stream=None) -> torch.Tensor:
    """a: bf16 [M,K]; w: bf16 [N,Kw] (Kw multiple of K); returns bf16/f32 [M,N] (or updates out)."""
    M, K = a.shape
    N, Kw = w.shape
    if out is None:
        out = torch.empty(M, N, device=a.device, dtype=torch.bfloat16 if kind == EPI_BF16 else torch.float32)
    check(lib.vpe_op_linear(_p(a), M, K, _p(w), N, Kw, _p(bias), _p(scale), _p(out), kind, act, bn, _s(stream)),
          "vpe_op_linear")
    return out


def conv(x: torch.Tensor, w: torch.Tensor, C_real: int, ks: int, bias=None, add1=None, add2=None, act=ACT_NONE,
         out=None, out_relu=None, ldo=None, stream=None):
    """x: bf16 NHWC [B,H,W,Cp]; w: bf16 [N, ks*ks*Cp]."""
    B, H, W, Cp = x.shape
    N = w.shape[0]
    ldo = ldo or N
    if out is None:
        out = torch.zeros(B, H, W, ldo, device=x.device, dtype=torch.bfloat16)
    check(lib.vpe_op_conv(_p(x), B, H, W, C_real, Cp, ks, _p(w), N, _p(bias), _p(add1), _p(add2), _p(out),
                          _p(out_relu), ldo, act, _s(stream)), "vpe_op_conv")
    return out


def conv_up_pack(w: torch.Tensor, stream=None) -> torch.Tensor:
    """[32, 9*Cp] tap-major bf16 conv weights -> the fused kernel's dy-stacked [3, 96, Cp] layout."""
    Cp = w.shape[1] // 9
    wp = torch.empty(3, 96, Cp, device=w.device, dtype=torch.bfloat16)
    check(lib.vpe_op_conv_up_pack(_p(w), Cp, _p(wp), _s(stream)), "vpe_op_conv_up_pack")
    return wp


def conv_up(x: torch.Tensor, w: torch.Tensor, Ho: int, Wo: int, bias=None, act=ACT_NONE, out=None, ldo=None,
            w3=None, b3=0.0, wpack=None, stream=None):
    """3x3 conv of the align_corners=True resize of x (bf16 NHWC [B,Hs,Ws,Cp]) to Ho x Wo, fused.
    With w3 ([32] f32): returns the DPT depth map relu(b3 + relu(conv + bias) . w3) [B,Ho,Wo] f32."""
    B, Hs, Ws, Cp = x.shape
    N = w.shape[0]
    ldo = ldo or N
    if wpack is None:
        wpack = conv_up_pack(w, stream)
    depth = None
    if w3 is not None:
        depth = out if out is not None else torch.empty(B, Ho, Wo, device=x.device)
        out = None
    elif out is None:
        out = torch.zeros(B, Ho, Wo, ldo, device=x.device, dtype=torch.bfloat16)
    check(lib.vpe_op_conv_up(_p(x), B, Hs, Ws, Cp, Ho, Wo, _p(wpack), N, _p(bias), _p(out), ldo, act, _p(w3), b3,
                             _p(depth), _s(stream)), "vpe_op_conv_up")
    return depth if w3 is not None else out


def attention(qkv: torch.Tensor, B: int, T: int, D: int, heads: int, stream=None) -> torch.Tensor:
    out = torch.empty(B * T, D, device=qkv.device, dtype=torch.bfloat16)
    check(lib.vpe_op_attention(_p(qkv), _p(out), B, T, D, heads, _s(stream)), "vpe_op_attention")
    return out


def layernorm(x: torch.Tensor, w, b, eps=1e-6, w2=None, b2=None, stream=None):
    M, D = x.shape
    out = torch.empty(M, D, device=x.device, dtype=torch.bfloat16)
    out2 = torch.empty_like(out) if w2 is not None else None
    check(lib.vpe_op_layernorm(_p(x), M, D, _p(w), _p(b), eps, _p(out), _p(w2), _p(b2), _p(out2), _s(stream)),
          "vpe_op_layernorm")
    return out if out2 is None else (out, out2)


def linear_resid_ln(a: torch.Tensor, w: torch.Tensor, bias, ls, resid: torch.Tensor, ln_w, ln_b, eps: float,
                    tap_w=None, tap_b=None, stream=None):
    """resid += ls * (a @ w.T + bias) in place; returns (LayerNorm(resid) bf16, tap bf16 or None)."""
    M, K = a.shape
    xln = torch.empty(M, 384, device=a.device, dtype=torch.bfloat16)
    tap = torch.empty(M, 384, device=a.device, dtype=torch.bfloat16) if tap_w is not None else None
    check(lib.vpe_op_linear_resid_ln(_p(a), M, K, _p(w), _p(bias), _p(ls), _p(resid), _p(ln_w), _p(ln_b), eps, _p(xln),
                                     _p(tap_w), _p(tap_b), _p(tap), _s(stream)), "vpe_op_linear_resid_ln")
    return xln, tap


def bilinear(x: torch.Tensor, Ho: int, Wo: int, C: int | None = None, stream=None) -> torch.Tensor:
    """NHWC bf16 [B,Hi,Wi,cp] -> [B,Ho,Wo,cp], bilinear align_corners=True on the first C channels."""
    B, Hi, Wi, cp = x.shape
    out = torch.zeros(B, Ho, Wo, cp, device=x.device, dtype=torch.bfloat16)
    check(lib.vpe_op_bilinear(_p(x), B, Hi, Wi, cp, C or cp, _p(out), Ho, Wo, _s(stream)), "vpe_op_bilinear")
    return out


def upsample_argmax(logits: torch.Tensor, h: int, resolution: int, classes: int | None = None, stream=None):
    """logits fp32 [B, h*h, cp] -> u8 labels [B, R, R] (bilinear align_corners=False, argmax)."""
    B, hw, cp = logits.shape
    assert hw == h * h and logits.dtype == torch.float32 and logits.is_contiguous()
    C = cp if classes is None else classes
    labels = torch.empty(B, resolution, resolution, device=logits.device, dtype=torch.uint8)
    check(lib.vpe_op_upsample_argmax(_p(logits), B, h, C, cp, resolution, _p(labels), _s(stream)),
          "vpe_op_upsample_argmax")
    return labels


def camera_im2col(frames_hwc: torch.Tensor, resolution: int, stream=None) -> torch.Tensor:
    """u8 [B,H,W,3] -> normalised bf16 patch rows [B*(R/14)^2, 640] (crop, resize, normalise fused)."""
    B, H, W, _ = frames_hwc.shape
    n = B * (resolution // 14) ** 2
    out = torch.empty(n, 640, device=frames_hwc.device, dtype=torch.bfloat16)
    check(lib.vpe_op_camera_im2col(_p(frames_hwc), B, H, W, resolution, _p(out), _s(stream)), "vpe_op_camera_im2col")
    return out
