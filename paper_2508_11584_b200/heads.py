"""Head backends ("b200_dpt", "b200_linseg", "b200_det"): pack canonical weights into the
sm_100a layouts and drive ``vpe_dpt_forward`` / ``vpe_seg_forward`` / ``vpe_det_forward``.

Each head reads its ring labels IN PLACE (device pointers of the leased slot) — no copy_out.

Weight transforms done once at init, in fp64 then rounded:
  * DPT reassemble 0/1: 1x1 projection composed with ConvTranspose(k=s) into one [k*k*C, D]
    matrix + bias (both linear); 3x3 kernels re-laid out tap-major [N, 9*Cpad] for implicit GEMM.
  * seg: BatchNorm (eval) folded into the 1x1 classifier; weights split W = hi + lo (bf16 pair)
    so the tensor-core GEMM on exact-bf16 ring features yields ~fp32 logits.
  * det: 3x3 conv split hi + lo likewise; the 1x1 cls/bbox convs stay fp32 (CUDA-core FFMA).
"""

from __future__ import annotations

import ctypes as C
import math

import torch

from . import _lib
from ._lib import check, lib
from .config import DetConfig, ModelConfig, grid


def _pad_ch(c: int) -> int:
    return c if c % 64 == 0 else (32 if c == 32 else (c + 63) // 64 * 64)


def _split(w: torch.Tensor, parts: int = 2) -> torch.Tensor:
    """fp32/fp64 [N, K] -> bf16 [N, parts*K] = [hi | mid | lo ...] whose sum reproduces w to
    ~2^-(8*parts+1) relative (2 parts ~ 2^-17, 3 parts ~ fp32 exact)."""
    r = w.double()
    out = []
    for _ in range(parts):
        p = r.to(torch.bfloat16)
        out.append(p)
        r = r - p.double()
    return torch.cat(out, 1)


def _conv_taps(w: torch.Tensor, cpad: int) -> torch.Tensor:
    """[N, Cin, k, k] -> [N, k*k*cpad] tap-major, channel zero-padded."""
    n, cin, k, _ = w.shape
    t = torch.zeros(n, k, k, cpad, dtype=w.dtype)
    t[..., :cin] = w.permute(0, 2, 3, 1)
    return t.reshape(n, k * k * cpad)


class _Packer:
    def __init__(self, device):
        self.device = device
        self.keep = []

    def f32(self, t) -> int:
        t = t.detach().to(self.device, torch.float32).contiguous()
        self.keep.append(t)
        return t.data_ptr()

    def bf16(self, t) -> int:
        t = t.detach().double().to(torch.bfloat16).to(self.device).contiguous()
        self.keep.append(t)
        return t.data_ptr()

    def raw(self, t) -> int:
        t = t.to(self.device).contiguous()
        self.keep.append(t)
        return t.data_ptr()


def _stream(stream, device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream if stream is None else stream)


def _p(x):
    if x is None:
        return None
    return x if isinstance(x, int) else x.data_ptr()


class DepthHead:
    """DepthAnything DPT neck + depth head over the 4 tap labels."""

    kind = "b200_dpt"

    def __init__(self, W: dict, cfg: ModelConfig, resolution: int, batch: int, device="cuda"):
        self.device = torch.device(device)
        self.resolution, self.batch = resolution, batch
        self.tap_labels = cfg.backbone.tap_labels
        dp, D = cfg.dpt, cfg.backbone.dim
        F = dp.fusion
        pk = _Packer(self.device)
        wc = _lib.DptWeightsC()
        for i, (ch, f) in enumerate(zip(dp.neck, dp.factors)):
            p = f"neck.reassemble_stage.layers.{i}."
            wp = W[p + "projection.weight"].double()[:, :, 0, 0]  # [C, D]
            bp = W[p + "projection.bias"].double()
            if f > 1:
                k = int(f)
                cp = (ch + 31) // 32 * 32  # each sub-pixel's channels padded to a 32-column chunk
                wt = W[p + "resize.weight"].double()  # [C_in, C_out, k, k]
                m = torch.zeros(k, k, cp, ch, dtype=torch.float64)
                m[:, :, :ch, :] = wt.permute(2, 3, 1, 0)  # [(ky,kx,co), c]
                m = m.reshape(k * k * cp, ch)
                bt = torch.zeros(cp, dtype=torch.float64)
                bt[:ch] = W[p + "resize.bias"].double()
                wc.rs_w[i] = pk.bf16(m @ wp)
                wc.rs_b[i] = pk.f32(m @ bp + bt.repeat(k * k))
            else:
                wc.rs_w[i] = pk.bf16(wp)
                wc.rs_b[i] = pk.f32(bp)
            if f < 1:
                wc.rs3_conv_w = pk.bf16(_conv_taps(W[p + "resize.weight"].double(), _pad_ch(ch)))
                wc.rs3_conv_b = pk.f32(W[p + "resize.bias"])
        for i, ch in enumerate(dp.neck):
            wc.neck_w[i] = pk.bf16(_conv_taps(W[f"neck.convs.{i}.weight"].double(), _pad_ch(ch)))
        names = ("residual_layer1.convolution1", "residual_layer1.convolution2",
                 "residual_layer2.convolution1", "residual_layer2.convolution2")
        for k in range(4):
            p = f"neck.fusion_stage.layers.{k}."
            wc.proj_w[k] = pk.bf16(W[p + "projection.weight"].double()[:, :, 0, 0])
            wc.proj_b[k] = pk.f32(W[p + "projection.bias"])
            for j, nm in enumerate(names):
                wc.rcu_w[k][j] = pk.bf16(_conv_taps(W[p + nm + ".weight"].double(), F))
                wc.rcu_b[k][j] = pk.f32(W[p + nm + ".bias"])
        wc.head1_w = pk.bf16(_conv_taps(W["head.conv1.weight"].double(), F))
        wc.head1_b = pk.f32(W["head.conv1.bias"])
        wc.head2_w = pk.bf16(_conv_taps(W["head.conv2.weight"].double(), _pad_ch(F // 2)))
        wc.head2_b = pk.f32(W["head.conv2.bias"])
        wc.head3_w = pk.f32(W["head.conv3.weight"].reshape(-1))
        wc.head3_b = float(W["head.conv3.bias"].reshape(-1)[0])
        cc = _lib.DptConfigC(dim=D, resolution=resolution, batch=batch, fusion=F, head_hidden=dp.head_hidden,
                             max_depth=dp.max_depth)
        for i, ch in enumerate(dp.neck):
            cc.neck[i] = ch
        h = C.c_void_p()
        torch.cuda.synchronize(self.device)
        check(lib.vpe_dpt_create(C.byref(cc), C.byref(wc), C.byref(h)), "vpe_dpt_create")
        self._h, self._keep, self._wc = h, pk.keep, wc

    # -- engine-facing backend interface (shared by every head kind) -------------------------
    def subscriptions(self) -> tuple[str, ...]:
        return self.tap_labels

    def outputs(self, debug: bool = False) -> dict[str, torch.Tensor]:
        R, B, dev = self.resolution, self.batch, self.device
        out = {"depth": torch.zeros(B, R, R, device=dev)}
        if debug:  # pre-final-ReLU map (parity grading only)
            out["depth_pre"] = torch.zeros(B, R, R, device=dev)
        return out

    def run(self, views: dict, outs: dict, stream=None) -> None:
        self.forward([views[l] for l in self.tap_labels], outs["depth"], outs.get("depth_pre"), stream)

    def forward(self, taps, depth, depth_pre=None, stream=None):
        ptrs = (C.c_void_p * 4)(*[_p(t) for t in taps])
        check(lib.vpe_dpt_forward(self._h, ptrs, C.c_void_p(_p(depth)), C.c_void_p(_p(depth_pre)),
                                  _stream(stream, self.device)), "vpe_dpt_forward")

    def close(self):
        if getattr(self, "_h", None):
            lib.vpe_dpt_destroy(self._h)
            self._h = None

    __del__ = close


class SegHead:
    """BN + 1x1 linear classifier + bilinear upsample + argmax over the `final` label."""

    kind = "b200_linseg"

    def __init__(self, W: dict, cfg: ModelConfig, resolution: int, batch: int, device="cuda"):
        self.device = torch.device(device)
        self.resolution, self.batch = resolution, batch
        self.classes = cfg.seg_classes
        D = cfg.backbone.dim
        s = W["seg.bn.weight"].double() / torch.sqrt(W["seg.bn.running_var"].double() + cfg.seg_bn_eps)
        shift = W["seg.bn.bias"].double() - W["seg.bn.running_mean"].double() * s
        wcl = W["seg.classifier.weight"].double()[:, :, 0, 0]  # [C, D]
        wf = wcl * s[None, :]
        bf = W["seg.classifier.bias"].double() + wcl @ shift
        cpad = (self.classes + 31) // 32 * 32
        wsplit = torch.zeros(cpad, 2 * D, dtype=torch.bfloat16)
        wsplit[: self.classes] = _split(wf)
        pk = _Packer(self.device)
        wc = _lib.SegWeightsC(w_split=pk.raw(wsplit), b=pk.f32(bf))
        cc = _lib.SegConfigC(dim=D, resolution=resolution, batch=batch, classes=self.classes)
        h = C.c_void_p()
        torch.cuda.synchronize(self.device)
        check(lib.vpe_seg_create(C.byref(cc), C.byref(wc), C.byref(h)), "vpe_seg_create")
        self._h, self._keep, self._wc = h, pk.keep, wc

    def subscriptions(self) -> tuple[str, ...]:
        return ("final",)

    def outputs(self, debug: bool = False) -> dict[str, torch.Tensor]:
        R, B = self.resolution, self.batch
        return {"labels": torch.zeros(B, R, R, dtype=torch.uint8, device=self.device)}

    def run(self, views: dict, outs: dict, stream=None) -> None:
        self.forward(views["final"], outs["labels"], stream=stream)

    def forward(self, final, labels, logits=None, stream=None):
        check(lib.vpe_seg_forward(self._h, C.c_void_p(_p(final)), C.c_void_p(_p(labels)), C.c_void_p(_p(logits)),
                                  _stream(stream, self.device)), "vpe_seg_forward")

    def close(self):
        if getattr(self, "_h", None):
            lib.vpe_seg_destroy(self._h)
            self._h = None

    __del__ = close


def base_anchors(dc: DetConfig) -> list[list[float]]:
    """anchor_utils.py:58-77 in fp32 (ratio-major then size, rounded)."""
    scales = torch.as_tensor(dc.sizes, dtype=torch.float32)
    ar = torch.as_tensor(dc.ratios, dtype=torch.float32)
    h_r = torch.sqrt(ar)
    w_r = 1 / h_r
    ws = (w_r[:, None] * scales[None, :]).view(-1)
    hs = (h_r[:, None] * scales[None, :]).view(-1)
    return (torch.stack([-ws, -hs, ws, hs], dim=1) / 2).round().tolist()


DET_SPLIT = 2  # det 3x3 conv weights as hi+lo bf16 (tensor-core fp32 accumulation is the floor)


class DetHead:
    """RPN-style head: 3x3 conv + ReLU, 1x1 cls / bbox, decode, top-k, NMS over `final`."""

    kind = "b200_det"

    def __init__(self, W: dict, cfg: ModelConfig, resolution: int, batch: int, device="cuda"):
        self.device = torch.device(device)
        dc = cfg.det
        self.dc, self.batch = dc, batch
        D, A = cfg.backbone.dim, dc.num_anchors
        self.A = A
        self.n = grid(resolution) ** 2 * A
        pk = _Packer(self.device)
        wconv = _conv_taps(W["det.conv.weight"].double(), D)  # [D, 9D]
        wc = _lib.DetWeightsC(conv_w_split=pk.raw(_split(wconv, DET_SPLIT)), conv_b=pk.f32(W["det.conv.bias"]),
                              cls_w=pk.f32(W["det.cls_logits.weight"].reshape(A, D)),
                              cls_b=pk.f32(W["det.cls_logits.bias"]),
                              box_w=pk.f32(W["det.bbox_pred.weight"].reshape(4 * A, D)),
                              box_b=pk.f32(W["det.bbox_pred.bias"]))
        cc = _lib.DetConfigC(dim=D, resolution=resolution, batch=batch, pre_nms_top_n=dc.pre_nms_top_n,
                             post_nms_top_n=dc.post_nms_top_n, nms_thresh=dc.nms_thresh, min_size=dc.min_size,
                             score_thresh=dc.score_thresh, num_anchors=A, bbox_clip=math.log(1000.0 / 16))
        for a, row in enumerate(base_anchors(dc)):
            for j in range(4):
                cc.base_anchors[a][j] = row[j]
        h = C.c_void_p()
        torch.cuda.synchronize(self.device)
        check(lib.vpe_det_create(C.byref(cc), C.byref(wc), C.byref(h)), "vpe_det_create")
        self._h, self._keep, self._wc = h, pk.keep, wc

    def subscriptions(self) -> tuple[str, ...]:
        return ("final",)

    def run(self, views: dict, outs: dict, stream=None) -> None:
        self.forward(views["final"], outs, stream=stream)

    def outputs(self, debug: bool = False):
        post, B, dev = self.dc.post_nms_top_n, self.batch, self.device
        return {"boxes": torch.zeros(B, post, 4, device=dev), "scores": torch.zeros(B, post, device=dev),
                "index": torch.zeros(B, post, dtype=torch.int64, device=dev),
                "count": torch.zeros(B, dtype=torch.int32, device=dev)}

    def forward(self, final, out: dict, stream=None):
        oc = _lib.DetOutputsC(boxes=_p(out["boxes"]), scores=_p(out["scores"]), index=_p(out["index"]),
                              count=_p(out["count"]), objectness=_p(out.get("objectness")),
                              deltas=_p(out.get("deltas")), top_index=_p(out.get("top_index")))
        check(lib.vpe_det_forward(self._h, C.c_void_p(_p(final)), C.byref(oc), _stream(stream, self.device)),
              "vpe_det_forward")

    def close(self):
        if getattr(self, "_h", None):
            lib.vpe_det_destroy(self._h)
            self._h = None

    __del__ = close


# backend descriptor kind (registry ModelCard.backend["kind"]) -> head class
HEAD_BACKENDS = {DepthHead.kind: DepthHead, SegHead.kind: SegHead, DetHead.kind: DetHead}
# the paper's example deployment by short head name
BUILTIN_HEADS = {"depth": DepthHead.kind, "seg": SegHead.kind, "det": DetHead.kind}
# which canonical weight group (weights.make_weights ``heads=``) a backend kind reads
WEIGHT_GROUP = {DepthHead.kind: "depth", SegHead.kind: "seg", DetHead.kind: "det"}
