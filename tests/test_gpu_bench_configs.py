"""Stage-wise head parity at exactly the configurations bench.py measures:

* C2: ViT-S/14 at 448, batch 16 (16 camera streams), depth + seg + det on every frame;
* C3: ViT-B/14 at 518, batch 16, depth 1:1 / seg 1:2 / det 1:4 — through the engine's gates;
* C5: ViT-L/14 at 518, batch 8, all three heads (seg and det at D = 1024).

Every head output of every frame of the batch is graded against the oracle head fed the exact
bf16 ring tensor the GPU wrote, with the BASELINE bars: depth pre/post-ReLU
rel-L2 <= 1e-2 and cos >= 0.999; seg argmax agreement >= 99.9%; det post-NMS detections
identical index for index except near-tie swaps the measured logit error explains
(tests/det_match.py; every such swap is recorded). The pre-NMS top-1000 ranking is compared position by position and
every swap is recorded (``VPE_PARITY_OUT`` = JSON artifact path, committed under profiles/);
a swap is only accepted between anchors whose oracle logits differ by less than twice the
measured logit error. The DPT oracle is expensive on the CPU at B/14 and L/14, so depth there is
graded on the first, a middle and the last frame of the batch."""

import json
import os

import pytest
import torch

from oracle import det as odet
from oracle import dpt as odpt
from oracle import seg as oseg
from det_match import align_to, kept_match
from paper_2508_11584_b200.config import grid, model_config
from paper_2508_11584_b200.weights import make_frames, make_weights

pytestmark = pytest.mark.gpu

RECORDS = []


def rel_l2(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def cosine(a, b):
    return torch.nn.functional.cosine_similarity(a.float().flatten(), b.float().flatten(), dim=0).item()


@pytest.fixture(scope="module", autouse=True)
def _artifact():
    yield
    path = os.environ.get("VPE_PARITY_OUT")
    if path and RECORDS:
        with open(path, "w") as f:
            json.dump(RECORDS, f, indent=1)


CONFIGS = {
    "C2": dict(model="vits14", R=448, B=16, rates=None, depth_frames=None),
    "C3": dict(model="vitb14", R=518, B=16, rates={"depth": "1:1", "seg": "1:2", "det": "1:4"}, depth_frames=(0, 8, 15)),
    "C5": dict(model="vitl14", R=518, B=8, rates=None, depth_frames=(0, 7)),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_bench_config_heads(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2508_11584_b200.engine import VPEngine
    c = CONFIGS[name]
    model, R, B = c["model"], c["R"], c["B"]
    cfg = model_config(model)
    W = make_weights(model)
    h = grid(R)
    # the bench's camera streams: stream i contributes frame i (bench.py run_ours)
    frames = torch.cat([make_frames(1, R, stream_id=s) for s in range(B)], 0)
    eng = VPEngine(model, R, B, weights=W, rates=c["rates"], debug_outputs=True)
    try:
        eng.channel.register_consumer(99)  # grader: reads the ring slot in place
        eng.pixels.copy_(frames.to(eng.device))
        torch.cuda.synchronize()
        # C3: the engine's frame-ratio gates decide; on frame 1 every head runs (1:n admits the
        # first frame), so grade frame set 1 and check the gate pattern over the next ones
        ran = eng.submit()
        eng.synchronize()
        assert set(ran) == {"depth", "seg", "det"}
        lease = eng.channel.acquire_latest(99)
        views = eng.channel.view(lease)
        taps = [views[l].float().cpu() for l in eng.labels]
        eng.channel.commit(lease)
        out = {n: {k: t.cpu() for k, t in o.items()} for n, o in eng.out.items()}
        if c["rates"]:
            pattern = [eng.submit() for _ in range(8)]
            eng.synchronize()
            assert sum("seg" in p for p in pattern) == 4 and sum("det" in p for p in pattern) == 2
            assert all("depth" in p for p in pattern)
        # det: also the raw maps and the pre-NMS top-k, from a standalone head on the same tap
        from paper_2508_11584_b200.heads import DetHead
        det = eng.heads["det"]
        dout = det.outputs()
        n = h * h * cfg.det.num_anchors
        dout["objectness"] = torch.empty(B, n, device=eng.device)
        dout["deltas"] = torch.empty(B, n, 4, device=eng.device)
        dout["top_index"] = torch.empty(B, min(n, cfg.det.pre_nms_top_n), dtype=torch.int64, device=eng.device)
        tap_dev = taps[3].to(eng.device).to(torch.bfloat16)
        assert isinstance(det, DetHead)
        det.forward(tap_dev, dout)
        torch.cuda.synchronize()
    finally:
        eng.close()
    # the standalone run on the same tap reproduces the engine's detections bit for bit
    for k in ("boxes", "scores", "index", "count"):
        assert torch.equal(dout[k].cpu(), out["det"][k]), k

    # ---- depth (pre- and post-final-ReLU)
    frames_d = range(B) if c["depth_frames"] is None else c["depth_frames"]
    for b in frames_d:
        rd, rp = odpt.dpt_forward([t[b:b + 1] for t in taps], W, cfg.dpt.factors, h, return_pre_relu=True)
        gp, gd = out["depth"]["depth_pre"][b:b + 1], out["depth"]["depth"][b:b + 1]
        e_pre, c_pre, e, cs = rel_l2(gp, rp), cosine(gp, rp), rel_l2(gd, rd), cosine(gd, rd)
        RECORDS.append(dict(config=name, head="depth", frame=b, rel_pre=e_pre, cos_pre=c_pre, rel=e, cos=cs))
        assert e_pre <= 1e-2 and c_pre >= 0.999, (name, b, e_pre, c_pre)
        assert e <= 1e-2 and cs >= 0.999, (name, b, e, cs)

    # ---- seg (every frame)
    agree = torch.tensor([(out["seg"]["labels"][b] == oseg.seg_forward(taps[3][b:b + 1], W, h, R)[0]).float().mean()
                          for b in range(B)])
    for b in range(B):
        RECORDS.append(dict(config=name, head="seg", frame=b, agreement=float(agree[b])))
    assert float(agree.min()) >= 0.999, (name, agree.tolist())

    # ---- det (every frame)
    obj, deltas, _ = odet.det_head_maps(taps[3], W, h)
    ref = odet.det_postprocess(obj, deltas, h, R, cfg.det)
    max_err = (dout["objectness"].cpu() - obj).abs().max().item()
    for b in range(B):
        k = int(out["det"]["count"][b])
        gi, ri = out["det"]["index"][b, :k], ref[b]["index"]
        gt, rt = dout["top_index"][b].cpu(), ref[b]["top_index"]
        diff = (gt != rt).nonzero().flatten()
        gap = (obj[b][gt[diff]] - obj[b][rt[diff]]).abs().max().item() if diff.numel() else 0.0
        ok, kswaps, kgap = kept_match(gi, ri, obj[b], max_err)
        RECORDS.append(dict(config=name, head="det", frame=b, kept=k, kept_identical=bool(torch.equal(gi, ri)),
                            kept_positions_swapped=kswaps, kept_max_swap_gap=kgap,
                            topk_positions_swapped=int(diff.numel()), topk_max_swap_gap=gap,
                            logit_max_err=max_err))
        assert ok, (name, b, kswaps, kgap, max_err)
        assert gap <= 2 * max_err, (name, b, gap, max_err)
        # box coordinates inherit the deltas' ~1e-5 relative error (fp32 tensor-core accumulation
        # over K = 9 D): measured up to 2.1e-3 px at D = 1024, R = 518
        p = align_to(gi, ri)
        torch.testing.assert_close(out["det"]["boxes"][b, :k][p], ref[b]["boxes"], rtol=1e-5, atol=1e-5 * R)
        torch.testing.assert_close(out["det"]["scores"][b, :k][p], ref[b]["scores"], rtol=1e-5, atol=1e-6)
