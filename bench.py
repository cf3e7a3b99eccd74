#!/usr/bin/env python
"""Headline benchmark: end-to-end frames/sec of DINOv2 ViT-S/14 + depth + seg + det heads at
448x448 (BASELINE.json config C2, all heads every frame) on N B200s, plus per-head p50 latency.

One step = one frame set of ``--batch`` camera frames (batch 1 per camera stream; the engine
co-schedules the cameras it serves through one backbone pass) through the full hot path:
H2D (e2e only) -> backbone -> ring publish -> depth/seg/det heads in place -> D2H (e2e only).
With ``--gpus N`` (N > 1) and no torchrun environment, bench.py re-launches itself under
``torch.distributed.run`` with one rank per GPU; each rank drives one GPU with its own shard of
camera streams; there is no collective on the data path — torch.distributed is used
only for the barrier and the max-over-ranks of the timed region.

  python bench.py --gpus N --steps K --warmup W [--batch B] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "end-to-end frames/sec (backbone+3 heads) at 1/2/4/8 B200; per-head p50 latency"
UNIT = "frames/s"
L2_BYTES = 126 * 1024 * 1024
BACKBONE_BN = 256  # csrc/vit.cu pick_bn() at the bench shapes


def workload_name(args) -> str:
    if args.model == "vits14" and args.resolution == 448 and not args.rates:
        return "C2: DINOv2 ViT-S/14 + depth + seg + det heads, 448x448, all heads every frame"
    name = {"vits14": "ViT-S/14", "vitb14": "ViT-B/14", "vitl14": "ViT-L/14"}.get(args.model, args.model)
    rates = f", head rates {args.rates}" if args.rates else ", all heads every frame"
    tag = "C3: " if args.model == "vitb14" and args.resolution == 518 and args.rates else (
        "C5: " if args.model == "vitl14" and args.resolution == 518 else "")
    return f"{tag}DINOv2 {name} + depth + seg + det heads, {args.resolution}x{args.resolution}{rates}"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--batch", type=int, default=int(os.environ.get("VPE_BATCH", "16")))
    p.add_argument("--model", default="vits14")
    p.add_argument("--resolution", type=int, default=448)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--sustained-seconds", type=float, default=10.0,
                   help="length of the sustained C2 window reported beside the --steps number (0 = skip)")
    p.add_argument("--rates", default="", help="per-head frame ratios, e.g. depth=1:1,seg=1:2,det=1:4 (config C3)")
    return p.parse_args()


# ------------------------------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """--gpus N without a torchrun environment: one process per GPU via torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def dist_setup(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n:
        raise SystemExit(f"bench.py: --gpus {n} but WORLD_SIZE={world}")
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if _cuda() else "gloo")
        return rank, world, local, dist
    return 0, 1, 0, None


def _cuda():
    import torch
    return torch.cuda.is_available()


class ClockSampler:
    """SM clocks + throttle reasons from NVML, sampled every 5 ms in a thread while the timed
    region runs, plus one sample right before and right after it. NVML is initialised here, in
    the caller's thread, before the window opens."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, gpu: int):
        self.rows, self.edges, self._stop = [], {}, threading.Event()
        self.err = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(gpu)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as exc:
            self.nv, self.max_mhz, self.err = None, None, repr(exc)
        self._t = threading.Thread(target=self._run, daemon=True)

    def sample(self):
        sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        return sm, rs

    def _run(self):
        while not self._stop.is_set():
            try:
                self.rows.append(self.sample())
            except Exception as exc:
                self.err = repr(exc)
                return
            self._stop.wait(0.005)

    def __enter__(self):
        if self.nv:
            self.edges["before"] = self.sample()
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self._t.join(timeout=6)
            self.edges["after"] = self.sample()

    def _names(self, mask):
        return sorted(name for bit, name in self.REASONS.items() if mask & bit)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "error": self.err}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for _, m in self.rows for n in self._names(m)})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "sm_mhz_min": min(sm),
                "before": {"sm_mhz": self.edges["before"][0], "reasons": self._names(self.edges["before"][1])},
                "after": {"sm_mhz": self.edges["after"][0], "reasons": self._names(self.edges["after"][1])}}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm": d["hbm_gbs"], "tensor": d["bf16_tflops"],
                "tensor_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "kind": "measured"}
    except Exception:  # /opt/skills/guides/B200_PROFILING.md fallbacks
        return {"hbm": 6650.0, "tensor": 1590.0, "tensor_sustained": 1400.0, "kind": "fallback"}


def frame_flops(cfg, R):
    """Algorithmic FLOPs per frame: backbone + DPT + seg conv + det conv."""
    from paper_2508_11584_b200.config import backbone_flops
    return backbone_flops(cfg.backbone, R) + {448: 16.32e9 + 0.12e9 + 2.75e9, 224: 4.08e9}.get(R, 0.0)


# ------------------------------------------------------------------------------------------------
def cpu_baseline(args, cfg, W, seconds):
    """Reference CPU path (fanpipe transport + fp32 oracle, all host threads) on a bounded sample."""
    from oracle.cpu_pipeline import CpuPipeline
    from paper_2508_11584_b200.weights import make_frames
    threads = os.cpu_count() or 1
    pipe = CpuPipeline(cfg, W, args.resolution, 1, threads=threads)
    frames = make_frames(1, args.resolution, 0)
    pipe.step(frames)  # warm-up
    t0, n = time.perf_counter(), 0
    while True:
        pipe.step(frames)
        n += 1
        if time.perf_counter() - t0 >= seconds or n >= 200:
            break
    dt = time.perf_counter() - t0
    pipe.close()
    return {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} frames of C2 (batch 1, S/14 448 + 3 heads), fp32 oracle over fanpipe LATEST channel, "
                      f"{dt:.1f}s, torch threads={threads}"}


def run_reference(args):
    """The reference's CPU path on the host cores: (i) sequential foundation -> heads over the
    unmodified fanpipe LATEST channel, (ii) the paper's deployment, one foundation process and
    one process per head over the same channel (oracle/cpu_pipeline.py). The line's value is the
    faster of the two (the stronger baseline)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.cpu_pipeline import CpuPipeline, multiprocess_pipeline
    from paper_2508_11584_b200.config import model_config
    from paper_2508_11584_b200.weights import make_frames, make_weights
    cfg = model_config(args.model)
    W = make_weights(args.model)
    threads = os.cpu_count() or 1
    pipe = CpuPipeline(cfg, W, args.resolution, 1, threads=threads)
    frames = make_frames(1, args.resolution, 0)
    for _ in range(args.warmup):
        pipe.step(frames)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        pipe.step(frames)
    dt = time.perf_counter() - t0
    pipe.close()
    seq = args.steps / dt
    try:
        mp = multiprocess_pipeline(args.model, args.resolution, max(5.0, min(20.0, 0.5 * dt)), threads=threads)
    except Exception as exc:  # reported, the sequential variant stands
        mp = {"error": repr(exc), "fps": 0.0}
    v = max(seq, mp["fps"])
    kind = "sequential" if v == seq else "multiprocess"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C2: DINOv2 ViT-S/14 + depth + seg + det heads, 448x448, all heads every frame",
                   "batch": 1, "host": "cpu"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"best of (i) {args.steps} frames (batch 1) sequential foundation -> 3 heads "
                                   f"through the unmodified fanpipe transport (baseline/_ref) + fp32 oracle, "
                                   f"{threads} torch threads: {seq:.2f} fps; (ii) 1 foundation + 3 head processes "
                                   f"over a fanpipe LATEST channel, threads {mp.get('threads')}: "
                                   f"{mp['fps']:.2f} fps -> {kind}"},
        "variants": {"sequential": {"fps": seq, "seconds": dt}, "multiprocess": mp},
        "cpu_model": _cpu_model(),
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    # the reference's shared-memory arena raises BufferError from __del__ at interpreter exit
    # while numpy views are alive (fanpipe/arena.py:269-276); the result is printed, leave quietly
    sys.stderr.flush()
    os._exit(0)


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------------------------------------
def _graph_time(fn, reps: int = 20, replays: int = 10) -> float:
    """Seconds per call of ``fn`` (kernel launches only), timed over CUDA-graph replays with
    CUDA events on the capturing stream, after warm-up."""
    import torch
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(replays):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / (reps * replays)


def _ncu_traffic(name, shape):
    """DRAM bytes per launch from the committed ncu --set full summary of this kernel when the
    captured shape matches (profiles/round2_ncu_<name>.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", f"round2_ncu_{name}.json")) as f:
            d = json.load(f)
        if d.get("shape") == shape:
            return d["dram_bytes_read"] + d["dram_bytes_write"]
    except Exception:
        pass
    return None


def kernel_rooflines(eng, peaks):
    """Each kernel class of the step timed alone at the step's exact shapes (CUDA events over
    graph replays): achieved = algorithmic FLOPs or bytes per launch / launch time, against the
    measured burst peak (tensor) or copy bandwidth (HBM). Returns (dominant, list)."""
    import torch
    from paper_2508_11584_b200 import _ops
    dev = eng.device
    D, T, B, R = eng.D, eng.T, eng.batch, eng.resolution
    H = eng.cfg.backbone.heads
    M = B * T
    g = torch.Generator(device="cpu").manual_seed(0)

    def rnd(*shape, std=1.0, dtype=torch.bfloat16):
        return (torch.randn(*shape, generator=g) * std).to(dev, dtype)

    out = []

    def tensor(name, kernel, shape, flops, fn):
        dur = _graph_time(fn)
        a = flops / dur / 1e12
        out.append({"kernel": kernel, "class": name, "shape": shape, "bound": "tensor", "achieved": a,
                    "peak": peaks["tensor"], "unit": "TFLOP/s", "frac": a / peaks["tensor"],
                    "duration_us": dur * 1e6, "algorithmic": flops, "traffic": _ncu_traffic(name, shape)})

    def hbm(name, kernel, shape, nbytes, fn, note=""):
        dur = _graph_time(fn)
        a = nbytes / dur / 1e9
        out.append({"kernel": kernel, "class": name, "shape": shape, "bound": "hbm", "achieved": a,
                    "peak": peaks["hbm"], "unit": "GB/s", "frac": a / peaks["hbm"], "duration_us": dur * 1e6,
                    "algorithmic": nbytes, "traffic": _ncu_traffic(name, shape), **({"note": note} if note else {})})

    qkv = rnd(M, 3 * D)
    tensor("attention", "attention_tc_kernel", {"B": B, "T": T, "H": H}, 4.0 * B * T * T * D,
           lambda: _ops.attention(qkv, B, T, D, H))
    xln = rnd(M, D)
    for nm, N, act in (("qkv", 3 * D, 0), ("fc1", 4 * D, 1)):
        w = rnd(N, D, std=0.02)
        bias = torch.zeros(N, device=dev)
        o = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        tensor(nm, f"gemm_tc_kernel<{BACKBONE_BN},64>" + (" +GELU" if act else ""), {"M": M, "N": N, "K": D},
               2.0 * M * N * D, lambda w=w, bias=bias, o=o, act=act: _ops.linear(xln, w, bias=bias, out=o, act=act,
                                                                                 bn=BACKBONE_BN))
    if D == 384 and (M + 127) // 128 >= 100:
        resid = rnd(M, D, dtype=torch.float32)
        lw, lb = torch.ones(D, device=dev), torch.zeros(D, device=dev)
        ls = torch.full((D,), 0.1, device=dev)
        for nm, K in (("proj_resid_ln", D), ("fc2_resid_ln", 4 * D)):
            a_ = rnd(M, K)
            w = rnd(D, K, std=0.02)
            bias = torch.zeros(D, device=dev)
            tensor(nm, "gemm_resid_ln_kernel", {"M": M, "N": D, "K": K}, 2.0 * M * D * K,
                   lambda a_=a_, w=w, bias=bias: _ops.linear_resid_ln(a_, w, bias, ls, resid, lw, lb, 1e-6))
            # the same kernel against HBM: A, W, old + new fp32 residual, bf16 LN output
            out[-1]["hbm_bytes"] = M * K * 2 + D * K * 2 + M * D * (4 + 4 + 2)
            out[-1]["hbm_frac"] = out[-1]["hbm_bytes"] / (out[-1]["duration_us"] * 1e-6) / 1e9 / peaks["hbm"]
    # DPT head (the engine's kernels): conv1 of the x2 resize and conv2 of the resize to R x R, each
    # with the resize built in shared memory (conv_up_kernel), conv2 with the fused 1x1 + ReLU depth
    # epilogue; algorithmic work = the two 3x3 convolutions at their output resolution
    F = eng.cfg.dpt.fusion
    Fh = F // 2
    S = 4 * (R // 14)
    if F == 64:
        po = rnd(B, S, S, F)
        w1 = rnd(Fh, 9 * F, std=0.05)
        w1p = _ops.conv_up_pack(w1)
        b1 = torch.zeros(Fh, device=dev)
        o1 = torch.empty(B, 2 * S, 2 * S, Fh, device=dev, dtype=torch.bfloat16)
        tensor("dpt_head1_conv_up", "conv_up_kernel<32,8,2>", {"B": B, "Hs": S, "Ho": 2 * S, "C": F, "N": Fh},
               2.0 * B * (2 * S) ** 2 * Fh * 9 * F,
               lambda: _ops.conv_up(po, w1, 2 * S, 2 * S, bias=b1, out=o1, wpack=w1p))
        h1 = rnd(B, 2 * S, 2 * S, Fh)
        w2 = rnd(32, 9 * Fh, std=0.05)
        w2p = _ops.conv_up_pack(w2)
        b2 = torch.zeros(32, device=dev)
        w3 = torch.randn(32, generator=g).to(dev) * 0.1
        dep = torch.empty(B, R, R, device=dev)
        tensor("dpt_head2_conv_up", "conv_up_kernel<32,4,4> +depth", {"B": B, "Hs": 2 * S, "Ho": R, "C": Fh, "N": 32},
               2.0 * B * R * R * 32 * 9 * Fh,
               lambda: _ops.conv_up(h1, w2, R, R, bias=b2, w3=w3, b3=0.1, out=dep, wpack=w2p))
    x2 = rnd(B, S, S, F)
    w2 = rnd(F, 9 * F, std=0.05)
    b2 = torch.zeros(F, device=dev)
    o2 = torch.empty(B, S, S, F, device=dev, dtype=torch.bfloat16)
    tensor("dpt_rcu_conv", "conv_halo_kernel<64,8,2,1>", {"B": B, "H": S, "C": F, "N": F},
           2.0 * B * S * S * F * 9 * F, lambda: _ops.conv(x2, w2, F, 3, bias=b2, out=o2))
    # seg: fused upsample + argmax, logits read once, u8 labels written
    h = R // 14
    C = eng.cfg.seg_classes
    cp = (C + 31) // 32 * 32
    # the engine's own seg logits (class pruning depends on the data: uncorrelated random logits
    # keep ~5x more candidate classes per block than the seeded head on backbone features)
    lg = torch.zeros(B, h * h, cp, device=dev)
    if "seg" in eng.heads:  # ring slot 0 holds a frame's `final` tap once the engine has run
        lab = torch.empty(B, R, R, device=dev, dtype=torch.uint8)
        lc = torch.empty(B, h * h, C, device=dev)
        eng.heads["seg"].forward(eng.channel.group_views(0)[eng.labels[-1]], lab, lc)
        lg[..., :C] = lc
    else:
        lg = rnd(B, h * h, cp, dtype=torch.float32)
    torch.cuda.synchronize()
    hbm("seg_upsample_argmax", "seg_upsample_argmax_pruned_kernel", {"B": B, "h": h, "C": C},
        B * (h * h * cp * 4 + R * R), lambda: _ops.upsample_argmax(lg, h, R, classes=C),
        note="issue-bound: per 7x7 block the classes whose corner range can reach the max, then the "
             "exact per-pixel bilinear + argmax over those")
    xr = rnd(M, D, dtype=torch.float32)
    lw, lb = torch.ones(D, device=dev), torch.zeros(D, device=dev)
    hbm("layernorm", "layernorm_kernel", {"M": M, "D": D}, M * D * (4 + 2), lambda: _ops.layernorm(xr, lw, lb))
    # every backbone class launches once per layer: the longest one dominates the step
    dom = max((r for r in out if r["class"] in ("attention", "qkv", "fc1", "proj_resid_ln", "fc2_resid_ln")),
              key=lambda r: r["duration_us"])
    return dom, out


def parity_e2e(eng, W, nframes=2):
    """End-to-end agreement (bf16 GPU pipeline vs the fp32 CPU oracle from the same u8 frames),
    reported beside the stage-wise bars the tests enforce: depth rel-L2,
    seg argmax agreement overall and on pixels whose oracle top-2 margin >= 1e-2, det top-100
    index overlap."""
    import torch
    from oracle import det as odet
    from oracle import dpt as odpt
    from oracle import seg as oseg
    from oracle import vit as ovit
    from paper_2508_11584_b200.weights import make_frames
    cfg, R, B = eng.cfg, eng.resolution, eng.batch
    frames = torch.cat([make_frames(1, R, stream_id=s) for s in range(B)], 0)
    # submit the same frame set until every head has run on it: with frame-ratio gates (C3: seg
    # 1:2, det 1:4) a single submit leaves the skipped heads' outputs from an earlier frame set
    pinned = frames.contiguous().pin_memory()
    done = set()
    for _ in range(16):
        done |= set(eng.submit(pinned))
        if done >= set(eng.out):
            break
    eng.synchronize()
    out = {n: {k: t.clone() for k, t in o.items()} for n, o in eng.out.items()}
    h = R // 14
    res = {"frames": nframes, "depth_rel_l2": [], "seg_agreement": [], "seg_agreement_margin_1e-2": [],
           "seg_margin_pixel_frac": [], "det_top100_overlap": [], "det_top100_identical": []}
    bb = cfg.backbone
    with torch.no_grad():
        for b in range(nframes):
            taps = ovit.backbone_forward(frames[b:b + 1], W, bb.depth, bb.heads, bb.taps)
            d = odpt.dpt_forward(taps, W, cfg.dpt.factors, h)
            g = out["depth"]["depth"][b:b + 1].cpu()
            res["depth_rel_l2"].append(((g - d).norm() / d.norm()).item())
            lab, _, up = oseg.seg_forward(taps[-1], W, h, R, return_logits=True)
            top2 = up.topk(2, dim=1).values
            margin = (top2[:, 0] - top2[:, 1])[0]
            agree = out["seg"]["labels"][b].cpu() == lab[0]
            m = margin >= 1e-2
            res["seg_agreement"].append(agree.float().mean().item())
            res["seg_agreement_margin_1e-2"].append(agree[m].float().mean().item())
            res["seg_margin_pixel_frac"].append(m.float().mean().item())
            ref = odet.det_forward(taps[-1], W, h, R, cfg.det)[0]["index"]
            k = int(out["det"]["count"][b])
            gi = out["det"]["index"][b, :k].cpu()
            res["det_top100_overlap"].append(len(set(gi.tolist()) & set(ref.tolist())) / max(1, ref.numel()))
            res["det_top100_identical"].append(bool(torch.equal(gi, ref)))
    return res


def latency_mode(args, W, device):
    """Per-head p50 latency the paper's way (insert -> head output): one camera
    stream, batch 1, each frame submitted alone and completed before the next, CUDA events on the
    producer and head streams."""
    from paper_2508_11584_b200.engine import VPEngine
    from paper_2508_11584_b200.weights import make_frames
    eng = VPEngine(args.model, args.resolution, 1, device=device, weights=W)
    frames = make_frames(1, args.resolution, 0).to(eng.device)
    eng.pixels.copy_(frames[0:1])
    for _ in range(5):
        eng.submit()
    eng.synchronize()
    eng.latencies_ms()
    for _ in range(50):
        eng.submit(record_latency=True)
        eng.synchronize()
    lat = eng.latencies_ms()
    eng.close()
    return {n: statistics.median(v) for n, v in lat.items() if v}


def run_ours(args):
    import torch
    rank, world, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    from paper_2508_11584_b200 import _lib
    from paper_2508_11584_b200.config import model_config
    from paper_2508_11584_b200.engine import VPEngine
    from paper_2508_11584_b200.sharding import max_over_ranks, streams_for_rank, total_frames
    from paper_2508_11584_b200.weights import make_frames, make_weights

    cfg = model_config(args.model)
    W = make_weights(args.model)
    B, R = args.batch, args.resolution
    rates = dict(kv.split("=") for kv in args.rates.split(",") if kv) if args.rates else None
    eng = VPEngine(args.model, R, B, device=local, weights=W, rates=rates)
    # input pool larger than L2, cycled: distinct frames every step (camera stream ids sharded by rank)
    frame_bytes = B * 3 * R * R
    npool = max(4, (2 * L2_BYTES) // frame_bytes + 1)
    # this rank's camera streams (stream i -> GPU i mod world); each contributes batch-1 frames
    my_streams = streams_for_rank(B * world, rank, world)
    base = torch.cat([make_frames(1, R, stream_id=s) for s in my_streams], 0)
    pool_dev = torch.empty(npool, B, 3, R, R, dtype=torch.uint8, device=eng.device)
    for i in range(npool):
        pool_dev[i].copy_(torch.roll(base, shifts=i * 7, dims=-1))
    pool_host = torch.empty(min(npool, 64), B, 3, R, R, dtype=torch.uint8).pin_memory()
    pool_host.copy_(pool_dev[: pool_host.shape[0]].cpu())
    sp = eng.s_prod.handle

    def step_device(i, record_latency=True):
        # device-resident inputs: D2D into the engine's input buffer on the producer stream
        _lib.lib.vpe_memcpy_async(_lib.C.c_void_p(eng.pixels.data_ptr()),
                                  _lib.C.c_void_p(pool_dev[i % npool].data_ptr()), frame_bytes, _lib.C.c_void_p(sp))
        eng.submit(record_latency=record_latency)

    def step_device_nolat(i):
        step_device(i, record_latency=False)

    def timed(fn, steps, warm, seconds=None):
        """Device time of ``steps`` steps (or of as many as fit in ``seconds`` of wall time),
        max over ranks; returns (seconds, launches, steps)."""
        for i in range(warm):
            fn(i)
        eng.synchronize()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ext = torch.cuda.ExternalStream(sp)
        launches0 = _lib.lib.vpe_kernel_launches()
        eng.latencies_ms()
        ev0.record(ext)
        n = 0
        t0 = time.perf_counter()
        while True:
            fn(warm + n)
            n += 1
            if seconds is None and n >= steps:
                break
            if seconds is not None and time.perf_counter() - t0 >= seconds:
                break
        for s in eng.s_head.values():
            e = torch.cuda.Event()
            e.record(torch.cuda.ExternalStream(s.handle))
            ext.wait_event(e)
        ev1.record(ext)
        eng.synchronize()
        torch.cuda.synchronize()
        dt = ev0.elapsed_time(ev1) * 1e-3
        launches = _lib.lib.vpe_kernel_launches() - launches0
        dt = max_over_ranks(dt, dist, eng.device)
        return dt, launches, n

    clk = ClockSampler(local)
    with clk:
        dt, launches, _ = timed(step_device, args.steps, args.warmup)
    lat = eng.latencies_ms()
    value = world * B * args.steps / dt

    sustained = None
    if args.sustained_seconds > 0:
        clk_s = ClockSampler(local)
        with clk_s:
            dts, _, ns = timed(step_device_nolat, 0, 3, seconds=args.sustained_seconds)
        eng.latencies_ms()
        frames_all = total_frames(B * ns, dist, eng.device)
        sustained = {"value": frames_all / dts, "unit": UNIT, "seconds": dts, "frames": frames_all,
                     "steps_rank0": ns, "clocks": clk_s.summary()}

    # e2e: host pinned frames in, every head output read back to pinned host memory
    eng.enable_host_outputs()
    nh = pool_host.shape[0]

    def step_host(i):
        eng.submit(pool_host[i % nh], record_latency=False)

    dt_e2e, _, _ = timed(step_host, args.steps, args.warmup)
    e2e = world * B * args.steps / dt_e2e
    d2h = eng.host_output_bytes()
    peaks = measured_peaks()
    roof, classes, par = None, None, None
    if rank == 0:
        roof, classes = kernel_rooflines(eng, peaks)
        roof = dict(roof, peak_kind=f"{peaks['kind']} burst")
        try:
            par = parity_e2e(eng, W)
        except Exception as exc:  # reported, never fatal to the GPU number
            par = {"error": repr(exc)}
    cnt = eng.counters()
    eng.close()
    p50_latency = latency_mode(args, W, local) if rank == 0 else None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N = 1 figure
            try:
                cpu = cpu_baseline(args, cfg, W, args.cpu_seconds)
            except Exception as exc:  # reported, never fatal to the GPU number
                cpu = {"error": repr(exc)}
        flops = frame_flops(cfg, R)
        p50 = {n: (statistics.median(v) if v else None) for n, v in lat.items()}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_name(args),
                       "model": f"dinov2_{args.model}+dpt+linseg+rpn (random init, seeded)", "resolution": R,
                       "batch_per_gpu": B, "camera_streams_per_gpu": B, "global_batch": B * world,
                       "parallelism": f"replicas x{world} (streams sharded, no collective)",
                       "l2": f"input pool {npool * frame_bytes / 2**20:.0f} MiB > 126 MiB L2, cycled",
                       "ring_capacity": eng.capacity},
            "per_head_p50_ms": p50_latency,
            "per_head_p50_ms_note": "latency mode: 1 stream, batch 1, one frame in flight, insert->head done",
            "per_head_p50_ms_throughput_mode": p50,
            "frame_gflop": flops / 1e9,
            "achieved_tflops_step": flops * value / world / 1e12,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": frame_bytes, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "roofline": roof,
            "roofline_classes": classes,
            "sustained": sustained,
            "parity_e2e": par,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "ring": {"pushed": cnt.pushed, "drops": cnt.producer_drops, "evictions": cnt.evictions,
                     "consumed": cnt.consumed},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
