"""The reference's CPU path for the hot path (TEST/BASELINE INFRASTRUCTURE ONLY).

Transport: the UNMODIFIED reference ``fanpipe`` (``baseline/_ref``, pip-installed from
/root/reference/pkg; compiled Cython atomics) — one LATEST channel carrying the four tap
labels, the foundation ``push``es with a writer, each head ``acquire_latest`` + ``consume``s
its label subset into processing slots (channels.py:274, 423, 454) — exactly the paper's
FM -> middle buffer -> heads data flow.
Compute: the fp32 oracle restatements (the reference has no NN code) on all host
threads. Used by bench.py's ``cpu_baseline`` leg and ``--impl reference``.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np
import torch

from . import det as odet
from . import dpt as odpt
from . import seg as oseg
from . import vit as ovit

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def load_fanpipe():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import fanpipe  # noqa: F401
    from fanpipe import arena, channels
    return arena, channels


class CpuPipeline:
    """Sequential single-process foundation + 3 heads over a fanpipe LATEST channel."""

    def __init__(self, cfg, W, resolution: int, batch: int = 1, heads=("depth", "seg", "det"),
                 threads: int | None = None):
        self.cfg, self.W, self.R, self.B = cfg, W, resolution, batch
        self.heads = tuple(heads)
        self.threads = threads or os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        bb = cfg.backbone
        self.h = resolution // 14
        T = self.h * self.h + 1
        self.labels = bb.tap_labels
        self.ar, self.ch = load_fanpipe()
        self.ns = self.ar.generate_namespace("vpref")
        specs = [self.ar.TensorSpec(lbl, self.ar.DType.F32, (batch, T, bb.dim)) for lbl in self.labels]
        self.chan, _ = self.ch.create_channel("features", self.ch.ChannelMode.LATEST, len(self.heads) + 2, specs,
                                              self.ns, expected_consumers=len(self.heads))
        self.cids = {n: i + 1 for i, n in enumerate(self.heads)}
        self.dst = {}
        for n in self.heads:
            self.chan.register_consumer(self.cids[n])
            want = self.labels if n == "depth" else (self.labels[-1],)
            self.dst[n] = (want, self.ch.create_processing_slots(
                self.ns, f"proc-{n}", [s for s in specs if s.label in want]))
        self.fid = 0

    def step(self, frames_u8: torch.Tensor) -> dict:
        bb = self.cfg.backbone
        taps = ovit.backbone_forward(frames_u8, self.W, bb.depth, bb.heads, bb.taps)
        self.fid += 1

        def writer(views):
            for lbl, t in zip(self.labels, taps):
                np.copyto(views[lbl], t.numpy())

        self.chan.push(self.fid, time.monotonic_ns(), writer)
        out = {}
        for n in self.heads:
            lease = self.chan.acquire_latest(self.cids[n])
            want, grp = self.dst[n]
            self.chan.consume(lease, grp, want)
            feats = [torch.from_numpy(grp.view(l)) for l in want]
            if n == "depth":
                out[n] = odpt.dpt_forward(feats, self.W, self.cfg.dpt.factors, self.h)
            elif n == "seg":
                out[n] = oseg.seg_forward(feats[0], self.W, self.h, self.R)
            else:
                out[n] = odet.det_forward(feats[0], self.W, self.h, self.R, self.cfg.det)
        return out

    def close(self):
        try:
            for _, grp in self.dst.values():  # drop the ndarray views first: they pin the mmap
                grp._views.clear()
                grp.arena.close()
            self.dst.clear()
            self.chan._group_views.clear()
            self.chan.close()
            self.chan.unlink()
            self.ar.clean_namespace(self.ns)
        except Exception:
            pass


# ---------------------------------------------------------------------------------------------
# Variant (ii) of SURVEY §8d: the paper's deployment on the CPU — one foundation process and one
# process per head over the reference's cross-process LATEST channel, torch
# threads split across the processes in proportion to their measured work.
_WORK = {"foundation": 168.0, "depth": 88.0, "seg": 79.0, "det": 15.0}  # SURVEY App. A.7 (ms, C2)


def _split_threads(total: int, roles) -> dict:
    w = {r: _WORK.get(r, 50.0) for r in roles}
    s = sum(w.values())
    out = {r: max(1 if total < 8 else 2, int(round(total * w[r] / s))) for r in roles}
    while sum(out.values()) > total and max(out.values()) > 1:
        out[max(out, key=out.get)] -= 1
    return out


def _mp_foundation(model, R, threads, hdict, barrier, stop, result):
    torch.set_num_threads(threads)
    from paper_2508_11584_b200.config import model_config
    from paper_2508_11584_b200.weights import make_frames, make_weights
    ar, ch = load_fanpipe()
    cfg = model_config(model)
    W = make_weights(model)
    chan = ch.open_channel(ch.ChannelHandle.from_dict(hdict))
    bb = cfg.backbone
    frames = make_frames(1, R, 0)
    ovit.backbone_forward(frames, W, bb.depth, bb.heads, bb.taps)  # warm-up
    barrier.wait()
    fid = 0
    while not stop.is_set():
        taps = ovit.backbone_forward(frames, W, bb.depth, bb.heads, bb.taps)
        fid += 1

        def writer(views, taps=taps):
            for lbl, t in zip(bb.tap_labels, taps):
                np.copyto(views[lbl], t.numpy())

        chan.push(fid, time.monotonic_ns(), writer)
    _finish(result, ("foundation", fid))


def _finish(result, item):
    # the reference's arena raises BufferError from __del__ at interpreter exit while numpy
    # views are alive (fanpipe/arena.py:269-276): hand the result over, then leave quietly
    result.put(item)
    result.close()
    result.join_thread()
    os._exit(0)


def _mp_head(model, R, name, cid, threads, hdict, barrier, stop, result):
    torch.set_num_threads(threads)
    from paper_2508_11584_b200.config import model_config
    from paper_2508_11584_b200.weights import make_weights
    ar, ch = load_fanpipe()
    cfg = model_config(model)
    W = make_weights(model)
    handle = ch.ChannelHandle.from_dict(hdict)
    chan = ch.open_channel(handle)
    chan.register_consumer(cid)
    labels = cfg.backbone.tap_labels if name == "depth" else (cfg.backbone.tap_labels[-1],)
    specs = [s for s in handle.specs if s.label in labels]
    ns = handle.namespace
    grp = ch.create_processing_slots(ns, f"proc-{name}", specs)
    h = R // 14

    def compute(feats):
        if name == "depth":
            return odpt.dpt_forward(feats, W, cfg.dpt.factors, h)
        if name == "seg":
            return oseg.seg_forward(feats[0], W, h, R)
        return odet.det_forward(feats[0], W, h, R, cfg.det)

    compute([torch.zeros(s.dims) for s in specs])  # warm-up
    barrier.wait()
    done = []
    while not stop.is_set():
        lease = chan.acquire_latest(cid)
        if lease is None:
            time.sleep(0.0005)
            continue
        chan.consume(lease, grp, labels)
        compute([torch.from_numpy(grp.view(l)) for l in labels])
        done.append(lease.frame_id)
    _finish(result, (name, done))


def multiprocess_pipeline(model: str, R: int, seconds: float, threads: int | None = None,
                          heads=("depth", "seg", "det")) -> dict:
    """Run the foundation + head processes for ``seconds`` and return the rates: fps of
    complete perception outputs = min over heads of outputs / s (a LATEST head skips frames it
    cannot keep up with, as in the paper), the foundation's frame rate and per-head rates."""
    import multiprocessing as mp
    from paper_2508_11584_b200.config import model_config
    threads = threads or os.cpu_count() or 1
    roles = ("foundation",) + tuple(heads)
    split = _split_threads(threads, roles)
    ar, ch = load_fanpipe()
    cfg = model_config(model)
    T = (R // 14) ** 2 + 1
    specs = [ar.TensorSpec(l, ar.DType.F32, (1, T, cfg.backbone.dim)) for l in cfg.backbone.tap_labels]
    ns = ar.generate_namespace("vpmp")
    chan, handle = ch.create_channel("features", ch.ChannelMode.LATEST, len(heads) + 2, specs, ns,
                                     expected_consumers=len(heads))
    ctx = mp.get_context("spawn")
    barrier, stop, result = ctx.Barrier(len(roles) + 1), ctx.Event(), ctx.Queue()
    hd = handle.to_dict()
    procs = [ctx.Process(target=_mp_foundation, args=(model, R, split["foundation"], hd, barrier, stop, result))]
    for i, n in enumerate(heads):
        procs.append(ctx.Process(target=_mp_head, args=(model, R, n, i + 1, split[n], hd, barrier, stop, result)))
    for p in procs:
        p.start()
    try:
        barrier.wait(timeout=600)
        t0 = time.perf_counter()
        time.sleep(seconds)
        stop.set()
        dt = time.perf_counter() - t0
        got = dict(result.get(timeout=600) for _ in procs)
    finally:
        stop.set()
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
        try:
            chan._group_views.clear()
            chan.close()
            chan.unlink()
        except Exception:
            pass
        ar.clean_namespace(ns)
    rates = {n: len(got[n]) / dt for n in heads}
    return {"fps": min(rates.values()), "foundation_fps": got["foundation"] / dt, "head_fps": rates,
            "seconds": dt, "threads": split}
