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
