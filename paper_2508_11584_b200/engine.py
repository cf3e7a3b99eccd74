"""VPEngine on one B200: foundation (backbone) + heads over an HBM feature ring.

This is the B200 re-design of the reference's foundation loop / head loops
and of the paper's multi-process, CUDA-IPC/MPS deployment:

* one process per GPU; the backbone runs on a producer stream, each head on its own
  higher-priority stream (replaces MPS time-slicing between processes);
* the backbone writes its four tap features straight into a LATEST ring slot
  (``channels.create_channel`` over ``vpe_ring``) — the "middle buffer";
* each admitted head leases the newest slot, its stream waits on the slot's ready event, its
  CUDA graph reads the slot IN PLACE, and ``commit`` records a done event that the producer
  waits on before it overwrites the slot (WAR) — the paper's IPC copy becomes zero copies;
* per-head ``RateGate``s decide on the host which head graphs launch;
* all device work is replayed from CUDA graphs: one backbone graph per ring slot and one graph
  per (head, slot), because the slot pointers are baked into the TMA descriptors.
"""

from __future__ import annotations

import ctypes as C
import time

import torch

from . import _lib
from .arena import DType, TensorSpec, generate_namespace
from .backbone import Backbone
from .channels import ChannelMode, create_channel
from .config import grid, model_config, tokens
from .heads import DepthHead, DetHead, SegHead
from .pipeline import gate_admit, make_gate, set_rate
from .weights import make_weights
from ._lib import check, lib

HEAD_IDS = {"depth": 1, "seg": 2, "det": 3}
_DT = {torch.float32: DType.F32, torch.uint8: DType.U8, torch.int64: DType.I64, torch.int32: DType.I32,
       torch.bfloat16: DType.BF16}


class _Stream:
    def __init__(self, priority: int):
        h = C.c_void_p()
        check(lib.vpe_stream_create(priority, C.byref(h)))
        self.handle = h.value

    def sync(self):
        check(lib.vpe_stream_sync(C.c_void_p(self.handle)))

    def close(self):
        if self.handle:
            lib.vpe_stream_destroy(C.c_void_p(self.handle))
            self.handle = None


class _Graph:
    def __init__(self, stream: _Stream, fn):
        check(lib.vpe_graph_begin(C.c_void_p(stream.handle)), "graph_begin")
        try:
            fn()
        finally:
            g = C.c_void_p()
            rc = lib.vpe_graph_end(C.c_void_p(stream.handle), C.byref(g))
        check(rc, "graph_end")
        self.h = g

    def launch(self, stream: _Stream):
        check(lib.vpe_graph_launch(self.h, C.c_void_p(stream.handle)), "graph_launch")

    def close(self):
        if self.h:
            lib.vpe_graph_destroy(self.h)
            self.h = None


class _Event:
    def __init__(self):
        h = C.c_void_p()
        check(lib.vpe_event_create(C.byref(h)))
        self.h = h

    def record(self, stream: _Stream):
        check(lib.vpe_event_record(self.h, C.c_void_p(stream.handle)))

    def elapsed_ms(self, later: "_Event") -> float:
        ms = C.c_float()
        check(lib.vpe_event_elapsed_ms(self.h, later.h, C.byref(ms)))
        return ms.value


class VPEngine:
    def __init__(self, model: str = "vits14", resolution: int = 448, batch: int = 1,
                 heads=("depth", "seg", "det"), capacity: int | None = None, rates: dict | None = None,
                 device: int = 0, weights: dict | None = None, graphs: bool = True, seed: int = 0,
                 namespace: str | None = None, max_latency_records: int = 4096,
                 camera: tuple[int, int] | None = None, pdl: bool | None = None):
        torch.cuda.set_device(device)
        self.device = torch.device(f"cuda:{device}")
        # programmatic dependent launch (opt-in): shortens latency-bound small batches (backbone
        # 0.752 -> 0.695 ms at batch 1) but with it the outputs were observed to vary bitwise in
        # ~10% of replays (tools/pdl_determinism.py; csrc/util.cuh), so it is off by default
        self.pdl = False if pdl is None else bool(pdl)
        check(lib.vpe_set_pdl(int(self.pdl)), "vpe_set_pdl")
        self.cfg = model_config(model)
        self.model, self.resolution, self.batch = model, resolution, batch
        self.head_names = tuple(heads)
        bb = self.cfg.backbone
        self.T, self.D, self.h = tokens(resolution), bb.dim, grid(resolution)
        W = weights if weights is not None else make_weights(model, seed=seed, heads=self.head_names)
        self.backbone = Backbone(W, bb, resolution, batch, self.device)
        self.labels = bb.tap_labels
        self.heads = {}
        if "depth" in heads:
            self.heads["depth"] = DepthHead(W, self.cfg, resolution, batch, self.device)
        if "seg" in heads:
            self.heads["seg"] = SegHead(W, self.cfg, resolution, batch, self.device)
        if "det" in heads:
            self.heads["det"] = DetHead(W, self.cfg, resolution, batch, self.device)
        specs = [TensorSpec(lbl, DType.BF16, (batch, self.T, self.D)) for lbl in self.labels]
        self.capacity = capacity or (len(self.heads) + 2)
        self.namespace = namespace or generate_namespace()
        self.channel, self.handle = create_channel("features", ChannelMode.LATEST, self.capacity, specs,
                                                   self.namespace, expected_consumers=len(self.heads),
                                                   device=device)
        self.s_prod = _Stream(0)
        self.s_head = {n: _Stream(-1) for n in self.heads}
        for n in self.heads:
            self.channel.register_consumer(HEAD_IDS[n])
        now = time.monotonic_ns()
        rates = rates or {}
        self.gates = {}
        for n in self.heads:
            r = rates.get(n)
            if isinstance(r, str) and r.startswith("1:"):
                self.gates[n] = make_gate(every_n=int(r[2:]), now_ns=now)
            else:
                self.gates[n] = make_gate(rate_hz=r, now_ns=now)
        R, B, dev = resolution, batch, self.device
        # camera=(H, W): frames arrive as u8 HWC camera images; crop/resize/normalise run fused
        # into the patch embedding (vpe_vit_forward_camera) instead of expecting [B,3,R,R]
        self.camera = tuple(camera) if camera else None
        if self.camera:
            self.pixels = torch.zeros(B, self.camera[0], self.camera[1], 3, dtype=torch.uint8, device=dev)
        else:
            self.pixels = torch.zeros(B, 3, R, R, dtype=torch.uint8, device=dev)
        self.out = {}
        if "depth" in self.heads:
            self.out["depth"] = {"depth": torch.zeros(B, R, R, device=dev), "depth_pre": torch.zeros(B, R, R, device=dev)}
        if "seg" in self.heads:
            self.out["seg"] = {"labels": torch.zeros(B, R, R, dtype=torch.uint8, device=dev)}
        if "det" in self.heads:
            self.out["det"] = self.heads["det"].outputs()
        self._slot_of = {self.channel.group_views(i)[self.labels[-1]].data_ptr(): i for i in range(self.capacity)}
        self.graphs = graphs
        self._g_bb, self._g_head = {}, {}
        # eager warm-up binds every plan, then capture one graph per slot / (head, slot)
        torch.cuda.synchronize()
        for slot in range(self.capacity):
            self._backbone_into(slot)
            for n in self.heads:
                self._head_on(n, slot)
        self.s_prod.sync()
        for s in self.s_head.values():
            s.sync()
        if graphs:
            for slot in range(self.capacity):
                self._g_bb[slot] = _Graph(self.s_prod, lambda slot=slot: self._backbone_into(slot))
                for n in self.heads:
                    self._g_head[(n, slot)] = _Graph(self.s_head[n], lambda n=n, slot=slot: self._head_on(n, slot))
        self._fid = 0
        self._ev_pool = [_Event() for _ in range(max_latency_records * (1 + len(self.heads)))]
        self._ev_next = 0
        self._lat_records = []
        self.host_out = None
        self.fifo = None
        self.output_drops = {}
        self.dropped = 0

    # ------------------------------------------------------------------ enqueue primitives
    def _taps(self, slot):
        v = self.channel.group_views(slot)
        return [v[l] for l in self.labels]

    def _backbone_into(self, slot):
        if self.camera:
            self.backbone.forward_camera(self.pixels, self._taps(slot), stream=self.s_prod.handle)
        else:
            self.backbone.forward(self.pixels, self._taps(slot), stream=self.s_prod.handle)

    def _head_on(self, name, slot):
        taps = self._taps(slot)
        st = self.s_head[name].handle
        o = self.out[name]
        if name == "depth":
            self.heads[name].forward(taps, o["depth"], o["depth_pre"], stream=st)
        elif name == "seg":
            self.heads[name].forward(taps[-1], o["labels"], stream=st)
        else:
            self.heads[name].forward(taps[-1], o, stream=st)

    def _event(self):
        if self._ev_next >= len(self._ev_pool):
            return None
        e = self._ev_pool[self._ev_next]
        self._ev_next += 1
        return e

    def enable_host_outputs(self):
        """Pinned host mirrors of every head output (the e2e path's device->host read)."""
        self.host_out = {n: {k: torch.empty_like(t, device="cpu").pin_memory() for k, t in o.items()}
                         for n, o in self.out.items()}
        return self.host_out

    def host_output_bytes(self) -> int:
        if not self.host_out:
            return 0
        return sum(t.numel() * t.element_size() for o in self.host_out.values() for t in o.values())

    def enable_output_fifos(self, capacity: int = 8) -> dict:
        """Per-head output queue ("push to output FIFO"; channels.py:377-421): a FIFO
        channel whose slots live in pinned host memory. Each admitted head run pushes its outputs
        with stream-ordered D2H copies on the head stream (READY = copies enqueued + event); a host
        consumer ``pop``s them in order. A full queue rejects the frame (producer_drops)."""
        self.fifo = {}
        for n, o in self.out.items():
            specs = [TensorSpec(k, _DT[t.dtype], tuple(t.shape)) for k, t in o.items()]
            ch, _ = create_channel(f"out-{n}", ChannelMode.FIFO, capacity, specs, self.namespace, device=-1)
            ch.register_consumer(1)
            self.fifo[n] = ch
        return self.fifo

    def pop_output(self, head: str, block: bool = True, timeout: float | None = 5.0):
        """Oldest queued output of ``head`` as host tensors, or None (channels.py:377-407)."""
        ch = self.fifo[head]
        dst = {s.label: torch.empty(s.dims, dtype=s.dtype.torch_dtype) for s in ch.specs}
        env = ch.pop(1, dst, block=block, timeout=timeout)
        return None if env is None else (env.frame_id, dst)

    # ------------------------------------------------------------------ one frame set
    def submit(self, host_frames: torch.Tensor | None = None, capture_ts: int | None = None,
               record_latency: bool = False) -> dict:
        """Foundation step + every admitted head, all asynchronous. ``host_frames`` (pinned u8
        [B,3,R,R]) is copied H2D on the producer stream first; otherwise ``self.pixels`` is used."""
        self._fid += 1
        fid = self._fid
        ts = capture_ts if capture_ts is not None else time.monotonic_ns()
        sp = self.s_prod
        if host_frames is not None:
            check(lib.vpe_memcpy_async(C.c_void_p(self.pixels.data_ptr()), C.c_void_p(host_frames.data_ptr()),
                                       self.pixels.numel(), C.c_void_p(sp.handle)))
        ev_in = self._event() if record_latency else None
        if ev_in is not None:
            ev_in.record(sp)

        def writer(views):
            slot = self._slot_of[views[self.labels[-1]].data_ptr()]
            if self.graphs:
                self._g_bb[slot].launch(sp)
            else:
                self._backbone_into(slot)

        outcome = self.channel.push(fid, ts, writer, stream=sp.handle)
        if not outcome.accepted:
            self.dropped += 1
        ran = {}
        now = time.monotonic_ns()
        for n in self.heads:
            if not gate_admit(self.gates[n], now):
                continue
            st = self.s_head[n]
            lease = self.channel.acquire_latest(HEAD_IDS[n], stream=st.handle)
            if lease is None:
                continue
            if self.graphs:
                self._g_head[(n, lease.slot_index)].launch(st)
            else:
                self._head_on(n, lease.slot_index)
            if self.host_out is not None:
                for k, t in self.out[n].items():
                    check(lib.vpe_memcpy_async(C.c_void_p(self.host_out[n][k].data_ptr()), C.c_void_p(t.data_ptr()),
                                               t.numel() * t.element_size(), C.c_void_p(st.handle)))
            if self.fifo is not None:
                outs = self.out[n]

                def out_writer(views, outs=outs, st=st):
                    for k, t in outs.items():
                        check(lib.vpe_memcpy_async(C.c_void_p(views[k].data_ptr()), C.c_void_p(t.data_ptr()),
                                                   t.numel() * t.element_size(), C.c_void_p(st.handle)))

                if not self.fifo[n].push(lease.frame_id, lease.capture_ts, out_writer, stream=st.handle).accepted:
                    self.output_drops[n] = self.output_drops.get(n, 0) + 1
            ev = self._event() if record_latency else None
            if ev is not None:
                ev.record(st)
            self.channel.commit(lease, stream=st.handle)
            ran[n] = lease.frame_id
            if ev_in is not None and ev is not None:
                self._lat_records.append((n, ev_in, ev))
        return ran

    def synchronize(self):
        self.s_prod.sync()
        for s in self.s_head.values():
            s.sync()

    def run(self, frames: torch.Tensor) -> dict:
        """Synchronous convenience: one frame set (u8 [B,3,R,R], host or device) -> outputs."""
        if frames.is_cuda:
            self.pixels.copy_(frames)
            torch.cuda.synchronize()
            self.submit()
        else:
            self.submit(frames.contiguous().pin_memory() if not frames.is_pinned() else frames)
        self.synchronize()
        return {n: {k: t.clone() for k, t in o.items()} for n, o in self.out.items()}

    def set_rate(self, head: str, hz=None, every_n: int | None = None):
        set_rate(self.gates, head, hz, time.monotonic_ns(), every_n=every_n)

    def latencies_ms(self) -> dict[str, list[float]]:
        out = {n: [] for n in self.heads}
        for n, a, b in self._lat_records:
            out[n].append(a.elapsed_ms(b))
        self._lat_records = []
        self._ev_next = 0
        return out

    def counters(self):
        return self.channel.counters()

    def close(self):
        for g in list(self._g_bb.values()) + list(self._g_head.values()):
            g.close()
        self._g_bb, self._g_head = {}, {}
        for h in self.heads.values():
            h.close()
        self.backbone.close()
        self.channel.close()
        for ch in (self.fifo or {}).values():
            ch.close()
        self.fifo = None
