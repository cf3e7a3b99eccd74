"""VPEngine on one B200: foundation (backbone) + heads over an HBM feature ring.

This is the B200 re-design of the reference's foundation loop / head loops,
its control module and of the paper's multi-process, CUDA-IPC/MPS deployment
(PAPER.md:95-121):

* one process per GPU; the backbone runs on a producer stream, each head on its own
  higher-priority stream (replaces MPS time-slicing between processes; VPE_PRIO overrides);
* the backbone writes its four tap features straight into a LATEST ring slot
  (``channels.create_channel`` over ``vpe_ring``) — the "middle buffer";
* each admitted head leases the newest slot, its stream waits on the slot's ready event, its
  CUDA graph reads the slot IN PLACE, and ``commit`` records a done event that the producer
  waits on before it overwrites the slot (WAR) — the paper's IPC copy becomes zero copies;
* per-head ``RateGate``s decide on the host which head graphs launch;
* all device work is replayed from CUDA graphs: one backbone graph per ring slot and one graph
  per (head, slot), because the slot pointers are baked into the TMA descriptors.

Two ways to drive it:

* ``submit()`` — one host thread enqueues the foundation step and every admitted head for one
  frame set, fully asynchronous (throughput mode: the producer stream is back-pressured by the
  heads' done events; every admitted head runs on every frame). ``bench.py`` uses this.
* ``start()`` / ``stop()`` — decentralized mode (PAPER.md "Decentralization"):
  a foundation thread paced by the frame source and one host thread per head, each running the
  SPEC head loop (gate -> acquire_latest -> run in place -> wait for its own completion ->
  commit -> output FIFO). A head holds its lease while its kernels run, so a slow, stalled or
  failed head never blocks the producer or the other heads (the producer evicts other slots).

Both are steered by ``dispatch()`` with SPEC's textual commands (``SETRATE``, ``PAUSE``,
``RESUME``, ``STOP``, ``STATS``, ``FAULT``; control.py serves them on a local socket).
Engines are built from explicit arguments or from registry model cards (``from_cards``).
"""

from __future__ import annotations

import collections
import ctypes as C
import os
import json
import logging
import threading
import time

import torch

from .arena import DType, TensorSpec, allocation_audit, copy_counter, generate_namespace
from .backbone import Backbone
from .channels import ChannelMode, create_channel
from .config import BACKBONES, grid, model_config, tokens
from .errors import ConfigError, EngineError, NotFound, ProtocolError, ShapeError
from .heads import BUILTIN_HEADS, HEAD_BACKENDS, WEIGHT_GROUP
from .pipeline import gate_admit, make_gate, set_rate
from .weights import make_weights
from ._lib import check, lib

log = logging.getLogger("vpe.engine")

_DT = {torch.float32: DType.F32, torch.uint8: DType.U8, torch.int64: DType.I64, torch.int32: DType.I32,
       torch.bfloat16: DType.BF16}
_TORCH_DT = {v: k for k, v in _DT.items()}

# worker states (SPEC.md:336-338 EngineStatus: Starting -> Running -> {Paused <-> Running, Failed, Stopped})
STARTING, RUNNING, PAUSED, FAILED, STOPPED = "Starting", "Running", "Paused", "Failed", "Stopped"


class InjectedFault(EngineError):
    """The FAULT control command: a panic inside a head worker."""


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

    def sync(self):
        check(lib.vpe_event_sync(self.h))

    def elapsed_ms(self, later: "_Event") -> float:
        ms = C.c_float()
        check(lib.vpe_event_elapsed_ms(self.h, later.h, C.byref(ms)))
        return ms.value

    def close(self):
        if self.h:
            lib.vpe_event_destroy(self.h)
            self.h = None


class HeadWorker:
    """Runtime state of one head: its backend, stream, gate, outputs and SPEC worker status."""

    def __init__(self, name: str, kind: str, cid: int, backend, stream: _Stream, gate, outs: dict):
        self.name, self.kind, self.cid = name, kind, cid
        self.backend, self.stream, self.gate, self.out = backend, stream, gate, outs
        self.labels = backend.subscriptions()
        self.state = STARTING
        self.iterations = 0   # gate admissions that led to a lease
        self.outputs = 0      # completed head runs
        self.errors = 0       # backend failures (skip-and-count)
        self.last_frame = 0
        self.fault = False    # FAULT pending: the next run panics
        self.stall_s = 0.0    # test hook: hold the next lease this long before running (SIGSTOP analog)
        self.history = collections.deque(maxlen=4096)  # frame ids of completed outputs (provenance)
        self.done_evt = None
        self.thread = None
        self.resume = threading.Event()
        self.resume.set()

    def status(self) -> dict:
        g = self.gate
        rate = f"1:{g.every_n}" if g.every_n else (None if g.rate_hz is None else float(g.rate_hz))
        return {"state": self.state, "kind": self.kind, "rate": rate, "iterations": self.iterations,
                "outputs": self.outputs, "errors": self.errors, "last_frame": self.last_frame}


def _parse_rate(r):
    """None / "unlimited" -> Unlimited; "1:n" -> frame-ratio gate; number -> Hz."""
    if r is None or (isinstance(r, str) and r.lower() in ("unlimited", "none", "inf")):
        return None, None
    if isinstance(r, str) and r.startswith("1:"):
        n = int(r[2:])
        if n < 1:
            raise ConfigError(f"bad frame ratio {r!r}")
        return None, n
    hz = float(r)
    if not hz > 0:
        raise ConfigError(f"rate must be positive, got {r}")
    return hz, None


class VPEngine:
    def __init__(self, model: str = "vits14", resolution: int = 448, batch: int = 1,
                 heads=("depth", "seg", "det"), capacity: int | None = None, rates: dict | None = None,
                 device: int = 0, weights: dict | None = None, graphs: bool = True, seed: int = 0,
                 namespace: str | None = None, max_latency_records: int = 4096,
                 camera: tuple[int, int] | None = None, pdl: bool | None = None,
                 debug_outputs: bool = False, shared: bool = False):
        """``heads``: short names of the paper's example heads ("depth", "seg", "det") or
        (name, backend kind) pairs; ``rates``: head -> Hz, "1:n" (frame ratio) or None
        (Unlimited); ``debug_outputs`` adds the pre-final-ReLU depth map (parity grading only);
        ``shared`` exports the ring for out-of-process consumers (channels.open_channel)."""
        torch.cuda.set_device(device)
        self.device = torch.device(f"cuda:{device}")
        # programmatic dependent launch with late release (each persistent backbone kernel lets
        # its dependent launch after its last TMA load): batch-1 p50 depth 1.01 -> 0.94 ms, C2
        # batch 16 5272 -> 5380 fps (csrc/util.cuh); outputs bit-identical (tools/pdl_determinism.py)
        self.pdl = True if pdl is None else bool(pdl)
        check(lib.vpe_set_pdl(2 if self.pdl else 0), "vpe_set_pdl")
        self.cfg = model_config(model)
        self.model, self.resolution, self.batch = model, resolution, batch
        head_specs = [(h, BUILTIN_HEADS[h]) if isinstance(h, str) else (str(h[0]), str(h[1])) for h in heads]
        if len({n for n, _ in head_specs}) != len(head_specs):
            raise ConfigError(f"duplicate head names in {head_specs}")
        for n, k in head_specs:
            if k not in HEAD_BACKENDS:
                raise ConfigError(f"head {n!r}: unknown backend kind {k!r}; have {sorted(HEAD_BACKENDS)}")
        self.head_names = tuple(n for n, _ in head_specs)
        bb = self.cfg.backbone
        self.T, self.D, self.h = tokens(resolution), bb.dim, grid(resolution)
        W = weights if weights is not None else make_weights(
            model, seed=seed, heads=tuple({WEIGHT_GROUP[k] for _, k in head_specs}))
        self.backbone = Backbone(W, bb, resolution, batch, self.device)
        self.labels = bb.tap_labels
        self.heads = {n: HEAD_BACKENDS[k](W, self.cfg, resolution, batch, self.device) for n, k in head_specs}
        specs = [TensorSpec(lbl, DType.BF16, (batch, self.T, self.D)) for lbl in self.labels]
        self.capacity = capacity or (len(self.heads) + 2)
        self.namespace = namespace or generate_namespace()
        self.channel, self.handle = create_channel("features", ChannelMode.LATEST, self.capacity, specs,
                                                   self.namespace, expected_consumers=len(self.heads),
                                                   device=device, shared=shared)
        # stream priorities (lower = higher), VPE_PRIO="prod,head": heads above the producer, so
        # an admitted head is never queued behind the next frame's backbone (equal priorities
        # measured 1% more C2 throughput, 5514 vs 5454 fps, and the same latency-mode p50)
        prio = [int(v) for v in os.environ.get("VPE_PRIO", "0,-1").split(",")]
        self.s_prod = _Stream(prio[0])
        self.s_head = {n: _Stream(prio[1]) for n in self.heads}
        now = time.monotonic_ns()
        rates = dict(rates or {})
        unknown = set(rates) - set(self.heads)
        if unknown:
            raise NotFound(f"rates given for unknown heads {sorted(unknown)}")
        self.gates = {}
        for n in self.heads:
            hz, every = _parse_rate(rates.get(n))
            self.gates[n] = make_gate(rate_hz=hz, every_n=every, now_ns=now)
        R, B, dev = resolution, batch, self.device
        # camera=(H, W): frames arrive as u8 HWC camera images; crop/resize/normalise run fused
        # into the patch embedding (vpe_vit_forward_camera) instead of expecting [B,3,R,R]
        self.camera = tuple(camera) if camera else None
        if self.camera:
            self.pixels = torch.zeros(B, self.camera[0], self.camera[1], 3, dtype=torch.uint8, device=dev)
        else:
            self.pixels = torch.zeros(B, 3, R, R, dtype=torch.uint8, device=dev)
        self.out = {n: hd.outputs(debug=debug_outputs) for n, hd in self.heads.items()}
        self.workers = {}
        for i, (n, k) in enumerate(head_specs):
            self.workers[n] = HeadWorker(n, k, i + 1, self.heads[n], self.s_head[n], self.gates[n], self.out[n])
            self.channel.register_consumer(i + 1)
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
        for w in self.workers.values():
            w.done_evt = _Event()
            w.state = RUNNING
        self._fid = 0
        self._ev_pool = [_Event() for _ in range(max_latency_records * (1 + len(self.heads)))]
        self._ev_next = 0
        self._lat_records = []
        self.host_out = None
        self.fifo = None
        self.output_drops = {}
        self.dropped = 0
        self.fm_state, self.fm_errors, self.fm_iterations = RUNNING, 0, 0
        self.source_skips = 0
        self._t0 = time.monotonic()
        self._threads_on = False
        self._stop = threading.Event()
        self._new_frame = threading.Condition()
        self._closed = False
        self.cards = None

    # ------------------------------------------------------------------ construction from cards
    @classmethod
    def from_cards(cls, fm, heads, rates: dict | None = None, device: int = 0, weights: dict | None = None,
                   seed: int = 0, **kw) -> "VPEngine":
        """Deploy registry model cards: the foundation card must describe the
        b200_vit backend's four tap outputs, every head card must pass ``validate_deployment``
        against it and name a known backend kind, and the head outputs the card declares must be
        what that backend produces. Rates: ``rates[name]`` overrides the card's default_rate."""
        from .registry import validate_deployment
        if fm.kind != "foundation":
            raise ConfigError(f"{fm.name}: expected a foundation card, got kind {fm.kind!r}")
        if fm.backend.get("kind") != "b200_vit":
            raise ConfigError(f"{fm.name}: foundation backend must be b200_vit, got {fm.backend.get('kind')!r}")
        model = fm.backend.get("model")
        if model is None:
            cand = [n for n, b in BACKBONES.items()
                    if b.dim == fm.backend.get("dim") and b.depth == fm.backend.get("depth")]
            if len(cand) != 1:
                raise ConfigError(f"{fm.name}: cannot tell the backbone from backend {fm.backend}")
            model = cand[0]
        if model not in BACKBONES:
            raise ConfigError(f"{fm.name}: unknown backbone {model!r}")
        if len(fm.input_specs) != 1 or fm.input_specs[0].dtype is not DType.U8 or len(fm.input_specs[0].dims) != 4:
            raise ConfigError(f"{fm.name}: input must be one u8 [B,3,R,R] image spec")
        B, _, R, R2 = fm.input_specs[0].dims
        R = int(fm.backend.get("resolution", R))
        if R2 != R:
            raise ConfigError(f"{fm.name}: non-square input {fm.input_specs[0].dims}")
        bb = BACKBONES[model]
        want = {lbl: TensorSpec(lbl, DType.BF16, (B, tokens(R), bb.dim)) for lbl in bb.tap_labels}
        have = {s.label: s for s in fm.output_specs}
        if have != want:
            raise ConfigError(f"{fm.name}: outputs {sorted(have)} do not match the b200_vit taps "
                              f"{[(s.label, s.dtype.value, s.dims) for s in want.values()]}")
        for h in heads:
            if h.kind != "head":
                raise ConfigError(f"{h.name}: expected a head card, got kind {h.kind!r}")
        report = validate_deployment(fm, list(heads))
        if report:
            m = report[0]
            raise ConfigError(f"deployment invalid: head {m.head!r} label {m.label!r}: {m.problem}")
        specs, rr = [], {}
        for h in heads:
            k = h.backend.get("kind")
            if k not in HEAD_BACKENDS:
                raise ConfigError(f"{h.name}: unknown head backend {k!r}; have {sorted(HEAD_BACKENDS)}")
            specs.append((h.name, k))
            rr[h.name] = (rates or {}).get(h.name, h.default_rate)
        if rates and set(rates) - set(rr):
            raise NotFound(f"rates for heads not in the deployment: {sorted(set(rates) - set(rr))}")
        classes = {int(h.backend["classes"]) for h in heads if "classes" in h.backend}
        if len(classes) > 1:
            raise ConfigError(f"seg heads disagree on the class count {sorted(classes)}")
        if classes and classes != {150}:
            raise ConfigError("seg class count other than 150 needs explicit weights / model_config")
        eng = cls(model, R, B, heads=specs, rates=rr, device=device, weights=weights, seed=seed, **kw)
        try:
            for h in heads:  # soundness: what the card promises is what the backend writes
                outs = eng.out[h.name]
                for s in h.output_specs:
                    t = outs.get(s.label)
                    if t is None or tuple(t.shape) != s.dims or _DT.get(t.dtype) is not s.dtype:
                        raise ConfigError(f"{h.name}: output {s.label!r} {s.dtype.value}{list(s.dims)} is not "
                                          f"what backend {h.backend['kind']} produces")
            eng.cards = (fm, tuple(heads))
        except Exception:
            eng.close()
            raise
        return eng

    # ------------------------------------------------------------------ enqueue primitives
    def _taps(self, slot):
        v = self.channel.group_views(slot)
        return {l: v[l] for l in self.labels}

    def _backbone_into(self, slot):
        taps = self._taps(slot)
        t = [taps[l] for l in self.labels]
        if self.camera:
            self.backbone.forward_camera(self.pixels, t, stream=self.s_prod.handle)
        else:
            self.backbone.forward(self.pixels, t, stream=self.s_prod.handle)

    def _head_on(self, name, slot):
        self.heads[name].run(self._taps(slot), self.out[name], stream=self.s_head[name].handle)

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

    def _check_frames(self, host_frames: torch.Tensor):
        if not isinstance(host_frames, torch.Tensor):
            raise ShapeError(f"frames must be a torch.Tensor, got {type(host_frames).__name__}")
        if host_frames.is_cuda:
            raise ShapeError("submit() takes host frames; copy device frames into engine.pixels instead")
        if (tuple(host_frames.shape) != tuple(self.pixels.shape) or host_frames.dtype != torch.uint8
                or not host_frames.is_contiguous()):
            raise ShapeError(f"frames must be contiguous u8 {tuple(self.pixels.shape)}, got "
                             f"{tuple(host_frames.shape)} {host_frames.dtype}"
                             f"{'' if host_frames.is_contiguous() else ' (non-contiguous)'}")

    # ------------------------------------------------------------------ foundation step
    def _publish(self, host_frames=None, capture_ts=None, record_latency=False):
        """Foundation step: optional H2D of the frame set, backbone graph into
        a claimed ring slot, ready event. Returns (frame id, push outcome, insert event)."""
        if self.fm_state == STOPPED:
            raise EngineError("engine stopped")
        if host_frames is not None:
            self._check_frames(host_frames)
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
        self.fm_iterations += 1
        if not outcome.accepted:
            self.dropped += 1
        return fid, outcome, ev_in

    def _launch_head(self, w: HeadWorker, lease):
        """Enqueue one head run on its stream, reading the leased slot in place, plus the output
        copies (host mirror / output FIFO). Raises InjectedFault when a FAULT is pending."""
        if w.fault:
            w.fault = False
            raise InjectedFault(f"head {w.name}: injected fault")
        st = w.stream
        if self.graphs:
            self._g_head[(w.name, lease.slot_index)].launch(st)
        else:
            self._head_on(w.name, lease.slot_index)
        if self.host_out is not None:
            for k, t in w.out.items():
                check(lib.vpe_memcpy_async(C.c_void_p(self.host_out[w.name][k].data_ptr()), C.c_void_p(t.data_ptr()),
                                           t.numel() * t.element_size(), C.c_void_p(st.handle)))
        if self.fifo is not None:
            outs = w.out

            def out_writer(views, outs=outs, st=st):
                for k, t in outs.items():
                    check(lib.vpe_memcpy_async(C.c_void_p(views[k].data_ptr()), C.c_void_p(t.data_ptr()),
                                               t.numel() * t.element_size(), C.c_void_p(st.handle)))

            if not self.fifo[w.name].push(lease.frame_id, lease.capture_ts, out_writer, stream=st.handle).accepted:
                self.output_drops[w.name] = self.output_drops.get(w.name, 0) + 1

    def _head_failed(self, w: HeadWorker, lease, exc: Exception) -> None:
        """Fault isolation: a panicking head is marked Failed and its
        lease released; any other backend error is skipped and counted."""
        try:
            self.channel.release(lease, stream=w.stream.handle)
        except Exception:  # the lease must not outlive the failure; log and continue
            log.exception("release after head failure")
        if isinstance(exc, InjectedFault):
            w.state = FAILED
            log.warning("head %s failed: %s", w.name, exc)
        else:
            w.errors += 1
            log.warning("head %s backend error (skipped, %d so far): %s", w.name, w.errors, exc)

    # ------------------------------------------------------------------ throughput mode
    def submit(self, host_frames: torch.Tensor | None = None, capture_ts: int | None = None,
               record_latency: bool = False) -> dict:
        """Foundation step + every admitted head, all asynchronous. ``host_frames`` (pinned u8,
        the shape of ``self.pixels``) is copied H2D on the producer stream first; otherwise
        ``self.pixels`` is used. Returns {head: frame id} for the heads that ran."""
        if self._threads_on:
            raise EngineError("submit() while the decentralized workers run; use stop() first")
        fid, _, ev_in = self._publish(host_frames, capture_ts, record_latency)
        ran = {}
        now = time.monotonic_ns()
        for n, w in self.workers.items():
            if w.state != RUNNING or not gate_admit(w.gate, now):
                continue
            st = w.stream
            lease = self.channel.acquire_latest(w.cid, stream=st.handle)
            if lease is None:
                continue
            w.iterations += 1
            try:
                self._launch_head(w, lease)
            except Exception as exc:
                self._head_failed(w, lease, exc)
                continue
            ev = self._event() if record_latency else None
            if ev is not None:
                ev.record(st)
            self.channel.commit(lease, stream=st.handle)
            w.outputs += 1
            w.last_frame = lease.frame_id
            w.history.append(lease.frame_id)
            ran[n] = lease.frame_id
            if ev_in is not None and ev is not None:
                self._lat_records.append((n, ev_in, ev))
        return ran

    def synchronize(self):
        self.s_prod.sync()
        for s in self.s_head.values():
            s.sync()

    def run(self, frames: torch.Tensor) -> dict:
        """Synchronous convenience: one frame set (u8, host or device) -> outputs."""
        if frames.is_cuda:
            if tuple(frames.shape) != tuple(self.pixels.shape) or frames.dtype != torch.uint8:
                raise ShapeError(f"frames must be u8 {tuple(self.pixels.shape)}, got {tuple(frames.shape)}")
            self.pixels.copy_(frames)
            torch.cuda.synchronize()
            self.submit()
        else:
            frames = frames.contiguous()
            self.submit(frames.pin_memory() if not frames.is_pinned() else frames)
        self.synchronize()
        return {n: {k: t.clone() for k, t in o.items()} for n, o in self.out.items()}

    # ------------------------------------------------------------------ decentralized mode
    def start(self, source_hz: float = 30.0, frames: torch.Tensor | None = None) -> None:
        """Run the foundation and every head as independent host workers:
        the foundation thread publishes one frame set per source tick (``source_hz``; frames
        from ``frames`` [n, *pixels.shape] cycled, host or device, else the resident
        ``self.pixels``); each head thread loops gate -> acquire_latest -> run -> commit."""
        if self._threads_on:
            raise EngineError("already started")
        if self.fm_state == STOPPED:
            raise EngineError("engine stopped")
        if not source_hz > 0:
            raise ConfigError(f"source rate must be positive, got {source_hz}")
        if frames is not None:
            if tuple(frames.shape[1:]) != tuple(self.pixels.shape) or frames.dtype != torch.uint8:
                raise ShapeError(f"frames must be u8 [n, {', '.join(map(str, self.pixels.shape))}]")
            if not frames.is_cuda and not frames.is_pinned():
                frames = frames.contiguous().pin_memory()
        self._stop.clear()
        self._threads_on = True
        self._fm_thread = threading.Thread(target=self._foundation_loop, args=(source_hz, frames),
                                           name="vpe-foundation", daemon=True)
        for w in self.workers.values():
            w.thread = threading.Thread(target=self._head_loop, args=(w,), name=f"vpe-head-{w.name}", daemon=True)
            w.thread.start()
        self._fm_thread.start()

    def _foundation_loop(self, source_hz: float, frames):
        period = int(1e9 / source_hz)
        t_next = time.monotonic_ns()
        i = 0
        while not self._stop.is_set():
            now = time.monotonic_ns()
            if now < t_next:
                self._stop.wait((t_next - now) / 1e9)
                continue
            behind = (now - t_next) // period
            if behind:  # the source produced frames the foundation could not take: skip to the newest
                self.source_skips += behind
                t_next += behind * period
            t_next += period
            try:
                host = None
                if frames is not None:
                    f = frames[i % frames.shape[0]]
                    if f.is_cuda:
                        check(lib.vpe_memcpy_async(C.c_void_p(self.pixels.data_ptr()), C.c_void_p(f.data_ptr()),
                                                   self.pixels.numel(), C.c_void_p(self.s_prod.handle)))
                    else:
                        host = f
                i += 1
                self._publish(host, capture_ts=now)
                self.s_prod.sync()  # the foundation worker is blocking, like the reference's loop
            except Exception:
                self.fm_errors += 1  # skip-and-count
                log.exception("foundation step failed")
            with self._new_frame:
                self._new_frame.notify_all()

    def _head_loop(self, w: HeadWorker):
        ch = self.channel
        while not self._stop.is_set() and w.state in (RUNNING, PAUSED):
            if w.state == PAUSED:
                w.resume.wait(0.05)
                continue
            now = time.monotonic_ns()
            ratio = w.gate.every_n
            if not ratio and not gate_admit(w.gate, now):
                # sleep to the next deadline (wakes early on stop / control commands)
                self._stop.wait(min(max(w.gate.next_deadline - now, 0) / 1e9, 0.005))
                continue
            lease = None
            while lease is None and not self._stop.is_set() and w.state == RUNNING:
                lease = ch.acquire_latest(w.cid, stream=w.stream.handle)
                if lease is None:
                    with self._new_frame:
                        self._new_frame.wait(0.05)
            if lease is None:
                continue
            if ratio and (lease.frame_id - 1) % ratio:
                ch.commit(lease, stream=w.stream.handle)  # frame-ratio gate: take 1 frame in n
                continue
            w.iterations += 1
            try:
                if w.stall_s:
                    stall, w.stall_s = w.stall_s, 0.0
                    self._stop.wait(stall)  # holds the lease (the slot stays pinned), like SIGSTOP
                self._launch_head(w, lease)
                w.done_evt.record(w.stream)
                w.done_evt.sync()  # the head waits for its own kernels; the lease covers them
            except Exception as exc:
                self._head_failed(w, lease, exc)
                continue
            ch.commit(lease, stream=w.stream.handle)
            w.outputs += 1
            w.last_frame = lease.frame_id
            w.history.append(lease.frame_id)

    def stop(self, timeout: float = 5.0) -> None:
        """Ordered shutdown of the workers: the source/foundation first, then the
        heads; outstanding device work is drained. The engine stays usable for submit()."""
        if not self._threads_on:
            return
        self._stop.set()
        with self._new_frame:
            self._new_frame.notify_all()
        for w in self.workers.values():
            w.resume.set()
        deadline = time.monotonic() + timeout
        self._fm_thread.join(max(0.0, deadline - time.monotonic()))
        for w in self.workers.values():
            w.thread.join(max(0.0, deadline - time.monotonic()))
        alive = [t.name for t in [self._fm_thread] + [w.thread for w in self.workers.values()] if t.is_alive()]
        self._threads_on = False
        self.synchronize()
        if alive:
            raise EngineError(f"workers did not stop within {timeout}s: {alive}")

    # ------------------------------------------------------------------ control
    def set_rate(self, head: str, hz=None, every_n: int | None = None):
        w = self.workers.get(head)
        if w is None or w.state == FAILED:
            raise NotFound(f"unknown or failed head {head!r}")
        set_rate(self.gates, head, hz, time.monotonic_ns(), every_n=every_n)

    def pause(self, head: str):
        w = self.workers.get(head)
        if w is None or w.state not in (RUNNING, PAUSED):
            raise NotFound(f"unknown or failed head {head!r}")
        w.resume.clear()
        w.state = PAUSED

    def resume(self, head: str):
        w = self.workers.get(head)
        if w is None or w.state not in (RUNNING, PAUSED):
            raise NotFound(f"unknown or failed head {head!r}")
        w.state = RUNNING
        w.resume.set()

    def inject_fault(self, head: str):
        w = self.workers.get(head)
        if w is None or w.state == FAILED:
            raise NotFound(f"unknown or failed head {head!r}")
        w.fault = True

    def status(self) -> dict:
        """EngineStatus snapshot: per-worker state and counters, channel
        counters (pushed = consumed-by-cursor + dropped + resident conservation is per head),
        copy counter, uptime, memory footprint."""
        c = self.channel.counters()
        return {
            "uptime_s": time.monotonic() - self._t0,
            "workers": {"foundation": {"state": self.fm_state, "iterations": self.fm_iterations,
                                       "errors": self.fm_errors, "source_skips": self.source_skips},
                        **{n: w.status() for n, w in self.workers.items()}},
            "channels": {"features": {"pushed": c.pushed, "producer_drops": c.producer_drops,
                                      "evictions": c.evictions, "consumed": c.consumed, "resident": c.resident},
                         **{f"out-{n}": vars(ch.counters()) for n, ch in (self.fifo or {}).items()}},
            "copy_counter": copy_counter(),
            "output_drops": dict(self.output_drops),
            "memory": self.memory_footprint(),
        }

    def memory_footprint(self) -> dict:
        """Device bytes in use (cudaMemGetInfo), torch's allocator view and the regions this
        process created (arena.allocation_audit): constant after init."""
        free, total = torch.cuda.mem_get_info(self.device)
        return {"device_used": int(total - free), "torch_reserved": int(torch.cuda.memory_reserved(self.device)),
                "torch_allocated": int(torch.cuda.memory_allocated(self.device)),
                "regions": len(allocation_audit())}

    def dispatch(self, cmd: str) -> str:
        """One control command in SPEC's textual encoding: ``SETRATE <head> <hz>``
        (hz may be "1:n" or "unlimited"), ``PAUSE <head>``, ``RESUME <head>``, ``STOP``,
        ``STATS``, ``FAULT <head>``. Replies ``OK [body]`` or ``ERR <code> <detail>``."""
        try:
            parts = cmd.strip().split()
            if not parts:
                raise ProtocolError("empty command")
            tag, args = parts[0].upper(), parts[1:]
            arity = {"SETRATE": 2, "PAUSE": 1, "RESUME": 1, "STOP": 0, "STATS": 0, "FAULT": 1}
            if tag not in arity:
                raise ProtocolError(f"unknown command {parts[0]!r}")
            if len(args) != arity[tag]:
                raise ProtocolError(f"{tag} takes {arity[tag]} argument(s), got {len(args)}")
            if tag == "SETRATE":
                try:
                    hz, every = _parse_rate(args[1])
                except ValueError as exc:
                    raise ConfigError(f"bad rate {args[1]!r}") from exc
                self.set_rate(args[0], hz, every_n=every)
                return "OK"
            if tag == "PAUSE":
                self.pause(args[0])
                return "OK"
            if tag == "RESUME":
                self.resume(args[0])
                return "OK"
            if tag == "FAULT":
                self.inject_fault(args[0])
                return "OK"
            if tag == "STATS":
                return "OK " + json.dumps(self.status(), sort_keys=True)
            self.stop()
            self.fm_state = STOPPED
            for w in self.workers.values():
                if w.state != FAILED:
                    w.state = STOPPED
            return "OK"
        except EngineError as exc:
            return f"ERR {type(exc).__name__} {exc}"

    # ------------------------------------------------------------------ measurement helpers
    def latencies_ms(self) -> dict[str, list[float]]:
        out = {n: [] for n in self.heads}
        for n, a, b in self._lat_records:
            b.sync()  # the pool may be recycled mid-run: wait for the head's end event first
            out[n].append(a.elapsed_ms(b))
        self._lat_records = []
        self._ev_next = 0
        return out

    def counters(self):
        return self.channel.counters()

    def close(self):
        if self._closed:
            return
        try:
            self.stop()
        finally:
            self._closed = True
            self.fm_state = STOPPED
            for g in list(self._g_bb.values()) + list(self._g_head.values()):
                g.close()
            self._g_bb, self._g_head = {}, {}
            for w in self.workers.values():
                if w.done_evt is not None:
                    w.done_evt.close()
            for e in self._ev_pool:
                e.close()
            for h in self.heads.values():
                h.close()
            self.backbone.close()
            self.channel.close()
            for ch in (self.fifo or {}).values():
                ch.close()
            self.fifo = None
            for s in [self.s_prod, *self.s_head.values()]:
                s.close()
