"""Channels — the reference's ``fanpipe.channels`` API (channels.py:68-594) over libvpe's device
ring (``vpe_ring_*``, include/vpe.h).

Same names, arguments, outcomes and exceptions as the reference: ``create_channel``,
``Channel.push / register_consumer / acquire_latest / consume / release / pop / counters /
slot_states / group_views / last_consumed``, ``ChannelHandle``, ``SlotGroup``,
``create_processing_slots`` / ``open_processing_slots``, ``PushKind`` / ``PushOutcome`` / ``Lease`` / ``FrameEnvelope`` /
``ChannelCounters``. The control block keeps the PECH1 byte layout; the state machine runs in
C++ with the reference's CAS protocol.

GPU additions:
  * ``writer(views)`` receives device tensors aliasing the claimed slot; work it enqueues on the
    channel's producer stream is ordered before READY by a CUDA event (``vpe_ring_publish``).
  * ``view(lease, labels)`` + ``commit(lease)`` consume IN PLACE: the consumer stream waits on the
    slot's ready event, heads read the HBM slot directly, ``commit`` records a done event
    (the producer waits on it before overwriting the slot) and advances the cursor like
    ``consume`` does (channels.py:470) — zero copies.
  * ``consume`` keeps the reference's single-copy semantics as a stream-ordered D2D/D2H copy.
"""

from __future__ import annotations

import ctypes as C
import logging
import time
from dataclasses import dataclass
from enum import Enum
from typing import Callable, Mapping, Sequence

import torch

from . import arena as ar
from ._lib import LeaseC, CountersC, TensorSpecC, check, lib
from .errors import (ConfigError, LabelError, NO_NEW_DATA, NotFound, OVERFLOW_REJECTED, ShapeError,
                     UseAfterConsume, WriterError)

log = logging.getLogger("vpe.channels")

STATE_FREE, STATE_WRITING, STATE_READY = 0, 1, 2
MAX_CONSUMERS = 16
_BACKOFF_CAP_S = 100e-6


class ChannelMode(Enum):
    FIFO = 0
    LATEST = 1


@dataclass(frozen=True)
class FrameEnvelope:
    frame_id: int
    capture_ts: int
    labels: tuple[str, ...]


class PushKind(Enum):
    ACCEPTED = "accepted"
    ACCEPTED_EVICTING = "accepted_evicting"
    OVERFLOW_REJECTED = "overflow_rejected"


@dataclass(frozen=True)
class PushOutcome:
    kind: PushKind
    evicted_frame_id: int | None = None
    slot: int | None = None

    @property
    def accepted(self) -> bool:
        return self.kind is not PushKind.OVERFLOW_REJECTED


@dataclass
class Lease:
    channel: "Channel"
    slot_index: int
    frame_id: int
    capture_ts: int
    consumer_id: int
    consumed: bool = False
    _c: LeaseC | None = None


@dataclass(frozen=True)
class ChannelCounters:
    pushed: int
    producer_drops: int
    evictions: int
    consumed: int
    resident: int


@dataclass(frozen=True)
class ChannelHandle:
    name: str
    namespace: str
    mode: ChannelMode
    capacity: int
    specs: tuple[ar.TensorSpec, ...]
    header: ar.ShareHandle
    data: ar.ShareHandle

    def to_dict(self) -> dict:
        return {"name": self.name, "namespace": self.namespace, "mode": self.mode.name.lower(),
                "capacity": self.capacity, "specs": [s.to_dict() for s in self.specs],
                "header": self.header.to_dict(), "data": self.data.to_dict()}

    @classmethod
    def from_dict(cls, d: dict) -> "ChannelHandle":
        return cls(name=d["name"], namespace=d["namespace"], mode=ChannelMode[d["mode"].upper()],
                   capacity=d["capacity"], specs=tuple(ar.TensorSpec.from_dict(s) for s in d["specs"]),
                   header=ar.ShareHandle.from_dict(d["header"]), data=ar.ShareHandle.from_dict(d["data"]))


class SlotGroup:
    """Caller-owned processing slots: one arena slot per channel label (channels.py:155-176)."""

    def __init__(self, accessor, refs: Mapping[str, ar.SlotRef]):
        self.arena = accessor
        self.refs = dict(refs)
        self._views = {lbl: accessor.data_view(ref.offset, ref.spec) for lbl, ref in self.refs.items()}

    @property
    def labels(self) -> tuple[str, ...]:
        return tuple(self.refs)

    def ref(self, label: str) -> ar.SlotRef:
        return self.refs[label]

    def view(self, label: str) -> torch.Tensor:
        return self._views[label]

    def spec(self, label: str) -> ar.TensorSpec:
        return self.refs[label].spec


class _PinnedArena:
    """A process-private arena in pinned host memory (D2H destinations of output queues)."""

    def __init__(self, handle: ar.ShareHandle):
        self.handle = handle
        self.device = -1
        self.buf = torch.zeros(handle.total_bytes, dtype=torch.uint8, pin_memory=torch.cuda.is_available())

    def data_view(self, offset: int, spec: ar.TensorSpec) -> torch.Tensor:
        return ar.view_of(self.buf, offset, spec)

    def close(self) -> None:
        self.buf = None


def _refs(handle: ar.ShareHandle, layout: ar.ArenaLayout) -> dict[str, ar.SlotRef]:
    return {spec.label: ar.SlotRef(handle, sid, spec, layout.offset_of(sid)) for sid, spec in layout.slots}


def create_processing_slots(namespace: str, region_name: str, specs: Sequence[ar.TensorSpec],
                            device: int | str = 0) -> SlotGroup:
    """Preallocate a consumer-private destination group for consume()/pop() (channels.py:179-186):
    an arena in HBM (device >= 0) or POSIX shared memory (-2 / "cpu"), both shareable through
    ``open_processing_slots``, or private pinned host memory (-1 / "host")."""
    dev = {"host": -1, "cpu": -2}.get(device, device) if isinstance(device, str) else int(device)
    layout = ar.ArenaLayout.from_specs(list(specs))
    if dev == -1:
        ar.validate_name("namespace", namespace)
        ar.validate_name("region_name", region_name)
        handle = ar.ShareHandle(namespace, region_name, layout.total_bytes, -1)
        ar.log_allocation(handle.os_name, layout.total_bytes)
        return SlotGroup(_PinnedArena(handle), _refs(handle, layout))
    accessor, handle = ar.create_arena(layout, namespace, region_name, device=dev)
    return SlotGroup(accessor, _refs(handle, layout))


def open_processing_slots(handle: ar.ShareHandle, specs: Sequence[ar.TensorSpec]) -> SlotGroup:
    """Map another process's processing slots (channels.py:189-196)."""
    accessor = ar.import_arena(handle)
    return SlotGroup(accessor, _refs(handle, ar.ArenaLayout.from_specs(list(specs))))


class _Backoff:
    def __init__(self):
        self._step = 0

    def pause(self):
        if self._step < 3:
            time.sleep(0)
        else:
            time.sleep(min(2 ** (self._step - 3) * 1e-6, _BACKOFF_CAP_S))
        self._step += 1


def _spec_c(spec: ar.TensorSpec) -> TensorSpecC:
    c = TensorSpecC()
    c.label = spec.label.encode()
    c.dtype = spec.dtype.code
    c.rank = len(spec.dims)
    for i, d in enumerate(spec.dims):
        c.dims[i] = d
    return c


def _sp(stream) -> C.c_void_p:
    return C.c_void_p(stream)


class Channel:
    """One endpoint of a device channel. Endpoints are not thread-safe (channels.py:219-223)."""

    def __init__(self, handle: ChannelHandle, ring: C.c_void_p, stream: int | None = None):
        self.handle = handle
        self.name = handle.name
        self.mode = handle.mode
        self.capacity = handle.capacity
        self.specs = handle.specs
        self.labels = tuple(s.label for s in handle.specs)
        self._label_idx = {s.label: i for i, s in enumerate(handle.specs)}
        self._ring = ring
        self.device = handle.data.device
        base, size = C.c_void_p(), C.c_size_t()
        check(lib.vpe_ring_data(ring, C.byref(base), C.byref(size)))
        self._raw = ar.alias_bytes(base.value, size.value, self.device)
        hb, hs = C.c_void_p(), C.c_size_t()
        check(lib.vpe_ring_header(ring, C.byref(hb), C.byref(hs)))
        self._hdr = (hb.value, hs.value)
        self._layout = ar.ArenaLayout.from_specs(list(handle.specs) * handle.capacity)
        self._group_views: list[dict[str, torch.Tensor]] = []
        self._group_ptrs: list[dict[str, int]] = []
        n = len(handle.specs)
        for i in range(handle.capacity):
            views, ptrs = {}, {}
            for j, spec in enumerate(handle.specs):
                off = self._layout.offset_of(i * n + j)
                views[spec.label] = ar.view_of(self._raw, off, spec)
                p = C.c_void_p()
                check(lib.vpe_ring_slot_ptr(ring, i, j, C.byref(p)))
                ptrs[spec.label] = p.value
            self._group_views.append(views)
            self._group_ptrs.append(ptrs)
        self._stream = stream
        self._cursor_registered: set[int] = set()

    # -- helpers ---------------------------------------------------------------------------
    def _s(self, stream):
        if stream is not None:
            return stream
        if self._stream is not None:
            return self._stream
        if self.device >= 0:
            return torch.cuda.current_stream(self.device).cuda_stream
        return None

    def header_bytes(self) -> bytes:
        """Snapshot of the PECH1 control block (channels.py:14-26 layout)."""
        return C.string_at(self._hdr[0], self._hdr[1])

    # -- producer side ---------------------------------------------------------------------
    def push(self, frame_id: int, capture_ts: int, writer: Callable[[Mapping[str, torch.Tensor]], None],
             stream: int | None = None) -> PushOutcome:
        """Publish one frame; ``writer`` fills the claimed slot group in place (channels.py:274-309).
        Device work the writer enqueues on ``stream`` is complete before any consumer reads it."""
        s = self._s(stream)
        slot, evf, ev = C.c_int32(), C.c_uint64(), C.c_int32()
        rc = lib.vpe_ring_claim(self._ring, frame_id, capture_ts, _sp(s), C.byref(slot), C.byref(evf), C.byref(ev))
        if rc == 20:  # ValueError: frame ordering (channels.py:284-287)
            raise ValueError(f"frame_id must increase / capture_ts non-decreasing (frame {frame_id})")
        check(rc, "push")
        if rc == OVERFLOW_REJECTED:
            return PushOutcome(PushKind.OVERFLOW_REJECTED)
        try:
            writer(self._group_views[slot.value])
        except Exception as exc:
            lib.vpe_ring_abort(self._ring, slot.value)
            raise WriterError(f"writer failed for frame {frame_id}: {exc}") from exc
        check(lib.vpe_ring_publish(self._ring, slot.value, _sp(s)), "publish")
        if ev.value:
            return PushOutcome(PushKind.ACCEPTED_EVICTING, evicted_frame_id=int(evf.value), slot=slot.value)
        return PushOutcome(PushKind.ACCEPTED, slot=slot.value)

    # -- consumer side ---------------------------------------------------------------------
    def register_consumer(self, consumer_id: int) -> None:
        if not 1 <= consumer_id <= 0xFFFFFFFF - 1:
            raise ConfigError(f"consumer_id must be a positive u32, got {consumer_id}")
        warn = C.c_int32()
        check(lib.vpe_ring_register_consumer(self._ring, consumer_id, C.byref(warn)), "register_consumer")
        self._cursor_registered.add(consumer_id)
        if warn.value:
            log.warning("channel %s: capacity %d below consumer count + 1; producer may see OverflowRejected "
                        "under load", self.name, self.capacity)

    def _require(self, consumer_id: int) -> None:
        if consumer_id not in self._cursor_registered:
            raise NotFound(f"consumer {consumer_id} not registered on {self.name}")

    def last_consumed(self, consumer_id: int) -> int:
        self._require(consumer_id)
        v = C.c_uint64()
        check(lib.vpe_ring_last_consumed(self._ring, consumer_id, C.byref(v)))
        return int(v.value)

    def acquire_latest(self, consumer_id: int, stream: int | None = None) -> Lease | None:
        """Lease the newest READY frame newer than the consumer cursor (channels.py:423-452);
        the consumer stream is made to wait on the slot's ready event. None = nothing newer."""
        self._require(consumer_id)
        lc = LeaseC()
        rc = lib.vpe_ring_acquire_latest(self._ring, consumer_id, _sp(self._s(stream)), C.byref(lc))
        if rc == NO_NEW_DATA:
            return None
        check(rc, "acquire_latest")
        return Lease(self, lc.slot, int(lc.frame_id), int(lc.capture_ts), consumer_id, False, lc)

    def view(self, lease: Lease, labels: Sequence[str] | None = None) -> dict[str, torch.Tensor]:
        """Zero-copy tensors over the leased slot (read in place; copy counter untouched)."""
        if lease.consumed:
            raise UseAfterConsume(f"lease on frame {lease.frame_id} already consumed")
        chosen = tuple(labels) if labels is not None else self.labels
        self._check_labels(chosen)
        return {lbl: self._group_views[lease.slot_index][lbl] for lbl in chosen}

    def slot_ptrs(self, slot: int) -> dict[str, int]:
        return self._group_ptrs[slot]

    def commit(self, lease: Lease, stream: int | None = None) -> FrameEnvelope:
        """In-place consumption finished on ``stream``: record done, advance cursor, release."""
        if lease.consumed:
            raise UseAfterConsume(f"lease on frame {lease.frame_id} already consumed")
        check(lib.vpe_ring_commit(self._ring, C.byref(lease._c), _sp(self._s(stream))), "commit")
        lease.consumed = True
        return FrameEnvelope(lease.frame_id, lease.capture_ts, self.labels)

    def _check_labels(self, chosen):
        unknown = [lbl for lbl in chosen if lbl not in self.labels]
        if unknown:
            raise LabelError(f"labels {unknown} not in channel label set {self.labels}")

    @staticmethod
    def _dst_tensor(dst, label):
        return dst.view(label) if isinstance(dst, SlotGroup) else dst[label]

    def _check_dst(self, dst: SlotGroup | Mapping[str, torch.Tensor], labels) -> list[int]:
        ptrs = []
        for lbl in labels:
            want = next(s for s in self.specs if s.label == lbl)
            t = dst.view(lbl) if isinstance(dst, SlotGroup) else dst.get(lbl)
            if t is None:
                raise ShapeError(f"dst group missing slot for label {lbl!r}")
            if (tuple(t.shape) != want.dims or t.dtype != want.dtype.torch_dtype or not t.is_contiguous()):
                raise ShapeError(f"dst spec mismatch for {lbl!r}: {tuple(t.shape)} {t.dtype} != {want}")
            ptrs.append(t.data_ptr())
        return ptrs

    def consume(self, lease: Lease, dst: SlotGroup | Mapping[str, torch.Tensor],
                labels: Sequence[str] | None = None, stream: int | None = None) -> FrameEnvelope:
        """Copy the leased frame's selected labels into ``dst`` (one copy per label), then
        release and advance the cursor (channels.py:454-474)."""
        if lease.consumed:
            raise UseAfterConsume(f"lease on frame {lease.frame_id} already consumed")
        chosen = tuple(labels) if labels is not None else self.labels
        self._check_labels(chosen)
        ptrs = self._check_dst(dst, chosen)
        idx = (C.c_int32 * len(chosen))(*[self._label_idx[lbl] for lbl in chosen])
        pp = (C.c_void_p * len(chosen))(*ptrs)
        s = self._s(stream)
        check(lib.vpe_ring_consume(self._ring, C.byref(lease._c), idx, len(chosen), pp, _sp(s)), "consume")
        if self.device != -2 and any(not self._dst_tensor(dst, l).is_cuda for l in chosen):
            # host destinations: the reference's consume returns with the bytes in dst
            check(lib.vpe_stream_sync(_sp(s)), "consume")
        lease.consumed = True
        return FrameEnvelope(lease.frame_id, lease.capture_ts, chosen)

    def release(self, lease: Lease, stream: int | None = None) -> None:
        """Drop a lease without consuming; the cursor does not move (channels.py:476-481)."""
        if lease.consumed:
            return
        rc = lib.vpe_ring_release(self._ring, C.byref(lease._c), _sp(self._s(stream)))
        check(rc, "release")
        lease.consumed = True

    def pop(self, consumer_id: int, dst: SlotGroup | Mapping[str, torch.Tensor], block: bool = False,
            timeout: float | None = None, stream: int | None = None) -> FrameEnvelope | None:
        """FIFO: copy the oldest READY frame into ``dst`` and free its slot (channels.py:377-407).
        Host destinations (CPU tensors) are filled synchronously; device ones stream-ordered."""
        if self.mode is not ChannelMode.FIFO:
            raise ConfigError(f"pop() requires a FIFO channel, {self.name} is {self.mode.name}")
        self._require(consumer_id)
        ptrs = self._check_dst(dst, self.labels)
        pp = (C.c_void_p * len(ptrs))(*ptrs)
        on_dev = [(dst.view(l) if isinstance(dst, SlotGroup) else dst[l]).is_cuda for l in self.labels]
        if any(on_dev) and not all(on_dev):
            raise ShapeError("pop destinations must be all host or all device tensors")
        host_dst = not any(on_dev)
        s = self._s(stream)
        backoff = _Backoff()
        deadline = None if timeout is None else time.monotonic() + timeout
        env = LeaseC()
        while True:
            rc = lib.vpe_ring_pop(self._ring, consumer_id, pp, int(host_dst), _sp(s), C.byref(env))
            if rc != NO_NEW_DATA:
                check(rc, "pop")
                return FrameEnvelope(int(env.frame_id), int(env.capture_ts), self.labels)
            if not block:
                return None
            if deadline is not None and time.monotonic() >= deadline:
                return None
            backoff.pause()

    # -- introspection -----------------------------------------------------------------------
    def counters(self) -> ChannelCounters:
        c = CountersC()
        check(lib.vpe_ring_counters(self._ring, C.byref(c)))
        return ChannelCounters(int(c.pushed), int(c.producer_drops), int(c.evictions), int(c.consumed),
                               int(c.resident))

    def slot_states(self) -> list[tuple[int, int]]:
        out = []
        for i in range(self.capacity):
            st, f = C.c_uint32(), C.c_uint64()
            check(lib.vpe_ring_slot_state(self._ring, i, C.byref(st), C.byref(f)))
            out.append((int(st.value), int(f.value)))
        return out

    def group_views(self, slot_index: int) -> dict[str, torch.Tensor]:
        return self._group_views[slot_index]

    def close(self) -> None:
        if self._ring:
            self._group_views = []
            self._raw = None
            lib.vpe_ring_destroy(self._ring)
            self._ring = None
            if not getattr(self, "_attached", False):
                ar.forget_allocation(self.handle.data.os_name)
                ar.forget_allocation(self.handle.header.os_name)

    def unlink(self) -> None:
        self.close()


def header_region_bytes(capacity: int) -> int:
    """channels.py:532-534."""
    need = 16 + capacity * 24 + MAX_CONSUMERS * 16 + 32
    return max(4096, (need + 4095) // 4096 * 4096)


def _shared_name(handle: ChannelHandle) -> bytes:
    return f"{handle.namespace}.{handle.name}".encode()


def create_channel(name: str, mode: ChannelMode, capacity: int, slot_group: Sequence[ar.TensorSpec],
                   namespace: str, expected_consumers: int | None = None, device: int = 0,
                   stream: int | None = None, shared: bool = False) -> tuple[Channel, ChannelHandle]:
    """Create the control block and the slot arena (HBM for device >= 0); all slots FREE.
    Validation and warnings follow channels.py:537-576. ``shared=True`` puts the control block in
    POSIX shared memory and exports the HBM arena and its events through CUDA IPC, so other
    processes can ``open_channel(handle)`` (the reference's cross-process channel)."""
    if capacity < 2:
        raise ConfigError(f"channel capacity must be >= 2, got {capacity}")
    specs = tuple(slot_group)
    if not specs:
        raise ConfigError("channel needs a non-empty slot group spec list")
    seen = set()
    for s in specs:
        if s.label in seen:
            raise ConfigError(f"duplicate label {s.label!r} in slot group")
        seen.add(s.label)
    if mode is ChannelMode.LATEST and expected_consumers is not None and capacity < expected_consumers + 1:
        log.warning("channel %s: LATEST capacity %d < expected consumers %d + 1", name, capacity,
                    expected_consumers)
    ar.validate_name("namespace", namespace)
    ar.validate_name("region_name", name)
    layout = ar.ArenaLayout.from_specs(list(specs) * capacity)
    arr = (TensorSpecC * len(specs))(*[_spec_c(s) for s in specs])
    ring = C.c_void_p()
    data_h = ar.ShareHandle(namespace, f"{name}-d", layout.total_bytes, device)
    hdr_h = ar.ShareHandle(namespace, f"{name}-c", header_region_bytes(capacity), -2)
    ar.log_allocation(data_h.os_name, layout.total_bytes)
    try:
        ar.log_allocation(hdr_h.os_name, hdr_h.total_bytes)
    except Exception:
        ar.forget_allocation(data_h.os_name)
        raise
    if device >= 0:
        torch.cuda.set_device(device)
    handle = ChannelHandle(name=name, namespace=namespace, mode=mode, capacity=capacity, specs=specs,
                           header=hdr_h, data=data_h)
    if shared:
        rc = lib.vpe_ring_create_shared(arr, len(specs), capacity, mode.value, device, _shared_name(handle),
                                        C.byref(ring))
    else:
        rc = lib.vpe_ring_create(arr, len(specs), capacity, mode.value, device, C.byref(ring))
    if rc:
        ar.forget_allocation(data_h.os_name)
        ar.forget_allocation(hdr_h.os_name)
    check(rc, "create_channel")
    return Channel(handle, ring, stream=stream), handle


def open_channel(handle: ChannelHandle, stream: int | None = None) -> Channel:
    """Attach to a channel created with ``shared=True`` in another process (channels.py:579-594):
    maps the shared control block, opens the HBM arena and the ready/done events through CUDA
    IPC, and validates the header (magic, mode, capacity) against the handle."""
    ring = C.c_void_p()
    if handle.data.device >= 0:
        torch.cuda.set_device(handle.data.device)
    check(lib.vpe_ring_attach(_shared_name(handle), C.byref(ring)), "open_channel")
    ch = Channel(handle, ring, stream=stream)
    hdr = ch.header_bytes()
    cap = int.from_bytes(hdr[8:12], "little")
    if hdr[:6] != b"PECH1\x00" or hdr[6] != handle.mode.value or cap != handle.capacity:
        ch._attached = True
        ch.close()
        raise ConfigError(f"channel {handle.name}: header does not match the handle")
    ch._attached = True
    return ch
