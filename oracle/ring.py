"""Pure-Python restatement of the reference channel state machine (TEST INFRASTRUCTURE).

Single-process, no shared memory, no atomics: a sequential oracle for the LATEST/FIFO slot
protocol of ``/root/reference/pkg/src/fanpipe/channels.py`` used to check the C++ device ring
(libvpe ``vpe_ring_*``) outcome-for-outcome on recorded schedules. Each method cites the
reference lines it restates. Pinned against the reference itself (``baseline/_ref/fanpipe``,
built from /root/reference by pip) in tests/test_oracle_ring.py, and against the SPEC
known-answer examples frozen in tests/golden/spec_examples.json.
"""

from __future__ import annotations

from dataclasses import dataclass

STATE_FREE, STATE_WRITING, STATE_READY = 0, 1, 2  # channels.py:54-56
MAX_CONSUMERS = 16                                 # channels.py:58


@dataclass
class OLease:
    slot: int
    frame_id: int
    capture_ts: int
    consumer_id: int
    consumed: bool = False


class OracleChannel:
    def __init__(self, mode: str, capacity: int, labels: tuple[str, ...]):
        if capacity < 2:                           # channels.py:547-548
            raise ValueError("capacity must be >= 2")
        self.mode, self.capacity, self.labels = mode, capacity, tuple(labels)
        self.state = [STATE_FREE] * capacity
        self.fid = [0] * capacity
        self.ts = [0] * capacity
        self.data = [dict() for _ in range(capacity)]
        self.cursors: dict[int, int] = {}
        self.drops = self.evictions = self.pushed = self.consumed = 0
        self.last_id = self.last_ts = 0

    # channels.py:311-331
    def _claim_slot(self):
        for i in range(self.capacity):
            if self.state[i] == STATE_FREE:
                return i, None
        if self.mode == "fifo":
            return None, None
        oldest, oldest_fid = -1, None
        for i in range(self.capacity):
            if self.state[i] == STATE_READY and (oldest_fid is None or self.fid[i] < oldest_fid):
                oldest, oldest_fid = i, self.fid[i]
        if oldest < 0:
            return None, None
        return oldest, oldest_fid

    # channels.py:274-309
    def push(self, frame_id: int, capture_ts: int, payload: dict):
        if frame_id <= self.last_id:
            raise ValueError("frame_id must increase")
        if capture_ts < self.last_ts:
            raise ValueError("capture_ts must be non-decreasing")
        slot, evicted = self._claim_slot()
        if slot is None:
            self.drops += 1
            self.pushed += 1
            return ("overflow_rejected", None, None)
        self.state[slot] = STATE_WRITING
        self.fid[slot], self.ts[slot] = frame_id, capture_ts
        self.data[slot] = {k: v.copy() for k, v in payload.items()}
        self.state[slot] = STATE_READY
        self.pushed += 1
        self.last_id, self.last_ts = frame_id, capture_ts
        if evicted is not None:
            self.evictions += 1
            return ("accepted_evicting", evicted, slot)
        return ("accepted", None, slot)

    # channels.py:335-358
    def register_consumer(self, cid: int) -> bool:
        if not 1 <= cid <= 0xFFFFFFFE:
            raise ValueError("consumer id")
        if cid in self.cursors:
            return False
        if len(self.cursors) >= MAX_CONSUMERS:
            raise RuntimeError("cursor table full")
        warn = self.mode == "latest" and len(self.cursors) + 2 > self.capacity
        self.cursors[cid] = 0
        return warn

    # channels.py:423-452
    def acquire_latest(self, cid: int):
        cursor = self.cursors[cid]
        best, best_fid = -1, cursor
        for i in range(self.capacity):
            if self.state[i] >= STATE_READY and self.fid[i] > best_fid:
                best, best_fid = i, self.fid[i]
        if best < 0:
            return None
        self.state[best] += 1
        return OLease(best, self.fid[best], self.ts[best], cid)

    # channels.py:483-489
    def _release(self, slot: int):
        if self.state[slot] <= STATE_READY:
            raise RuntimeError("released while not leased")
        self.state[slot] -= 1

    # channels.py:454-474
    def consume(self, lease: OLease, labels=None):
        if lease.consumed:
            raise RuntimeError("use after consume")
        chosen = tuple(labels) if labels is not None else self.labels
        for lbl in chosen:
            if lbl not in self.labels:
                raise KeyError(lbl)
        out = {lbl: self.data[lease.slot][lbl].copy() for lbl in chosen}
        self.cursors[lease.consumer_id] = lease.frame_id
        self.consumed += 1
        self._release(lease.slot)
        lease.consumed = True
        return out

    # channels.py:476-481
    def release(self, lease: OLease):
        if lease.consumed:
            return
        self._release(lease.slot)
        lease.consumed = True

    # channels.py:377-421
    def pop(self, cid: int):
        if self.mode != "fifo":
            raise RuntimeError("pop requires FIFO")
        best, best_fid = -1, None
        for i in range(self.capacity):
            if self.state[i] == STATE_READY and (best_fid is None or self.fid[i] < best_fid):
                best, best_fid = i, self.fid[i]
        if best < 0:
            return None
        out = {lbl: self.data[best][lbl].copy() for lbl in self.labels}
        self.cursors[cid] = best_fid
        self.consumed += 1
        self.state[best] = STATE_FREE
        return best_fid, out

    # channels.py:493-504
    def counters(self):
        resident = sum(1 for s in self.state if s >= STATE_READY)
        return dict(pushed=self.pushed, producer_drops=self.drops, evictions=self.evictions,
                    consumed=self.consumed, resident=resident)
