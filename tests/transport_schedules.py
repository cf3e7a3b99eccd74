"""Transport scenarios run identically against three implementations of the channel protocol:

* ``ref``     the unmodified reference ``fanpipe`` (baseline/_ref, built from /root/reference)
* ``oracle``  the pure-Python restatement (oracle/ring.py)
* ``vpe``     the product device ring (libvpe ``vpe_ring_*`` through channels.py), on the GPU or,
              in CPU-only tests, with its data arena in pageable host memory (device=-2)

Each scenario is a list of ops; ``run(adapter, scenario)`` returns the list of observable
outcomes (push kinds, evicted ids, leased frame ids, consumed payload checksums, counters),
which must match element for element. The SPEC known-answer examples and
seeded random schedules are both expressed this way; outcomes produced by the reference are
frozen in tests/golden/spec_examples.json by tests/golden/make_golden.py.
"""

from __future__ import annotations

import random

import numpy as np

LABELS = ("final", "layer3", "layer6", "layer9")
DIMS = (2, 3)


def payload(fid: int, label_idx: int) -> np.ndarray:
    return (np.arange(6, dtype=np.float32).reshape(DIMS) + fid * 100 + label_idx * 10)


def checksum(arr) -> float:
    return float(np.asarray(arr, dtype=np.float64).sum())


# ---------------------------------------------------------------------- scenarios
def spec_scenarios() -> dict[str, dict]:
    return {
        # SPEC.md:169  FIFO cap 2: push f1, f2, f3 with no consumer -> f3 OverflowRejected
        "fifo_overflow": dict(mode="fifo", cap=2, ops=[("push", 1), ("push", 2), ("push", 3), ("counters",)]),
        # SPEC.md:170  LATEST cap 2: f3 AcceptedEvicting(f1); latest reader sees f3
        "latest_evict": dict(mode="latest", cap=2, ops=[("register", 1), ("push", 1), ("push", 2), ("push", 3),
                                                         ("acquire", 1), ("consume", 1, None), ("counters",)]),
        # SPEC.md:171 / Appendix A.5: both slots leased -> OverflowRejected; release one -> evicts
        "lease_saturation": dict(mode="latest", cap=2, ops=[
            ("register", 1), ("register", 2), ("push", 1), ("acquire", 1), ("push", 2), ("acquire", 2),
            ("push", 3), ("counters",), ("release", 1), ("push", 4), ("counters",)]),
        # SPEC.md:178-180  FIFO order, empty pop
        "fifo_order": dict(mode="fifo", cap=4, ops=[("register", 1), ("push", 1), ("push", 2), ("pop", 1),
                                                     ("pop", 1), ("pop", 1), ("counters",)]),
        # SPEC.md:187-189  freshness, duplicate suppression, two leases on one frame
        "freshness": dict(mode="latest", cap=4, ops=[
            ("register", 1), ("register", 2), ("push", 4), ("push", 5), ("acquire", 1), ("consume", 1, None),
            ("acquire", 1), ("acquire", 2), ("state", ), ("consume", 2, ("final",)), ("push", 6),
            ("acquire", 1), ("consume", 1, ("layer3", "final")), ("counters",)]),
        # SPEC.md:196-198  selective consumption (copy counts checked by the caller)
        "selective": dict(mode="latest", cap=5, ops=[
            ("register", 1), ("register", 2), ("register", 3), ("push", 1), ("acquire", 1), ("acquire", 2),
            ("acquire", 3), ("consume", 1, LABELS), ("consume", 2, ("final",)), ("consume", 3, ("final",)),
            ("counters",)]),
        # channels.py:342-344  consumer restart keeps its cursor
        "restart_cursor": dict(mode="latest", cap=3, ops=[
            ("register", 7), ("push", 1), ("push", 2), ("acquire", 7), ("consume", 7, None), ("register", 7),
            ("acquire", 7), ("push", 3), ("acquire", 7), ("consume", 7, None), ("counters",)]),
    }


def random_scenario(seed: int, mode: str = "latest", cap: int = 5, consumers: int = 3, n: int = 600) -> dict:
    rng = random.Random(seed)
    ops = [("register", c) for c in range(1, consumers + 1)]
    fid = 0
    for _ in range(n):
        r = rng.random()
        if r < 0.35:
            fid += rng.choice([1, 1, 1, 2])
            ops.append(("push", fid))
        elif mode == "fifo" and r < 0.6:
            ops.append(("pop", rng.randint(1, consumers)))
        elif r < 0.7:
            ops.append(("acquire", rng.randint(1, consumers)))
        elif r < 0.9:
            sub = tuple(l for l in LABELS if rng.random() < 0.5) or ("final",)
            ops.append(("consume", rng.randint(1, consumers), sub))
        elif r < 0.97:
            ops.append(("release", rng.randint(1, consumers)))
        else:
            ops.append(("counters",))
    ops.append(("counters",))
    return dict(mode=mode, cap=cap, ops=ops)


# ---------------------------------------------------------------------- runner
def run(adapter, scenario: dict) -> list:
    adapter.open(scenario["mode"], scenario["cap"])
    leases: dict[int, object] = {}
    out = []
    try:
        for op in scenario["ops"]:
            kind = op[0]
            if kind == "push":
                r = adapter.push(op[1])
                out.append(["push", op[1], r[0], r[1]])
            elif kind == "register":
                adapter.register(op[1])
                out.append(["register", op[1]])
            elif kind == "acquire":
                c = op[1]
                if c in leases:
                    out.append(["acquire", c, "held"])
                    continue
                le = adapter.acquire(c)
                if le is None:
                    out.append(["acquire", c, None])
                else:
                    leases[c] = le
                    out.append(["acquire", c, adapter.lease_fid(le)])
            elif kind == "consume":
                c = op[1]
                if c not in leases:
                    out.append(["consume", c, "nolease"])
                    continue
                labels = op[2]
                got = adapter.consume(leases.pop(c), labels)
                out.append(["consume", c, {k: checksum(v) for k, v in sorted(got.items())}])
            elif kind == "release":
                c = op[1]
                if c not in leases:
                    out.append(["release", c, "nolease"])
                    continue
                adapter.release(leases.pop(c))
                out.append(["release", c])
            elif kind == "pop":
                r = adapter.pop(op[1])
                out.append(["pop", op[1], None if r is None else [r[0], {k: checksum(v) for k, v in sorted(r[1].items())}]])
            elif kind == "counters":
                out.append(["counters", adapter.counters()])
            elif kind == "state":
                out.append(["state", adapter.states()])
    finally:
        adapter.close()
    return out


class OracleAdapter:
    def open(self, mode, cap):
        from oracle.ring import OracleChannel
        self.ch = OracleChannel(mode, cap, LABELS)

    def push(self, fid):
        kind, ev, _ = self.ch.push(fid, fid * 1000, {l: payload(fid, i) for i, l in enumerate(LABELS)})
        return kind, ev

    def register(self, c):
        self.ch.register_consumer(c)

    def acquire(self, c):
        return self.ch.acquire_latest(c)

    def lease_fid(self, le):
        return le.frame_id

    def consume(self, le, labels):
        return self.ch.consume(le, labels)

    def release(self, le):
        self.ch.release(le)

    def pop(self, c):
        return self.ch.pop(c)

    def counters(self):
        return self.ch.counters()

    def states(self):
        return sorted(self.ch.state)

    def close(self):
        pass


class RefAdapter:
    """The unmodified reference fanpipe (needs baseline/_ref and /dev/shm)."""

    def open(self, mode, cap):
        from oracle.cpu_pipeline import load_fanpipe
        self.ar, self.chm = load_fanpipe()
        self.ns = self.ar.generate_namespace("vpgold")
        specs = [self.ar.TensorSpec(l, self.ar.DType.F32, DIMS) for l in LABELS]
        m = self.chm.ChannelMode.FIFO if mode == "fifo" else self.chm.ChannelMode.LATEST
        self.ch, _ = self.chm.create_channel("g", m, cap, specs, self.ns)
        self.dst = self.chm.create_processing_slots(self.ns, "dst", specs)

    def push(self, fid):
        def w(views):
            for i, l in enumerate(LABELS):
                views[l][...] = payload(fid, i)
        o = self.ch.push(fid, fid * 1000, w)
        return o.kind.value, o.evicted_frame_id

    def register(self, c):
        self.ch.register_consumer(c)

    def acquire(self, c):
        return self.ch.acquire_latest(c)

    def lease_fid(self, le):
        return le.frame_id

    def consume(self, le, labels):
        env = self.ch.consume(le, self.dst, labels)
        return {l: self.dst.view(l).copy() for l in env.labels}

    def release(self, le):
        self.ch.release(le)

    def pop(self, c):
        env = self.ch.pop(c, self.dst)
        if env is None:
            return None
        return env.frame_id, {l: self.dst.view(l).copy() for l in LABELS}

    def counters(self):
        c = self.ch.counters()
        return dict(pushed=c.pushed, producer_drops=c.producer_drops, evictions=c.evictions,
                    consumed=c.consumed, resident=c.resident)

    def states(self):
        return sorted(s for s, _ in self.ch.slot_states())

    def close(self):
        self.ch.close()
        self.ch.unlink()
        self.ar.clean_namespace(self.ns)


class VpeAdapter:
    """The product device ring through paper_2508_11584_b200.channels."""

    def __init__(self, device: int = -2):
        self.device = device

    def open(self, mode, cap):
        import torch
        from paper_2508_11584_b200 import arena as ar
        from paper_2508_11584_b200 import channels as ch
        self.torch, self.chm = torch, ch
        self.ns = ar.generate_namespace("vpt")
        specs = [ar.TensorSpec(l, ar.DType.F32, DIMS) for l in LABELS]
        m = ch.ChannelMode.FIFO if mode == "fifo" else ch.ChannelMode.LATEST
        self.ch, _ = ch.create_channel("g", m, cap, specs, self.ns, device=self.device)
        dev = -2 if self.device < 0 else self.device
        self.dst = ch.create_processing_slots(self.ns, "dst", specs, device=dev)

    def push(self, fid):
        def w(views):
            for i, l in enumerate(LABELS):
                views[l].copy_(self.torch.from_numpy(payload(fid, i)))
        o = self.ch.push(fid, fid * 1000, w)
        return o.kind.value, o.evicted_frame_id

    def register(self, c):
        self.ch.register_consumer(c)

    def acquire(self, c):
        return self.ch.acquire_latest(c)

    def lease_fid(self, le):
        return le.frame_id

    def consume(self, le, labels):
        env = self.ch.consume(le, self.dst, labels)
        if self.device >= 0:
            self.torch.cuda.synchronize()
        return {l: self.dst.view(l).cpu().numpy().copy() for l in env.labels}

    def release(self, le):
        self.ch.release(le)

    def pop(self, c):
        env = self.ch.pop(c, self.dst)
        if env is None:
            return None
        if self.device >= 0:
            self.torch.cuda.synchronize()
        return env.frame_id, {l: self.dst.view(l).cpu().numpy().copy() for l in LABELS}

    def counters(self):
        c = self.ch.counters()
        return dict(pushed=c.pushed, producer_drops=c.producer_drops, evictions=c.evictions,
                    consumed=c.consumed, resident=c.resident)

    def states(self):
        return sorted(s for s, _ in self.ch.slot_states())

    def close(self):
        self.ch.close()
        from paper_2508_11584_b200 import arena as ar
        self.dst.arena.close()
        if hasattr(self.dst.arena, "unlink"):
            self.dst.arena.unlink()
        ar.forget_allocation(f"{self.ns}.dst")
        assert not ar.shm_census(self.ns), ar.shm_census(self.ns)
