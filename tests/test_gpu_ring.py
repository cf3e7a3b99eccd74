"""The HBM feature ring on the B200 (SPEC.md:123-219 channel properties, reference
channels.py): the reference's golden outcomes replayed on a device ring, RAW/WAR ordering with a
legacy-default-stream consumer, a >= 1e5-frame torn-read stress with concurrent producer and
consumer streams, long-held leases, and cross-process HBM arenas through CUDA IPC."""

import json
import os
import subprocess
import sys

import pytest
import torch

from transport_schedules import VpeAdapter, run

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


def _norm(x):
    return json.loads(json.dumps(x))


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2508_11584_b200 import arena as ar
    from paper_2508_11584_b200 import channels as ch
    return ar, ch


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_device_ring_matches_reference_golden(mods, name):
    """Every golden scenario from the unmodified reference, on an HBM ring (device 0)."""
    g = GOLDEN[name]
    sc = _norm(g["scenario"])
    sc["ops"] = [tuple(o) for o in sc["ops"]]
    assert _norm(run(VpeAdapter(device=0), sc)) == g["outcomes"]


def _ring(mods, cap, n=2 ** 16, labels=("a", "b"), consumers=(1,)):
    ar, ch = mods
    ns = ar.generate_namespace("vpg")
    specs = [ar.TensorSpec(l, ar.DType.F32, (n,)) for l in labels]
    c, _ = ch.create_channel("r", ch.ChannelMode.LATEST, cap, specs, ns, device=0)
    for cid in consumers:
        c.register_consumer(cid)
    return c, specs, ns


def test_default_stream_consumer_raw_and_war(mods):
    """a consumer that passes no stream (legacy default stream) must still
    wait for the producer's writes (RAW) and the producer must wait for its reads (WAR); no
    host synchronisation in between."""
    ar, ch = mods
    c, specs, ns = _ring(mods, cap=2)
    prod = torch.cuda.Stream()
    n = specs[0].dims[0]

    def writer(fid):
        def w(views):
            with torch.cuda.stream(prod):
                torch.cuda._sleep(20_000_000)  # ~10 ms: the producer is slow to finish
                for v in views.values():
                    v.fill_(float(fid))
        return w

    c.push(1, 1, writer(1), stream=prod.cuda_stream)
    lease = c.acquire_latest(1)  # default stream
    dst = {s.label: torch.empty(n, device="cuda") for s in specs}
    torch.cuda._sleep(20_000_000)  # a slow reader on the legacy stream
    c.consume(lease, dst)
    # the producer immediately overwrites every slot (capacity 2): frame 1's slot must not be
    # written before the legacy-stream copy out of it has run
    for fid in (2, 3, 4):
        c.push(fid, fid, writer(fid), stream=prod.cuda_stream)
    torch.cuda.synchronize()
    for v in dst.values():
        assert bool((v == 1.0).all()), float(v.min())
    c.close()


def test_torn_read_stress(mods):
    """>= 1e5 frames, producer on its own stream, three consumers on three streams
    reading the leased slot IN PLACE (view + commit); every read must see exactly the frame id
    it leased. Mismatches are counted on the device (no host sync inside the loop)."""
    ar, ch = mods
    c, specs, ns = _ring(mods, cap=5, n=4096, labels=("l0", "l1", "l2", "final"), consumers=(1, 2, 3))
    prod = torch.cuda.Stream()
    cons = {cid: torch.cuda.Stream(priority=-1) for cid in (1, 2, 3)}
    bad = torch.zeros(3, dtype=torch.int64, device="cuda")
    reads = [0, 0, 0]
    g = torch.Generator().manual_seed(5)
    jitter = torch.randint(0, 4, (1 << 12,), generator=g).tolist()
    N = 100_000
    for fid in range(1, N + 1):
        j = jitter[fid % len(jitter)]

        def w(views, fid=fid, j=j):
            with torch.cuda.stream(prod):
                if j == 0:
                    torch.cuda._sleep(2000)
                for v in views.values():
                    v.fill_(float(fid))

        c.push(fid, fid, w, stream=prod.cuda_stream)
        for k, cid in enumerate((1, 2, 3)):
            if (fid + k) % (k + 1):  # consumers at 1:1, 1:2, 1:3
                continue
            s = cons[cid]
            lease = c.acquire_latest(cid, stream=s.cuda_stream)
            if lease is None:
                continue
            v = c.view(lease, ["l0", "final"])
            with torch.cuda.stream(s):
                if j == 1:
                    torch.cuda._sleep(3000)
                bad[k] += (v["l0"] != float(lease.frame_id)).sum() + (v["final"] != float(lease.frame_id)).sum()
            c.commit(lease, stream=s.cuda_stream)
            reads[k] += 1
    torch.cuda.synchronize()
    assert bad.tolist() == [0, 0, 0]
    assert reads[0] > 0.9 * N and min(reads) > N / 4
    cnt = c.counters()
    assert cnt.pushed == N and cnt.consumed == sum(reads)
    c.close()


def test_long_lease_never_overwritten(mods):
    """a slot under a long-held lease is never overwritten; the producer evicts
    other slots, and only when every slot is leased does it see OverflowRejected."""
    ar, ch = mods
    c, specs, ns = _ring(mods, cap=3, consumers=(1, 2))
    prod = torch.cuda.Stream()

    def w(fid):
        def f(views):
            with torch.cuda.stream(prod):
                for v in views.values():
                    v.fill_(float(fid))
        return f

    c.push(1, 1, w(1), stream=prod.cuda_stream)
    held = c.acquire_latest(1)
    view = c.view(held)
    for fid in range(2, 2002):
        assert c.push(fid, fid, w(fid), stream=prod.cuda_stream).accepted
        if fid % 97 == 0:
            torch.cuda.synchronize()
            assert all(bool((t == 1.0).all()) for t in view.values())
    # a second long lease on the newest frame: now 2 of 3 slots are pinned, pushes still succeed
    second = c.acquire_latest(2)
    assert second.frame_id == 2001
    for fid in range(2002, 2010):
        assert c.push(fid, fid, w(fid), stream=prod.cuda_stream).accepted
    third = c.acquire_latest(1)  # consumer 1 takes a second lease: all 3 slots leased
    assert third is not None
    out = c.push(2010, 2010, w(2010), stream=prod.cuda_stream)
    assert not out.accepted and c.counters().producer_drops == 1
    torch.cuda.synchronize()
    assert all(bool((t == 1.0).all()) for t in view.values())
    for le in (held, second, third):
        c.release(le)
    assert c.push(2011, 2011, w(2011), stream=prod.cuda_stream).accepted
    c.close()


def test_hbm_arena_cross_process(mods):
    """create_arena in HBM, import_arena in another process through CUDA IPC: write-through
    both ways (SPEC.md:71-73 on device memory), then census / clean of the namespace."""
    ar, ch = mods
    ns = ar.generate_namespace("vph")
    spec = ar.TensorSpec("final", ar.DType.F32, (1025, 384))
    lay = ar.ArenaLayout.from_specs([spec, spec])
    a, h = ar.create_arena(lay, ns, "feat", device=0)
    ref0, ref1 = ar.SlotRef(h, 0, spec, lay.offset_of(0)), ar.SlotRef(h, 1, spec, lay.offset_of(1))
    ar.write_tensor(ref0, torch.arange(1025 * 384, dtype=torch.float32).reshape(1025, 384))
    assert set(ar.shm_census(ns)) == {f"{ns}.feat"}
    code = f"""
import json, sys, torch
sys.path.insert(0, {ROOT!r})
from paper_2508_11584_b200 import arena as ar
h = ar.ShareHandle.from_dict(json.loads({json.dumps(json.dumps(h.to_dict()))}))
spec = ar.TensorSpec("final", ar.DType.F32, (1025, 384))
lay = ar.ArenaLayout.from_specs([spec, spec])
a = ar.import_arena(h)
print(float(a.data_view(lay.offset_of(0), spec).double().sum()))
ar.copy_out(ar.SlotRef(h, 0, spec, lay.offset_of(0)), ar.SlotRef(h, 1, spec, lay.offset_of(1)))
torch.cuda.synchronize()
a.close()
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    n = 1025 * 384
    assert float(r.stdout.strip()) == float(n * (n - 1) // 2)
    assert torch.equal(ar.read_view(ref1).cpu(), torch.arange(n, dtype=torch.float32).reshape(1025, 384))
    a.close()
    assert ar.clean_namespace(ns) == [f"{ns}.feat"] and ar.shm_census(ns) == {}
