"""Transport parity on CPU (no GPU needed): the oracle restatement and the product ring
(libvpe's C++ state machine, data arena in host memory) reproduce the UNMODIFIED reference's
outcomes on the SPEC known-answer examples and on seeded random schedules."""

import ctypes
import json
import os
import re

import numpy as np
import pytest

from transport_schedules import OracleAdapter, RefAdapter, VpeAdapter, random_scenario, run

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))
HAVE_REF = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "fanpipe"))


def _norm(x):
    return json.loads(json.dumps(x))


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_oracle_matches_reference_golden(name):
    g = GOLDEN[name]
    sc = _norm(g["scenario"])
    sc["ops"] = [tuple(o) if not isinstance(o, str) else o for o in sc["ops"]]
    assert _norm(run(OracleAdapter(), sc)) == g["outcomes"]


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_vpe_ring_matches_reference_golden(name):
    g = GOLDEN[name]
    sc = _norm(g["scenario"])
    sc["ops"] = [tuple(o) for o in sc["ops"]]
    assert _norm(run(VpeAdapter(device=-2), sc)) == g["outcomes"]


@pytest.mark.skipif(not HAVE_REF, reason="baseline/_ref not installed")
@pytest.mark.parametrize("seed,mode,cap", [(11, "latest", 3), (12, "latest", 6), (13, "fifo", 3)])
def test_live_three_way(seed, mode, cap):
    sc = random_scenario(seed, mode, cap, consumers=3, n=400)
    ref = _norm(run(RefAdapter(), sc))
    assert _norm(run(OracleAdapter(), sc)) == ref
    assert _norm(run(VpeAdapter(device=-2), sc)) == ref


def test_single_copy_discipline():
    """SPEC.md:196-198 + arena.py:367-373: one copy per consumed label, views copy nothing."""
    from paper_2508_11584_b200 import arena as ar
    sc = GOLDEN["selective"]["scenario"]
    sc = dict(sc, ops=[tuple(o) for o in sc["ops"]])
    before = ar.copy_counter()
    run(VpeAdapter(device=-2), sc)
    assert ar.copy_counter() - before == 4 + 1 + 1


def test_view_and_commit_are_zero_copy():
    import torch
    from paper_2508_11584_b200 import arena as ar
    from paper_2508_11584_b200 import channels as ch
    ns = ar.generate_namespace("vz")
    specs = [ar.TensorSpec("final", ar.DType.BF16, (2, 5, 8))]
    c, h = ch.create_channel("z", ch.ChannelMode.LATEST, 3, specs, ns, device=-2)
    c.register_consumer(1)
    c.push(1, 10, lambda v: v["final"].fill_(3.0))
    before = ar.copy_counter()
    lease = c.acquire_latest(1)
    v = c.view(lease, ["final"])["final"]
    assert v.dtype == torch.bfloat16 and float(v.float().mean()) == 3.0
    env = c.commit(lease)
    assert env.frame_id == 1 and c.last_consumed(1) == 1
    assert ar.copy_counter() == before
    with pytest.raises(Exception) as ei:
        c.commit(lease)
    assert type(ei.value).__name__ == "UseAfterConsume"
    assert c.acquire_latest(1) is None
    # PECH1 header layout (channels.py:14-26)
    hdr = c.header_bytes()
    assert hdr[:6] == b"PECH1\x00" and hdr[6] == 1 and int.from_bytes(hdr[8:12], "little") == 3
    state0 = int.from_bytes(hdr[16:20], "little")
    assert state0 == 2  # READY, lease dropped
    c.close()


def test_errors_match_reference():
    from paper_2508_11584_b200 import arena as ar
    from paper_2508_11584_b200 import channels as ch
    from paper_2508_11584_b200.errors import ConfigError, LabelError, ShapeError, WriterError
    ns = ar.generate_namespace("ve")
    specs = [ar.TensorSpec("final", ar.DType.F32, (4,)), ar.TensorSpec("layer3", ar.DType.F32, (4,))]
    with pytest.raises(ConfigError):
        ch.create_channel("a", ch.ChannelMode.LATEST, 0, specs, ns, device=-2)
    with pytest.raises(ConfigError):
        ch.create_channel("b", ch.ChannelMode.LATEST, 2, [specs[0], specs[0]], ns, device=-2)
    with pytest.raises(ShapeError):
        ar.TensorSpec("bad label", ar.DType.F32, (4,))
    c, _ = ch.create_channel("c", ch.ChannelMode.LATEST, 2, specs, ns, device=-2)
    c.register_consumer(1)

    def boom(v):
        raise RuntimeError("x")

    with pytest.raises(WriterError):
        c.push(1, 1, boom)
    assert c.slot_states()[0][0] == 0  # freed
    c.push(2, 2, lambda v: None)
    with pytest.raises(ValueError):
        c.push(2, 3, lambda v: None)  # frame ids strictly increase
    lease = c.acquire_latest(1)
    with pytest.raises(LabelError):
        c.consume(lease, {}, ["nope"])
    c.release(lease)
    assert c.last_consumed(1) == 0  # release does not advance the cursor
    c.close()


def test_arena_layout_examples():
    """SPEC.md:62-63 known answers."""
    from paper_2508_11584_b200 import arena as ar
    lay = ar.ArenaLayout.from_specs([ar.TensorSpec("x", ar.DType.F32, (3, 224, 224))])
    assert lay.total_bytes >= 602112 and lay.offsets == (0,)
    lay2 = ar.ArenaLayout.from_specs([ar.TensorSpec("a", ar.DType.U8, (5,)), ar.TensorSpec("b", ar.DType.U8, (5,))])
    assert lay2.offsets[1] == 64
    # C2 tap labels: 4 x bf16 [1,1025,384] -> offsets 0 / 787200 / 1574400 / 2361600
    specs = [ar.TensorSpec(l, ar.DType.BF16, (1, 1025, 384)) for l in ("layer3", "layer6", "layer9", "final")]
    assert ar.ArenaLayout.from_specs(specs).offsets == (0, 787200, 1574400, 2361600)


def test_atomic_buffer_semantics():
    """_kernels.pyx:56-98: acquire/release word ops, CAS returns previous, ValueError on bad offsets."""
    from paper_2508_11584_b200.kernels import AtomicBuffer, HAVE_COMPILED, active_backend
    assert HAVE_COMPILED and active_backend() == "compiled"
    buf = np.zeros(64, dtype=np.uint8)
    a = AtomicBuffer(buf)
    a.u32_store(0, 7)
    assert a.u32_load(0) == 7
    assert a.u32_cas(0, 7, 9) == 7 and a.u32_load(0) == 9
    assert a.u32_cas(0, 7, 11) == 9 and a.u32_load(0) == 9
    a.u64_store(8, 2**40)
    assert a.u64_add(8, 5) == 2**40 and a.u64_load(8) == 2**40 + 5
    for bad in (-4, 2, 62, 64):
        with pytest.raises(ValueError):
            a.u32_load(bad)
    with pytest.raises(ValueError):
        a.u64_load(4)
    if HAVE_REF:
        from oracle.cpu_pipeline import load_fanpipe
        load_fanpipe()
        from fanpipe import _kernels
        r = _kernels.AtomicBuffer(bytearray(64))
        for off in (-4, 2, 62, 64):
            with pytest.raises(ValueError):
                r.u32_load(off)


def test_library_exports_every_declared_symbol():
    """include/vpe.h is the drop-in boundary; libvpe.so must export all of it."""
    from paper_2508_11584_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "vpe.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+\*?(vpe_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 60
    so = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(so, s)]
    assert not missing, missing
    assert declared <= set(_lib.EXPORTS)
