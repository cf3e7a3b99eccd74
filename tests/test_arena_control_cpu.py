"""CPU tests of the drop-in arena surface (reference arena.py:233-413 /
channels.py:179-196), the control transport and registry-driven deployment
validation (VPEngine.from_cards). Regions here use the POSIX shared-memory
placement (device=-2); the HBM placement runs the same code in tests/test_gpu_ring.py."""

import json
import os
import subprocess
import sys
import threading

import pytest
import torch

from paper_2508_11584_b200 import arena as ar
from paper_2508_11584_b200 import channels as chm
from paper_2508_11584_b200.control import ControlServer, read_message, send, write_message
from paper_2508_11584_b200.errors import AlreadyExists, ConfigError, CorruptHandle, NotFound, ShapeError

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
HAVE_REF = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "fanpipe"))
HOST = -2


@pytest.fixture
def ns():
    n = ar.generate_namespace("vpa")
    yield n
    ar.clean_namespace(n)


def test_arena_layout_examples(ns):
    """one F32 [3,224,224] slot -> >= 602,112 bytes at offset 0; two U8 [5]
    slots -> second offset 64; a duplicate region name -> AlreadyExists."""
    lay = ar.ArenaLayout.from_specs([ar.TensorSpec("x", ar.DType.F32, (3, 224, 224))])
    a, h = ar.create_arena(lay, ns, "one", device=HOST)
    assert h.total_bytes >= 602112 and lay.offset_of(0) == 0
    lay2 = ar.ArenaLayout.from_specs([ar.TensorSpec("a", ar.DType.U8, (5,)), ar.TensorSpec("b", ar.DType.U8, (5,))])
    assert lay2.offset_of(1) == 64
    with pytest.raises(AlreadyExists):
        ar.create_arena(lay, ns, "one", device=HOST)
    hdr = bytes(a.buf[:24].numpy())
    assert hdr[:6] == b"PEAR1\x00" and int.from_bytes(hdr[8:16], "little") == h.total_bytes
    assert int.from_bytes(hdr[16:20], "little") == 1
    a.close()


def test_import_write_through_and_errors(ns):
    """0xAB written by the creator is read by an importer; a tampered handle
    -> CorruptHandle; an unknown region -> NotFound."""
    spec = ar.TensorSpec("x", ar.DType.U8, (16,))
    lay = ar.ArenaLayout.from_specs([spec])
    a, h = ar.create_arena(lay, ns, "wt", device=HOST)
    ref = ar.SlotRef(h, 0, spec, 0)
    a.data_view(0, spec)[5] = 0xAB
    b = ar.import_arena(h)
    assert int(b.data_view(0, spec)[5]) == 0xAB
    b.data_view(0, spec)[6] = 0xCD  # and back
    assert int(ar.read_view(ref)[6]) == 0xCD
    with pytest.raises(CorruptHandle):
        ar.import_arena(ar.ShareHandle(h.namespace, h.region_name, h.total_bytes + 4096, HOST))
    with pytest.raises(CorruptHandle):
        ar.import_arena(ar.ShareHandle(h.namespace, h.region_name, h.total_bytes - 4096, HOST))
    with pytest.raises(NotFound):
        ar.import_arena(ar.ShareHandle(ns, "nope", 4096, HOST))
    b.close()
    a.close()


def test_write_tensor_read_view_copy_out(ns):
    """write_tensor roundtrip / ShapeError; read_view aliases and copies
    nothing; copy_out snapshots and bumps the copy counter by exactly one."""
    spec = ar.TensorSpec("img", ar.DType.F32, (3, 224, 224))
    lay = ar.ArenaLayout.from_specs([spec, spec])
    a, h = ar.create_arena(lay, ns, "rw", device=HOST)
    src, dst = ar.SlotRef(h, 0, spec, lay.offset_of(0)), ar.SlotRef(h, 1, spec, lay.offset_of(1))
    data = torch.randn(3, 224, 224)
    ar.write_tensor(src, data.numpy().tobytes())
    c0 = ar.copy_counter()
    v = ar.read_view(src)
    assert torch.equal(v, data) and ar.copy_counter() == c0
    with pytest.raises(ShapeError):
        ar.write_tensor(src, b"\x00" * 10)
    ar.copy_out(src, dst)
    assert ar.copy_counter() == c0 + 1
    ar.write_tensor(src, torch.zeros(3, 224, 224))
    assert torch.equal(ar.read_view(dst), data)       # snapshot: dst unchanged by the later write
    assert float(v.abs().sum()) == 0.0                 # the view aliases: it sees the overwrite
    other = ar.SlotRef(h, 1, ar.TensorSpec("img", ar.DType.F32, (3, 224, 223)), lay.offset_of(1))
    with pytest.raises(ShapeError):
        ar.copy_out(src, other)
    a.close()


def test_census_and_clean(ns):
    lay = ar.ArenaLayout.from_specs([ar.TensorSpec("x", ar.DType.U8, (8,))])
    a, h = ar.create_arena(lay, ns, "c1", device=HOST)
    a2, _ = ar.create_arena(lay, ns, "c2", device=HOST)
    cen = ar.shm_census(ns)
    assert set(cen) == {f"{ns}.c1", f"{ns}.c2"} and all(v == h.total_bytes for v in cen.values())
    assert sorted(ar.clean_namespace(ns)) == sorted(cen)
    assert ar.shm_census(ns) == {}
    a.close()
    a2.close()


def test_cross_process_processing_slots(ns):
    """open_processing_slots (channels.py:189-196) in another process sees the creator's bytes
    and its writes come back (POSIX placement; the HBM placement is the GPU test)."""
    specs = [ar.TensorSpec("final", ar.DType.F32, (4, 8)), ar.TensorSpec("aux", ar.DType.I64, (3,))]
    g = chm.create_processing_slots(ns, "dst", specs, device=HOST)
    g.view("final").copy_(torch.arange(32, dtype=torch.float32).reshape(4, 8))
    h = g.ref("final").arena
    code = f"""
import json, sys, torch
sys.path.insert(0, {ROOT!r})
from paper_2508_11584_b200 import arena as ar, channels as chm
h = ar.ShareHandle.from_dict(json.loads({json.dumps(json.dumps(h.to_dict()))}))
specs = [ar.TensorSpec("final", ar.DType.F32, (4, 8)), ar.TensorSpec("aux", ar.DType.I64, (3,))]
g = chm.open_processing_slots(h, specs)
print(float(g.view("final").sum()))
g.view("aux").copy_(torch.tensor([7, 8, 9]))
g.arena.close()
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert float(r.stdout.strip()) == float(sum(range(32)))
    assert g.view("aux").tolist() == [7, 8, 9]
    g.arena.close()


@pytest.mark.skipif(not HAVE_REF, reason="baseline/_ref not installed")
def test_arena_layout_matches_reference(ns):
    """Offsets, total size and the 64-byte PEAR1 header are byte-identical to the unmodified
    reference's create_arena for the C2 ring's slot group."""
    from oracle.cpu_pipeline import load_fanpipe
    rar, _ = load_fanpipe()
    dims = (1, 1025, 384)
    ours = ar.ArenaLayout.from_specs([ar.TensorSpec(l, ar.DType.F16_RAW, dims) for l in ("a", "b", "c", "d")] * 5)
    theirs = rar.ArenaLayout.from_specs([rar.TensorSpec(l, rar.DType.F16_RAW, dims) for l in ("a", "b", "c", "d")] * 5)
    assert ours.offsets == theirs.offsets and ours.total_bytes == theirs.total_bytes
    a, _ = ar.create_arena(ours, ns, "mine", device=HOST)
    b, hb = rar.create_arena(theirs, ns, "theirs")
    assert bytes(a.buf[:64].numpy()) == bytes(b.buf[:64])
    a.close()
    b.close()


def test_atomic_buffer_pins_its_buffer():
    """the export stays pinned while the AtomicBuffer lives (no resize under it)."""
    from paper_2508_11584_b200.kernels import make_atomics
    buf = bytearray(64)
    a = make_atomics(buf)
    a.u64_store(8, 41)
    assert a.u64_add(8, 1) == 41 and a.u64_load(8) == 42
    with pytest.raises(BufferError):
        buf.extend(b"x")
    a.close()
    buf.extend(b"x")


# ---- control transport ------------------------------------------------------------------------
def test_control_roundtrip(tmp_path):
    """Length-prefixed request/reply, one reply per request in order; malformed payload ->
    ProtocolError reply; the CLI client in another process."""
    seen = []

    def dispatch(cmd):
        seen.append(cmd)
        tag = cmd.split()[0]
        return "OK" if tag != "STATS" else "OK " + json.dumps({"n": len(seen)})

    path = str(tmp_path / "ctl.sock")
    with ControlServer(dispatch, path):
        r = send(path, "SETRATE depth 10", "PAUSE seg", "STATS")
        assert r[:2] == ["OK", "OK"] and json.loads(r[2][3:]) == {"n": 3}
        import socket
        import struct
        with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as s:
            s.connect(path)
            s.sendall(struct.pack("<I", 2) + b"\xff\xfe")
            assert read_message(s).startswith("ERR ProtocolError")
        out = subprocess.run([sys.executable, "-m", "paper_2508_11584_b200.control", path, "RESUME", "seg"],
                             capture_output=True, text=True, cwd=ROOT, timeout=120)
        assert out.returncode == 0 and out.stdout.strip() == "OK", out.stderr
    assert seen == ["SETRATE depth 10", "PAUSE seg", "STATS", "RESUME seg"]
    assert not os.path.exists(path)


def test_control_concurrent_clients(tmp_path):
    lock = threading.Lock()
    count = [0]

    def dispatch(cmd):
        with lock:
            count[0] += 1
        return f"OK {cmd}"

    path = str(tmp_path / "c.sock")
    with ControlServer(dispatch, path):
        res = {}

        def client(i):
            res[i] = send(path, *[f"PAUSE h{i}_{k}" for k in range(20)])

        ts = [threading.Thread(target=client, args=(i,)) for i in range(4)]
        [t.start() for t in ts]
        [t.join() for t in ts]
    assert count[0] == 80
    for i in range(4):
        assert res[i] == [f"OK PAUSE h{i}_{k}" for k in range(20)]


# ---- registry-driven deployment: validation happens before any device work --------------------
def _cards(R=224, B=1):
    from paper_2508_11584_b200.config import model_config
    from paper_2508_11584_b200.registry import demo_cards
    return demo_cards(model_config("vits14"), R, B)


def test_from_cards_rejects_invalid_deployments():
    from dataclasses import replace

    from paper_2508_11584_b200.engine import VPEngine
    from paper_2508_11584_b200.arena import DType, TensorSpec
    fm, heads = _cards()
    with pytest.raises(ConfigError, match="foundation"):
        VPEngine.from_cards(heads[0], heads)
    with pytest.raises(ConfigError, match="b200_vit"):
        VPEngine.from_cards(replace(fm, backend={"kind": "trt"}), heads)
    # FM outputs that are not what b200_vit writes (dtype F32 instead of BF16)
    bad_out = tuple(TensorSpec(s.label, DType.F32, s.dims) for s in fm.output_specs)
    with pytest.raises(ConfigError, match="taps"):
        VPEngine.from_cards(replace(fm, output_specs=bad_out), heads)
    # a head subscribing a label the FM does not emit (validate_deployment report)
    ghost = replace(heads[1], input_specs=(TensorSpec("layer99", DType.BF16, fm.output_specs[0].dims),))
    with pytest.raises(ConfigError, match="layer99"):
        VPEngine.from_cards(fm, [heads[0], ghost])
    with pytest.raises(ConfigError, match="unknown head backend"):
        VPEngine.from_cards(fm, [replace(heads[2], backend={"kind": "pytorch_frcnn"})])
    with pytest.raises(ConfigError, match="expected a head card"):
        VPEngine.from_cards(fm, [fm])
