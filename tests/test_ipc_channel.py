"""Cross-process feature ring (each head runs in its own
process). A producer process creates a shared LATEST channel; a consumer process attaches with
``open_channel(handle)`` and reads the frames in place. The control block is POSIX shared memory
with the reference's CAS protocol; on the GPU the HBM arena and the ready / done events cross the
process boundary through CUDA IPC."""
import os
import time

import pytest
import torch
import torch.multiprocessing as mp

N_FRAMES = 40
CID = 7


def _specs():
    from paper_2508_11584_b200.arena import DType, TensorSpec
    return [TensorSpec("final", DType.BF16, (2, 17, 64)), TensorSpec("layer3", DType.F32, (2, 17, 64))]


def _producer(device, box, registered, done):
    import torch
    from paper_2508_11584_b200.arena import generate_namespace
    from paper_2508_11584_b200.channels import ChannelMode, create_channel
    if device >= 0:
        torch.cuda.set_device(device)
    ch, handle = create_channel("feat", ChannelMode.LATEST, 4, _specs(), generate_namespace(),
                                expected_consumers=1, device=device, shared=True)
    box["handle"] = handle.to_dict()
    assert registered.wait(60), "consumer never attached"
    for fid in range(1, N_FRAMES + 1):
        def writer(views, fid=fid):
            for t in views.values():
                t.fill_(float(fid % 200))
        ch.push(fid, fid * 1000, writer)
        if device >= 0:
            torch.cuda.current_stream().synchronize()
        time.sleep(0.002)
    assert done.wait(60), "consumer did not finish"
    c = ch.counters()
    box["pushed"] = int(c.pushed)
    box["consumed"] = int(c.consumed)
    ch.close()


def _consumer(device, box, registered, done):
    import torch
    from paper_2508_11584_b200.channels import ChannelHandle, open_channel
    if device >= 0:
        torch.cuda.set_device(device)
    t0 = time.time()
    while "handle" not in box:
        assert time.time() - t0 < 60
        time.sleep(0.01)
    ch = open_channel(ChannelHandle.from_dict(box["handle"]))
    ch.register_consumer(CID)
    registered.set()
    seen, bad, last = 0, 0, 0
    t0 = time.time()
    while last < N_FRAMES and time.time() - t0 < 60:
        lease = ch.acquire_latest(CID)
        if lease is None:
            time.sleep(0.0005)
            continue
        views = ch.view(lease)
        want = float(lease.frame_id % 200)
        ok = all(bool((v == want).all()) for v in views.values())  # read in place (zero copy)
        bad += 0 if ok else 1
        assert lease.frame_id > last
        last = lease.frame_id
        seen += 1
        ch.commit(lease)
    box["seen"], box["bad"], box["last"] = seen, bad, last
    done.set()
    ch.close()


def _role(rank, device, box, registered, done):
    (_producer if rank == 0 else _consumer)(device, box, registered, done)


def _run(device):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    box, registered, done = mgr.dict(), mgr.Event(), mgr.Event()
    mp.start_processes(_role, args=(device, box, registered, done), nprocs=2, join=True, start_method="spawn")
    return dict(box)


def test_shared_channel_two_processes_host():
    """VPE_HOST_PLAIN ring: control block + data in POSIX shared memory, no CUDA."""
    out = _run(-2)
    assert out["bad"] == 0
    assert out["last"] == N_FRAMES            # the newest frame always reaches the consumer
    assert 1 <= out["seen"] <= N_FRAMES
    assert out["pushed"] == N_FRAMES
    assert out["consumed"] == out["seen"]     # counters are shared across the processes


def test_attach_missing_channel_is_not_found():
    from paper_2508_11584_b200 import _lib  # noqa: F401
    from paper_2508_11584_b200.arena import generate_namespace
    from paper_2508_11584_b200.channels import ChannelHandle, ChannelMode, create_channel, open_channel
    from paper_2508_11584_b200.errors import AlreadyExists, NotFound
    ns = generate_namespace()
    ch, handle = create_channel("solo", ChannelMode.LATEST, 3, _specs(), ns, device=-2, shared=True)
    with pytest.raises(AlreadyExists):  # one creator per name
        create_channel("solo", ChannelMode.LATEST, 3, _specs(), ns, device=-2, shared=True)
    d = handle.to_dict()
    ch.close()                               # creator unlinks the segments
    with pytest.raises(NotFound):
        open_channel(ChannelHandle.from_dict(d))


@pytest.mark.gpu
def test_shared_channel_two_processes_cuda_ipc():
    """HBM ring exported with cudaIpcGetMemHandle; ready/done events are interprocess events."""
    out = _run(0)
    assert out["bad"] == 0
    assert out["last"] == N_FRAMES
    assert out["pushed"] == N_FRAMES
    assert out["consumed"] == out["seen"]
