"""World-size-2 gloo run of the multi-GPU host logic (stream sharding, barrier, max-over-ranks)
on CPU: each rank drives its own shard of camera streams through the CPU oracle with no
collective on the data path; only the timing is reduced."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_11584_b200.sharding import max_over_ranks, streams_for_rank, total_frames
    from paper_2508_11584_b200.weights import make_frames
    mine = streams_for_rank(6, rank, world)
    # per-stream work: seeded frames (stream-specific seeds); no cross-rank exchange
    checks = [int(make_frames(1, 28, s).sum()) for s in mine]
    dist.barrier()
    dt = max_over_ranks(0.5 + rank, dist)
    n = total_frames(len(mine), dist)
    out[rank] = (mine, checks, dt, n)
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    s0, c0, dt0, n0 = out[0]
    s1, c1, dt1, n1 = out[1]
    assert sorted(s0 + s1) == list(range(6)) and not set(s0) & set(s1)
    assert dt0 == dt1 == 1.5          # max over ranks
    assert n0 == n1 == 6              # whole-job frame count
    from paper_2508_11584_b200.weights import make_frames
    assert c0[0] == int(make_frames(1, 28, s0[0]).sum())


def test_streams_for_rank_errors():
    from paper_2508_11584_b200.sharding import streams_for_rank
    with pytest.raises(ValueError):
        streams_for_rank(4, 2, 2)
    assert streams_for_rank(8, 3, 8) == [3]
