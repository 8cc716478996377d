"""Multi-process host logic of the video-sharded path, world_size 2 over gloo
on CPU (the GPU runs use NCCL through the same functions)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_06545_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = D.shard_videos(7, world, rank)
        allv = D.gather_objects(mine)
        slowest = D.max_over_ranks(1.5 + rank)
        t = torch.tensor([1.0 + rank, 2.0], dtype=torch.float64)
        D.allreduce_sum(t)
        q.put((rank, allv, slowest, t.tolist(), D.video_seeds(mine, 100)))
    finally:
        dist.destroy_process_group()


def test_shard_and_collectives_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, allv, slowest, t, seeds in res:
        flat = sorted(v for part in allv for v in part)
        assert flat == list(range(7))                     # disjoint and complete
        assert slowest == 2.5                             # max over ranks
        assert t == [3.0, 4.0]                            # summed decision inputs
        assert seeds == [100 + v for v in allv[rank]]     # seed follows the video


@pytest.mark.parametrize("n,w", [(1, 1), (8, 8), (10, 4), (3, 4)])
def test_shard_balance(n, w):
    parts = [D.shard_videos(n, w, r) for r in range(w)]
    assert sorted(v for p in parts for v in p) == list(range(n))
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
