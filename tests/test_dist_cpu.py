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


# ---------------------------------------------------------------- synchronised mode
L_SYNC, H_SYNC, V_SYNC, SHAPE = 3, 2, 5, (6, 4)


def _sync_features():
    """Deterministic per-video features: out/ref/prev per layer, the SRAP
    pairs, x_{t-1} and its history."""
    import numpy as np
    rng = np.random.default_rng(11)
    f = lambda *s: rng.standard_normal(s).astype(np.float32)
    return dict(out=f(L_SYNC, V_SYNC, *SHAPE), ref=f(L_SYNC, V_SYNC, *SHAPE),
                prev=f(L_SYNC, V_SYNC, *SHAPE), a=f(L_SYNC, V_SYNC, *SHAPE),
                b=f(L_SYNC, V_SYNC, *SHAPE), x=f(V_SYNC, *SHAPE), hist=f(H_SYNC, V_SYNC, *SHAPE))


def _local_sums(fe, vids):
    """The per-(layer, video) sums the device reductions produce."""
    import numpy as np
    d = lambda k: np.asarray(fe[k], np.float64)[:, vids]
    hlc = np.stack([np.abs(d("out") - d("ref")).sum((2, 3)),
                    ((d("out") - d("prev")) ** 2).sum((2, 3))], -1)
    srap = np.stack([(d("a") * d("b")).sum((2, 3)), (d("a") ** 2).sum((2, 3)),
                     (d("b") ** 2).sum((2, 3))], -1)
    x = np.asarray(fe["x"], np.float64)[vids]
    l1 = np.abs(x[None] - d("hist")).sum((2, 3))
    return hlc, srap, l1


def _sync_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = D.shard_videos(V_SYNC, world, rank)
        hlc, srap, l1 = (torch.from_numpy(a) for a in _local_sums(_sync_features(), mine))
        vec = torch.zeros(D.decision_vector_len(L_SYNC, H_SYNC - 1), dtype=torch.float64)
        D.pack_decision_sums(vec, hlc, srap, l1)
        D.allreduce_sum(vec)
        q.put((rank, vec.tolist()))
    finally:
        dist.destroy_process_group()


def test_sync_decision_allreduce_equals_concatenated_batch():
    """One all-reduce of the packed per-rank sums gives every rank the
    reference formulas (divergence, similarity, variation; schedule.py:67-133)
    evaluated on the concatenated batch of all ranks' videos."""
    import numpy as np
    from oracle import qc_oracle as O
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sync_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1]                      # every rank: identical inputs
    vec = np.array(res[0][1])
    fe = _sync_features()
    L = L_SYNC
    for l in range(L):
        k = 3
        d_got = (vec[2 * l] / k) * np.sqrt(vec[2 * l + 1])
        d_ref = O.divergence5(fe["out"][l], fe["ref"][l], k, fe["out"][l], fe["prev"][l])
        assert d_got == pytest.approx(d_ref, rel=1e-12)
        dot, na, nb = vec[2 * L + 3 * l: 2 * L + 3 * l + 3]
        assert dot / (np.sqrt(na) * np.sqrt(nb)) == pytest.approx(
            O.similarity(fe["a"][l], fe["b"][l]), rel=1e-12)
    v_got = vec[5 * L:5 * L + H_SYNC].sum()
    assert v_got == pytest.approx(O.variation(list(fe["hist"]), fe["x"]), rel=1e-12)
