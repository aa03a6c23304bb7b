"""Multi-rank host logic on CPU: world_size-2 gloo process groups exercise the
argmin reduction, sharding and matrix broadcast used by the multi-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2105_14088_b200 import dist as rwdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def _argmin_case(rank, world):
    # rank 0 owns (5.0, key 9), rank 1 owns (5.0, key 4): tie on cost -> smaller key wins
    cost, key = (5.0, 9) if rank == 0 else (5.0, 4)
    payload = np.full(6, rank, dtype=np.int32)
    return rwdist.reduce_argmin(cost, key, payload, 6)


def test_reduce_argmin_ties_to_smallest_key():
    res = run(_argmin_case)
    for best, key, payload in res:
        assert best == 5.0 and key == 4 and payload.tolist() == [1] * 6


def _argmin_cost_case(rank, world):
    cost, key = (3.0, 100) if rank == 1 else (7.0, 1)
    return rwdist.reduce_argmin(cost, key, np.arange(4, dtype=np.int32) + 10 * rank, 4)


def test_reduce_argmin_smaller_cost_wins():
    for best, key, payload in run(_argmin_cost_case):
        assert best == 3.0 and key == 100 and payload.tolist() == [10, 11, 12, 13]


def _bcast_case(rank, world):
    m = np.arange(16, dtype=np.float64).reshape(4, 4) if rank == 0 else None
    return rwdist.broadcast_matrix(m, 4)


def test_broadcast_matrix():
    for m in run(_bcast_case):
        assert np.array_equal(m, np.arange(16, dtype=np.float64).reshape(4, 4))


@pytest.mark.parametrize("total,world", [(10, 2), (479001600, 4), (3, 4), (65536, 8)])
def test_shard_partition(total, world):
    parts = [rwdist.shard(total, r, world) for r in range(world)]
    assert sum(c for _, c in parts) == total
    assert all(parts[k][0] + parts[k][1] == parts[k + 1][0] for k in range(world - 1))


def _world4_case(rank, world):
    # exhaustive-style reduction: each rank's (min cost, min lex index) of its slice
    data = {0: (12.0, 7), 1: (11.0, 250), 2: (11.0, 130), 3: (15.0, 2)}
    return rwdist.reduce_argmin(*data[rank])[:2]


def test_world4_exhaustive_reduction():
    for best, key in run(_world4_case, world=4):
        assert (best, key) == (11.0, 130)
