"""The N>1 bench path (replicas, max-over-ranks device time) on CPU with gloo, world size 2."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local = 0.5 + rank  # pretend device seconds
    t_max = bench.reduce_max(local, device="cpu")
    value = bench.replica_value(n_sub=512, steps=100, world=world, t_max=t_max)
    q.put((rank, t_max, value, bench._dist()))
    dist.destroy_process_group()


def test_replicas_take_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [1.5, 1.5]
    assert all(abs(r[2] - 2 * 512 * 100 / 1.5) < 1e-6 for r in res)
    assert res[1][3] == (2, 1, 1)
