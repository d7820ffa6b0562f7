"""World-size-2 gloo test of the multi-GPU host logic (sharding, counter and
kept-id reduction) on CPU; the same code runs over NCCL in bench.py."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_11535_b200 import dist as m3dist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f0, n = m3dist.shard(1000, rank, world, weak=True)
        assert (f0, n) == (rank * 1000, 1000)
        lo, cnt = m3dist.shard(1001, rank, world, weak=False)
        counters = torch.tensor([n, 10 * (rank + 1), rank + 1], dtype=torch.float64)
        tot, tmax = m3dist.reduce_counters(counters, step_seconds=0.5 + rank)
        kept_local = torch.arange(rank + 2, dtype=torch.int32) * 3
        ids = m3dist.gather_kept(kept_local, f0)
        q.put((rank, tot.tolist(), tmax, ids.tolist(), (lo, cnt)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, tot, tmax, ids, (lo, cnt) in res:
        assert tot == [2000.0, 30.0, 3.0]
        assert tmax == 1.5
        assert ids == [0, 3, 1000, 1003, 1006]
    assert [r[4] for r in res] == [(0, 500), (500, 501)]
