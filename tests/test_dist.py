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


def test_bench_spawns_ranks_for_gpus_n():
    """bench.py --gpus 2 without an outer torchrun re-launches itself under
    torch.distributed.run (2 ranks, 127.0.0.1); on the reference arm rank 0 alone
    prints the JSON line and rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--ref-frames", "20"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["cpu_baseline"]["cores"] >= 1
