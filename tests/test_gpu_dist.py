"""Multi-process path on one GPU (Sec. V: "each computer working
independently on their individual batch of consecutive frames"): two ranks on
cuda:0 with a gloo group, each filtering its shard of the frames through
m3e_filter, then paper_2206_11535_b200.dist's reduction of counters and
gathering of accepted global frame ids.  The result must equal one process
filtering all frames (the same code runs over NCCL, one GPU per rank, in
bench.py --gpus N)."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_FRAMES, SEED = 30011, 4242


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _counters(res, n):
    sm = res.summary_np()
    kept = int(sum(sm["kept_by_reason"][1:]))
    return [n, int(sm["tracks"]), kept, int(sm["kept_hits"])] + [int(v) for v in sm["kept_by_reason"]], kept


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import synth
    from paper_2206_11535_b200 import dist as m3dist
    from paper_2206_11535_b200 import m3e
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f0, n = m3dist.shard(N_FRAMES, rank, world, weak=False)
        d = synth.generate(synth.preset("phase1_sig", seed=SEED), n, frame0=f0)
        ctx = m3e.Context(0)
        res = m3e.run_filter(ctx, m3e.make_params(m3e.load_config()), m3e.DeviceFrames(d))
        torch.cuda.synchronize()
        c, kept = _counters(res, n)
        tot, tmax = m3dist.reduce_counters(torch.tensor(c, dtype=torch.float64), step_seconds=1.0 + rank)
        ids = m3dist.gather_kept(res.kept_frame[:kept].cpu(), f0)
        q.put((rank, tot.tolist(), tmax, ids.tolist()))
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_process():
    import torch.multiprocessing as mp

    import synth
    from paper_2206_11535_b200 import m3e
    world, port = 2, _free_port()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    ps = [mpc.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    # one process over all frames
    d = synth.generate(synth.preset("phase1_sig", seed=SEED), N_FRAMES)
    ctx = m3e.Context(0)
    res = m3e.run_filter(ctx, m3e.make_params(m3e.load_config()), m3e.DeviceFrames(d))
    torch.cuda.synchronize()
    c, kept = _counters(res, N_FRAMES)
    ids = res.kept_frame[:kept].cpu().numpy().astype(np.int64).tolist()
    ctx.close()
    for rank, tot, tmax, gids in out:
        assert [int(v) for v in tot] == c
        assert tmax == 2.0            # slowest rank's step time (max over ranks)
        assert gids == ids            # accepted global frame ids, in frame order
    assert kept > 50
