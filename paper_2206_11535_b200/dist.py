"""Multi-GPU host logic: one process per GPU, frames sharded across ranks.

Frames are independent (Sec. V: "each computer working independently on
their individual batch of consecutive frames"), so the data path has no
collective at all; the only communication is the final reduction of the run
counters and of the accepted-frame indices (north_star).  Works with NCCL (GPU
tensors) and gloo (CPU tensors, used by the tests).
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist

COUNTER_NAMES = ["frames", "hits", "kept", "tracks", "kept_hits", "none", "triplet_overflow",
                 "track_overflow", "comb_overflow", "vertex_found", "invalid"]


def shard(total_frames: int, rank: int, world: int, weak: bool = True) -> Tuple[int, int]:
    """(first frame id, frame count) of this rank.  weak: every rank filters its
    own `total_frames` (distinct ids); strong: `total_frames` split evenly."""
    if weak:
        return rank * total_frames, total_frames
    lo = total_frames * rank // world
    hi = total_frames * (rank + 1) // world
    return lo, hi - lo


def reduce_counters(counters: torch.Tensor, step_seconds: float, group=None) -> Tuple[torch.Tensor, float]:
    """Sum the per-rank counters and take the slowest rank's step time (the
    multi-GPU time is the max over ranks)."""
    c = counters.clone()
    t = torch.tensor([step_seconds], dtype=torch.float64, device=c.device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return c, float(t.item())


def gather_kept(kept_frames: torch.Tensor, frame0: int, group=None) -> torch.Tensor:
    """All accepted global frame ids, in rank order (each rank's list is already in
    frame order).  Variable-length all_gather via padding to the longest list."""
    ids = kept_frames.to(torch.int64) + frame0
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return ids
    world = dist.get_world_size(group)
    n = torch.tensor([ids.numel()], dtype=torch.int64, device=ids.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    m = int(max(int(v.item()) for v in ns))
    pad = torch.full((m,), -1, dtype=torch.int64, device=ids.device)
    pad[:ids.numel()] = ids
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:int(k.item())] for o, k in zip(outs, ns)])
