#!/usr/bin/env python3
"""BASELINE.json configs[2]: 1e6 frames at 1e8 mu/s with mu->eee injected in 1%
of frames — track and vertex efficiency of the CUDA path vs the oracle on the
same generated frames (Sec. VI-A).

The CUDA path (m3e_filter) runs on all frames; the oracle (oracle/, fp64 C) runs
on all frames too (host threads on contiguous slices: kept decisions, reduction
factor) and, frame by frame, on the signal frames (their track lists, for the
signal-track efficiency).  Both are scored with the same truth bookkeeping
(synth/truth.py).

  python tools/configs2_efficiency.py [--frames N] [--json out.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from synth.truth import signal_efficiency  # noqa: E402

SEED = 20220624   # differs from the bench / tuning seeds


def oracle_outputs(P, d, n, threads):
    """frame records and frame-ordered tracks in the C-ABI layouts, from the
    oracle: every frame's reason (process_frames, threaded), the signal frames'
    track lists (process_frame)"""
    from paper_2206_11535_b200.m3e import FRAME_DTYPE, TRACK_DTYPE
    fr = oracle.Frames(d)
    cuts = [n * i // threads for i in range(threads + 1)]
    parts = [None] * threads

    def run(i):
        parts[i] = oracle.results_to_numpy(oracle.process_frames(P, fr, first=cuts[i], count=cuts[i + 1] - cuts[i]))

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(threads)))
    reason = np.concatenate([p["reason"] for p in parts])
    n_tracks = np.concatenate([p["n_tracks"] for p in parts])
    frames = np.zeros(n, FRAME_DTYPE)
    frames["reason"] = reason
    frames["n_tracks"] = n_tracks
    sc = synth.preset("phase1_sig", seed=SEED)
    tracks = []
    for f in range(n):
        frames["track_first"][f] = len(tracks)
        if reason[f] == oracle.REASON_TRIPLET_OVERFLOW or n_tracks[f] == 0:
            continue
        if not any(p["kind"] in (1, 2) for p in synth.particles(sc, f)):
            continue   # only signal frames' tracks are scored
        _, otr = oracle.process_frame(P, fr, f)
        for t in otr:
            r = np.zeros(1, TRACK_DTYPE)[0]
            r["frame"], r["hit"] = f, t.hit
            tracks.append(r)
        frames["n_tracks"][f] = len(otr)
    return frames, np.array(tracks, TRACK_DTYPE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=1_000_000)
    ap.add_argument("--json")
    a = ap.parse_args()
    import torch
    from paper_2206_11535_b200 import m3e
    cfg = m3e.load_config()
    n = a.frames
    sc = synth.preset("phase1_sig", seed=SEED)
    d = synth.generate(sc, n, truth=True)
    # CUDA path
    ctx = m3e.Context(0)
    res = m3e.run_filter(ctx, m3e.make_params(cfg), m3e.DeviceFrames(d))
    torch.cuda.synchronize()
    sm = res.summary_np()
    g_frames = res.frames_np(n)
    g_tracks = res.tracks_np(int(sm["track_slots"]))
    g_eff = signal_efficiency(sc, d, g_frames, g_tracks, cfg["max_tracks"])
    g_kept = int(np.count_nonzero(g_frames["reason"]))
    ctx.close()
    # oracle
    threads = len(os.sched_getaffinity(0))
    t = time.time()
    o_frames, o_tracks = oracle_outputs(oracle.make_params(cfg), d, n, threads)
    t_oracle = time.time() - t
    o_eff = signal_efficiency(sc, d, o_frames, o_tracks, cfg["max_tracks"])
    o_kept = int(np.count_nonzero(o_frames["reason"]))
    same = int(np.count_nonzero(g_frames["reason"] == o_frames["reason"]))
    out = {"config": "BASELINE configs[2]: %d frames of phase-I data (1e8 mu/s), mu->eee in 1%% of frames, seed %d"
                     % (n, SEED),
           "cuda": dict(g_eff, kept=g_kept, reduction_factor=round(n / g_kept, 2)),
           "oracle": dict(o_eff, kept=o_kept, reduction_factor=round(n / o_kept, 2)),
           "frames_with_equal_decision": same, "oracle_seconds": round(t_oracle, 1), "oracle_threads": threads}
    print(json.dumps(out, indent=1))
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(out, fh, indent=1)
    return out


if __name__ == "__main__":
    main()
