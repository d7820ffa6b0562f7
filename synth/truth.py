"""Truth bookkeeping of generated frames: which true particles are
reconstructible and whether the filter's outputs contain them.  Evaluation
only (north-star efficiencies: signal-track and signal-event efficiency); it
holds none of the filter's arithmetic and is imported by bench.py and tests.

  reconstructible particle : hits on all four layers (Sec. IV: tracks
                             are triplets on layers 0-2 extended to layer 3)
  signal-track efficiency  : reconstructible mu->eee daughters found as an output
                             track with exactly their four hits
  signal-event efficiency  : frames whose three mu->eee daughters are all
                             reconstructible and that the filter keeps
"""
from __future__ import annotations

import numpy as np

from . import SynthConfig, particles

SIGNAL_KINDS = (1, 2)   # synth_core.h: 1 signal e+, 2 signal e-


def true_hits(d: dict, f: int) -> dict:
    """{particle index: {layer: hit index inside the layer}} of frame f (needs
    generate(..., truth=True))."""
    hp, off = d["hit_particle"], d["offsets"]
    out: dict = {}
    for layer in range(4):
        lo, hi = int(off[4 * f + layer]), int(off[4 * f + layer + 1])
        for g in range(lo, hi):
            if hp[g] >= 0:
                out.setdefault(int(hp[g]), {})[layer] = g - lo
    return out


def signal_efficiency(cfg: SynthConfig, d: dict, frames_out: np.ndarray, tracks_out: np.ndarray,
                      max_tracks: int) -> dict:
    """Efficiencies over the frames of `d` (frame ids d['frame0'] + f) given the
    filter's per-frame records (m3e_frame_out) and frame-ordered tracks."""
    n = int(d["n_frames"])
    f0 = int(d.get("frame0", 0))
    n_sig_frames = n_recon_frames = n_kept_recon = n_vertex_recon = 0
    n_sig_tracks = n_found = 0
    for f in range(n):
        parts = particles(cfg, f0 + f)
        sig = [i for i, p in enumerate(parts) if p["kind"] in SIGNAL_KINDS]
        if not sig:
            continue
        n_sig_frames += 1
        th = true_hits(d, f)
        rec = f_out = frames_out[f]
        first, nt = int(f_out["track_first"]), min(int(f_out["n_tracks"]), max_tracks)
        out_hits = {tuple(int(h) for h in t["hit"]) for t in tracks_out[first:first + nt]} \
            if int(f_out["reason"]) != 1 else set()
        recon = [i for i in sig if len(th.get(i, {})) == 4]
        for i in recon:
            n_sig_tracks += 1
            n_found += tuple(th[i][l] for l in range(4)) in out_hits
        if len(recon) == len(sig) == 3:
            n_recon_frames += 1
            n_kept_recon += int(rec["reason"]) != 0
            n_vertex_recon += int(rec["reason"]) == 4
    return {"signal_frames": n_sig_frames, "signal_tracks_reconstructible": n_sig_tracks,
            "signal_track_eff": round(n_found / n_sig_tracks, 4) if n_sig_tracks else None,
            "signal_frames_reconstructible": n_recon_frames,
            "signal_event_eff": round(n_kept_recon / n_recon_frames, 4) if n_recon_frames else None,
            "signal_event_vertex_eff": round(n_vertex_recon / n_recon_frames, 4) if n_recon_frames else None}
