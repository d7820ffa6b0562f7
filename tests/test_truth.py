"""The truth bookkeeping behind the north-star efficiencies (synth/truth.py),
checked on the CPU with the ORACLE's outputs standing in for the filter's: a
frame's reconstructible signal tracks are found iff the oracle kept a track with
their four true hits; the counts are exact by construction."""
import numpy as np

import oracle
import synth
from synth.truth import signal_efficiency, true_hits
from paper_2206_11535_b200.m3e import FRAME_DTYPE, TRACK_DTYPE, load_config


def _oracle_outputs(P, d, n):
    fr = oracle.Frames(d)
    frames = np.zeros(n, FRAME_DTYPE)
    tracks = []
    for f in range(n):
        res, trk = oracle.process_frame(P, fr, f)
        frames["reason"][f] = res.reason
        frames["n_tracks"][f] = res.n_tracks
        frames["track_first"][f] = len(tracks)
        for t in trk[:P.max_tracks]:
            r = np.zeros(1, TRACK_DTYPE)[0]
            r["frame"] = f
            r["hit"] = [t.hit[0], t.hit[1], t.hit[2], t.hit[3]]
            tracks.append(r)
    return frames, np.array(tracks, TRACK_DTYPE)


def test_true_hits_are_one_per_layer():
    d = synth.generate(synth.preset("signal_only", seed=41), 20, truth=True)
    for f in range(20):
        off = d["offsets"].astype(np.int64)
        for pid, lay in true_hits(d, f).items():
            for layer, i in lay.items():
                assert 0 <= i < off[4 * f + layer + 1] - off[4 * f + layer]


def test_signal_efficiency_with_oracle_outputs():
    cfg = load_config()
    P = oracle.make_params(cfg)
    sc = synth.preset("signal_only", seed=42)
    n = 150
    d = synth.generate(sc, n, truth=True)
    frames, tracks = _oracle_outputs(P, d, n)
    e = signal_efficiency(sc, d, frames, tracks, P.max_tracks)
    assert e["signal_frames"] == n
    assert e["signal_tracks_reconstructible"] > n
    assert e["signal_track_eff"] >= 0.9
    assert e["signal_event_eff"] >= 0.7
    # dropping every output track makes every signal track lost
    none = signal_efficiency(sc, d, frames, tracks[:0], P.max_tracks)
    assert none["signal_track_eff"] == 0.0
