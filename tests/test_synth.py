"""Checks of the input generator (synth/) against the physics it claims:
Poisson occupancy, Eq. 1 conservation for signal, Michel spectrum, noiseless
closure on helices, determinism.  (The generator is input synthesis only.)"""
import math

import numpy as np
import pytest

import synth
from helix import Helix

M_MU, M_E = 105.6583755, 0.51099895


def test_poisson_occupancy():
    cfg = synth.preset("phase1_bg", seed=1)
    n = 20000
    decays = [max([p["decay"] for p in synth.particles(cfg, f)], default=-1) + 1 for f in range(n)]
    # Sec. VI: 1e8 mu/s x 64 ns = 6.4 decays per frame
    assert np.mean(decays) == pytest.approx(6.4, abs=0.06)
    assert np.var(decays) == pytest.approx(6.4, rel=0.05)


def test_signal_conservation():
    cfg = synth.preset("signal_only", seed=2)
    for f in range(300):
        ps = synth.particles(cfg, f)
        assert [p["charge"] for p in ps] == [1, 1, -1]
        P = np.array([p["p"] for p in ps])
        E = np.sqrt((P ** 2).sum(1) + M_E ** 2)
        assert np.abs(P.sum(0)).max() < 1e-9            # Eq. 1: sum p = 0
        assert E.sum() == pytest.approx(M_MU, abs=1e-9)  # Eq. 1: sum E = m_mu
        assert len({p["v"] for p in ps}) == 1            # common vertex
        v = ps[0]["v"]
        assert math.hypot(v[0], v[1]) == pytest.approx(19.0 * (1 - abs(v[2]) / 50.0), abs=1e-9)


def test_michel_spectrum():
    cfg = synth.SynthConfig(fixed_michel=1, fixed_signal=0, seed=3)
    pmax = math.sqrt(((M_MU ** 2 + M_E ** 2) / (2 * M_MU)) ** 2 - M_E ** 2)
    x = np.sort([np.linalg.norm(synth.particles(cfg, f)[0]["p"]) / pmax for f in range(20000)])
    assert x.max() <= 1.0
    cdf = x ** 3 * (2 - x)  # integral of 6 x^2 (3 - 2x)/... normalised: x^3 (2 - x)
    ks = np.max(np.abs(cdf - np.arange(1, len(x) + 1) / len(x)))
    assert ks < 0.012


def test_noiseless_hits_on_helix():
    cfg = synth.SynthConfig(fixed_michel=3, fixed_signal=1, noise_per_layer=0.0, ms_on=False,
                            sigma_pixel=0.0, seed=4)
    d = synth.generate(cfg, 50, truth=True)
    off = d["offsets"].astype(int)
    for f in range(50):
        parts = synth.particles(cfg, f)
        for layer in range(4):
            for g in range(off[4 * f + layer], off[4 * f + layer + 1]):
                p = parts[d["hit_particle"][g]]
                h = Helix(p["v"], p["p"], p["charge"])
                hit = np.array([d["x"][g], d["y"][g], d["z"][g]], float)
                # on the cylinder and on the helix (float32 storage)
                assert math.hypot(hit[0], hit[1]) == pytest.approx(cfg.layer_r[layer], abs=2e-5)
                assert math.hypot(hit[0] - h.c[0], hit[1] - h.c[1]) == pytest.approx(h.Rt, abs=1e-4)


def test_layout_and_determinism():
    cfg = synth.preset("phase1_sig", seed=5)
    a = synth.generate(cfg, 1000, threads=1)
    b = synth.generate(cfg, 1000, threads=7)
    for k in ("x", "y", "z", "offsets"):
        assert np.array_equal(a[k], b[k])
    off = a["offsets"]
    assert off[0] == 0 and off[-1] == len(a["x"]) and np.all(np.diff(off.astype(np.int64)) >= 0)
    # frames are independent: a sub-range regenerates the same hits
    c = synth.generate(cfg, 10, frame0=500)
    lo, hi = int(off[4 * 500]), int(off[4 * 510])
    assert np.array_equal(c["x"], a["x"][lo:hi])
    radii = np.hypot(a["x"], a["y"])
    layer = np.zeros(len(a["x"]), int)
    for f in range(1000):
        for l in range(4):
            layer[off[4 * f + l]:off[4 * f + l + 1]] = l
    for l in range(4):
        assert np.allclose(radii[layer == l], cfg.layer_r[l], atol=2e-5)
