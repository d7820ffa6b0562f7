"""Pins of the oracle's triplet fit (Sec. IV-B, Eq. 6-8, Alg. 3)."""
import math

import numpy as np
import pytest

import oracle
import synth
from helix import Helix, track_hits

LAYERS = [23.3, 29.8, 73.9, 86.3]


def _frame_from_hits(hits_by_layer):
    """build a one-frame Frames object from per-layer hit lists"""
    xs, ys, zs, off = [], [], [], [0]
    for layer in hits_by_layer:
        for h in layer:
            xs.append(h[0]); ys.append(h[1]); zs.append(h[2])
        off.append(len(xs))
    return oracle.Frames({"x": np.array(xs, np.float32), "y": np.array(ys, np.float32),
                          "z": np.array(zs, np.float32), "offsets": np.array(off, np.uint32)})


@pytest.mark.parametrize("q", [+1, -1])
@pytest.mark.parametrize("p,theta_deg,phi_deg", [(15.0, 70.0, 10.0), (30.0, 100.0, 200.0),
                                                 (50.0, 55.0, 300.0), (22.0, 125.0, 95.0)])
def test_noiseless_helix_is_fixed_point(P, q, p, theta_deg, phi_deg):
    """No scattering: the circle solution is the helix, Theta_MS = 0, so the fit
    returns the true 3D curvature with chi2 = 0 (Sec. IV-B, Eq. 6)."""
    th, ph = math.radians(theta_deg), math.radians(phi_deg)
    mom = p * np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
    hits = track_hits((3.0, -5.0, 7.0), mom, q, LAYERS[:3])
    t = oracle.fit_triplet(P, *hits)
    assert t.ok and t.q == q
    assert t.kappa == pytest.approx(q * 0.299792458 / p, rel=1e-9)
    assert t.chi2 < 1e-12
    assert t.k_c[0] == pytest.approx(t.k_c[1], rel=1e-9)
    assert t.theta_c[0] == pytest.approx(th, abs=1e-9)


@pytest.mark.parametrize("q", [+1, -1])
@pytest.mark.parametrize("seed", range(12))
def test_linearised_minimum_matches_brute_force(P, q, seed):
    """The closed-form minimiser of the linearised chi2 agrees with a brute-force
    grid minimisation of the EXACT chi2(k) (exact arc relation, same weights)
    to 1e-3 relative (the linearisation error is second order)."""
    rng = np.random.default_rng(seed)
    p = rng.uniform(15, 50)
    th = rng.uniform(0.9, 2.2)
    ph = rng.uniform(0, 2 * math.pi)
    mom = p * np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
    sig = 0.01 * 20 / p
    hits = track_hits(rng.normal(size=3) * 5, mom, q, LAYERS[:3],
                      kinks=[None, (rng.normal() * sig, rng.normal() * sig)])
    t = oracle.fit_triplet(P, *hits)
    assert t.ok

    def chi2_exact(k):
        a = oracle.scattering_angles(*hits, t.q, k)
        if a is None:
            return np.inf
        return a[0] ** 2 * t.w_phi + a[1] ** 2 * t.w_theta

    kc = 0.5 * (t.k_c[0] + t.k_c[1])
    grid = np.linspace(0.8 * kc, 1.2 * kc, 4001)
    vals = np.array([chi2_exact(k) for k in grid])
    i = int(np.argmin(vals))
    lo, hi = grid[max(i - 1, 0)], grid[min(i + 1, len(grid) - 1)]
    fine = np.linspace(lo, hi, 2001)
    kbest = fine[int(np.argmin([chi2_exact(k) for k in fine]))]
    assert t.k_hat == pytest.approx(kbest, rel=1e-3)
    # and the linearised chi2 at the minimum approximates the exact one
    assert t.chi2 == pytest.approx(chi2_exact(kbest), rel=2e-2, abs=1e-3)


def test_weighted_mean_eq8_and_global_chi2(P):
    """Eq. 8: kappa-bar lies between the triplet curvatures; with MS the global
    chi2 (Eq. 7) at kappa-bar is the sum of the two linearised chi2_t."""
    sc = synth.SynthConfig(fixed_signal=0, fixed_michel=6, noise_per_layer=0.0, seed=5)
    d = synth.generate(sc, 60, truth=True)
    fr = oracle.Frames(d)
    n = 0
    for f in range(fr.n):
        cands, _ = oracle.select(P, fr, f)
        for c in cands:
            t = oracle.fit_candidate(P, fr, f, c)
            if t.status not in (oracle.FIT_OK, oracle.FIT_CHI2):
                continue
            k1, k2 = t.t1.kappa, t.t2.kappa
            assert min(k1, k2) - 1e-15 <= t.kappa <= max(k1, k2) + 1e-15
            w1, w2 = 1 / t.t1.var_kappa, 1 / t.t2.var_kappa
            assert t.kappa == pytest.approx((k1 * w1 + k2 * w2) / (w1 + w2), rel=1e-12)
            n += 1
    assert n > 100


@pytest.mark.parametrize("q", [+1, -1])
@pytest.mark.parametrize("p,theta_deg", [(20.0, 80.0), (45.0, 60.0), (30.0, 120.0)])
def test_extrapolation_noiseless(P, q, p, theta_deg):
    """Sec. IV-B 'the hit position in the fourth layer is estimated': for an
    unscattered helix the prediction is the true layer-3 crossing."""
    th = math.radians(theta_deg)
    mom = p * np.array([math.sin(th) * 0.6, math.sin(th) * 0.8, math.cos(th)])
    hits = track_hits((2.0, 1.0, -4.0), mom, q, LAYERS)
    pred = oracle.extrapolate(P, hits[1], hits[2], q, 0.299792458 / p)
    assert np.allclose(pred, hits[3], atol=1e-8)


def test_full_track_noiseless(P):
    """Alg. 3 on an unscattered 4-hit track: accepted, kappa exact, chi2 = 0,
    transverse circle = helix circle."""
    for q in (+1, -1):
        mom = np.array([-12.0, 21.0, 9.0])
        v = (5.0, 3.0, -12.0)
        hits = track_hits(v, mom, q, LAYERS)
        fr = _frame_from_hits([[h] for h in hits])
        c = oracle.Candidate(0, 0, 0, 0, oracle.circle_radius(*[fr.hit(0, l, 0) for l in range(3)]))
        t = oracle.fit_candidate(P, fr, 0, c)
        h = Helix(v, mom, q)
        assert t.status == oracle.FIT_OK and t.accepted and t.hit[3] == 0
        assert t.kappa == pytest.approx(q * 0.299792458 / np.linalg.norm(mom), rel=2e-6)  # float32 hits
        assert t.chi2 < 1e-6
        assert t.rt == pytest.approx(h.Rt, rel=2e-6)
        assert (t.cx, t.cy) == pytest.approx(tuple(h.c), abs=2e-3)
        assert t.cos_theta01 == pytest.approx(mom[2] / np.linalg.norm(mom), abs=1e-5)


@pytest.mark.parametrize("q", [+1, -1])
@pytest.mark.parametrize("mom", [(-12.0, 21.0, 9.0), (30.0, 4.0, -20.0), (3.0, -18.0, 1.0)])
def test_track_params_recover_helix_circle(P, q, mom):
    """Reading R11 at the TRUE curvature of a helix (test-side model, not the
    oracle): the circle through h0, h1 of radius sin(theta)/|kappa| is the helix's
    transverse circle, cos(theta01) its p_z / p, p and E the true ones; a curvature
    too small to join h0 and h1 by a short arc has no parameters."""
    mom = np.array(mom)
    v = (2.0, -3.0, 7.0)
    hits = track_hits(v, mom, q, LAYERS)
    h = Helix(v, mom, q)
    kap = q * 0.299792458 / np.linalg.norm(mom)
    t = oracle.track_params(P, hits[0], hits[1], kap)
    assert t is not None and t.q == q
    assert t.rt == pytest.approx(h.Rt, rel=1e-9)
    assert (t.cx, t.cy) == pytest.approx(tuple(h.c), abs=1e-7)
    assert t.cos_theta01 == pytest.approx(mom[2] / np.linalg.norm(mom), abs=1e-9)
    assert t.p == pytest.approx(np.linalg.norm(mom), rel=1e-12)
    assert t.energy == pytest.approx(math.hypot(np.linalg.norm(mom), 0.51099895), rel=1e-12)
    d01 = math.hypot(hits[1][0] - hits[0][0], hits[1][1] - hits[0][1])
    assert oracle.track_params(P, hits[0], hits[1], q * 2.5 / d01) is None   # 1/k^2 < d^2/4


def test_closest_layer3_hit_chosen(P):
    """Alg. 3 find_closest_layer3_hit: the true hit is picked among decoys."""
    mom = np.array([15.0, 20.0, -6.0])
    hits = track_hits((0.0, 4.0, 3.0), mom, +1, LAYERS)
    ang = math.atan2(hits[3][1], hits[3][0])
    decoys = [(86.3 * math.cos(ang + d), 86.3 * math.sin(ang + d), hits[3][2] + dz)
              for d, dz in [(0.05, 0.0), (-0.03, 1.0), (0.0, 4.0), (1.0, 0.0)]]
    layer3 = decoys[:2] + [tuple(hits[3])] + decoys[2:]
    fr = _frame_from_hits([[hits[0]], [hits[1]], [hits[2]], layer3])
    c = oracle.Candidate(0, 0, 0, 0, oracle.circle_radius(*[fr.hit(0, l, 0) for l in range(3)]))
    t = oracle.fit_candidate(P, fr, 0, c)
    assert t.hit[3] == 2 and t.accepted


def test_mirror_symmetries(P):
    """y -> -y mirrors the sense of rotation: kappa flips sign, |kappa| and chi2
    unchanged.  z -> -z leaves kappa and chi2 unchanged."""
    sc = synth.SynthConfig(fixed_signal=0, fixed_michel=5, noise_per_layer=0.0, seed=9)
    d = synth.generate(sc, 40)
    for mode in ("y", "z"):
        dm = dict(d)
        dm[mode] = -d[mode]
        fr, frm = oracle.Frames(d), oracle.Frames(dm)
        n = 0
        for f in range(fr.n):
            cands, _ = oracle.select(P, fr, f)
            candm, _ = oracle.select(P, frm, f)
            assert [(c.i0, c.i1, c.i2) for c in cands] == [(c.i0, c.i1, c.i2) for c in candm]
            for c, cm in zip(cands, candm):
                t, tm = oracle.fit_candidate(P, fr, f, c), oracle.fit_candidate(P, frm, f, cm)
                assert t.status == tm.status
                if t.status == oracle.FIT_OK:
                    sgn = -1 if mode == "y" else 1
                    assert tm.kappa == pytest.approx(sgn * t.kappa, rel=1e-9)
                    assert tm.chi2 == pytest.approx(t.chi2, rel=1e-6, abs=1e-9)
                    n += 1
        assert n > 50


@pytest.mark.slow
def test_chi2_follows_three_dof_when_model_matches(P):
    """Statistical pin of Eq. 6-8 and of the sigma model (readings R6-R8): with
    Highland scattering at normal incidence (the fit's model) and no pixel
    smearing, the global chi2 of true tracks has mean = 4 measurements - 1
    parameter = 3, and kappa-bar is unbiased."""
    sc = synth.SynthConfig(fixed_signal=0, fixed_michel=6, noise_per_layer=0.0, sigma_pixel=0.0,
                           normal_incidence=True, seed=21)
    n = 700
    d = synth.generate(sc, n, truth=True)
    fr = oracle.Frames(d)
    hp, off = d["hit_particle"], d["offsets"].astype(int)
    chis, rel = [], []
    for f in range(n):
        parts = synth.particles(sc, f)
        for pi, p in enumerate(parts):
            if p["layer_mask"] != 15:
                continue
            idx = [int(np.nonzero(hp[off[4 * f + l]:off[4 * f + l + 1]] == pi)[0][0]) for l in range(4)]
            c = oracle.Candidate(idx[0], idx[1], idx[2], 0,
                                 oracle.circle_radius(*[fr.hit(f, l, idx[l]) for l in range(3)]))
            t = oracle.fit_candidate(P, fr, f, c)
            if t.status in (oracle.FIT_OK, oracle.FIT_CHI2) and t.hit[3] == idx[3]:
                chis.append(t.chi2)
                rel.append(t.kappa / (0.299792458 / np.linalg.norm(p["p"])) - 1)
    chis, rel = np.array(chis), np.array(rel)
    assert len(chis) > 2500
    assert np.mean(chis) == pytest.approx(3.0, abs=0.2)
    assert abs(np.mean(rel)) < 0.003
