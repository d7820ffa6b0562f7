"""Pins of the oracle's vertex stage (Sec. IV-C, Eq. 9-12, Alg. 4)."""
import math

import numpy as np
import pytest

import oracle
import synth
from helix import Helix, track_hits

LAYERS = [23.3, 29.8, 73.9, 86.3]
M_MU = 105.6583755


def _vtrack_from_helix(v, p, q):
    """vertex-stage track built directly from a known helix (no fit)."""
    hits = track_hits(v, p, q, LAYERS[:1])
    h = Helix(v, p, q)
    pabs = np.linalg.norm(p)
    return oracle.VTrack(q * 0.299792458 / pabs, p[2] / pabs, h.c[0], h.c[1], tuple(hits[0]))


def _signal_momenta(rng):
    """three momenta with sum 0 and total energy m_mu (Eq. 1), built by hand."""
    me = 0.51099895
    while True:
        E1, E2 = rng.uniform(15, 52, size=2)
        E3 = M_MU - E1 - E2
        if E3 < 12:
            continue
        p1, p2, p3 = (math.sqrt(E * E - me * me) for E in (E1, E2, E3))
        c = (p3 * p3 - p1 * p1 - p2 * p2) / (2 * p1 * p2)
        if abs(c) > 1:
            continue
        a = np.array([0, 0, p1])
        b = np.array([p2 * math.sqrt(1 - c * c), 0, p2 * c])
        m = np.stack([a, b, -a - b])
        # rotate so that all three are reasonably transverse
        th = rng.uniform(0, 2 * math.pi)
        R = np.array([[1, 0, 0], [0, math.cos(th), -math.sin(th)], [0, math.sin(th), math.cos(th)]])
        m = m @ np.array([[0, 0, 1], [1, 0, 0], [0, 1, 0]]).T @ R.T
        if min(np.hypot(m[:, 0], m[:, 1])) < 12:
            continue
        return m


@pytest.mark.parametrize("seed", range(8))
def test_exact_signal_vertex_recovered(P, seed):
    """Three exact helices from one vertex with sum p = 0, sum E = m_mu:
    the vertex stage finds the vertex (all circles meet there), chi2 = 0,
    |sum p| = 0 at the points of closest approach, and keeps the frame."""
    rng = np.random.default_rng(seed)
    m = _signal_momenta(rng)
    ph = rng.uniform(0, 2 * math.pi)
    zv = rng.uniform(-40, 40)
    rho = 19 * (1 - abs(zv) / 50)
    v = (rho * math.cos(ph), rho * math.sin(ph), zv)
    vt = [_vtrack_from_helix(v, m[0], +1), _vtrack_from_helix(v, m[1], +1), _vtrack_from_helix(v, m[2], -1)]
    res, verts = oracle.vertex_frame(P, vt)
    assert res.n_combs == 1
    assert res.keep and res.reason == oracle.REASON_VERTEX
    vx = res.vertex
    assert (vx.x, vx.y, vx.z) == pytest.approx(v, abs=1e-6)
    assert vx.chi2 < 1e-9
    assert vx.p_total < 1e-6
    assert vx.target_dist < 1e-6


def test_vertex_rotation_invariance(P):
    """Rotating all tracks about the beam axis rotates the vertex and leaves
    chi2, |sum p| and the target distance unchanged."""
    rng = np.random.default_rng(11)
    m = _signal_momenta(rng)
    v = (8.0, -6.0, 10.0)
    kicks = rng.normal(size=(3, 3)) * 0.4
    base = [(m[0] + kicks[0], +1), (m[1] + kicks[1], +1), (m[2] + kicks[2], -1)]
    vt = [_vtrack_from_helix(v, p, q) for p, q in base]
    res, verts = oracle.vertex_frame(P, vt)
    assert verts
    a = 0.7
    Rm = np.array([[math.cos(a), -math.sin(a), 0], [math.sin(a), math.cos(a), 0], [0, 0, 1]])
    vr = tuple(Rm @ np.array(v))
    vt2 = [_vtrack_from_helix(vr, Rm @ p, q) for p, q in base]
    res2, verts2 = oracle.vertex_frame(P, vt2)
    assert len(verts2) == len(verts)
    for u, w in zip(verts, verts2):
        assert w.chi2 == pytest.approx(u.chi2, rel=1e-6, abs=1e-9)
        assert w.p_total == pytest.approx(u.p_total, rel=1e-6)
        assert w.target_dist == pytest.approx(u.target_dist, rel=1e-6, abs=1e-9)
        assert np.allclose(Rm @ np.array([u.x, u.y, u.z]), [w.x, w.y, w.z], atol=1e-6)


def test_energy_precheck_and_charges(P, cfg):
    """Alg. 4 phase 1: only (e+, e+, e-) triples inside the energy window count."""
    rng = np.random.default_rng(2)
    m = _signal_momenta(rng)
    v = (5.0, 5.0, 0.0)
    vt = [_vtrack_from_helix(v, m[0], +1), _vtrack_from_helix(v, m[1], +1), _vtrack_from_helix(v, m[2], -1)]
    # all positive: no triple
    allpos = [_vtrack_from_helix(v, m[i], +1) for i in range(3)]
    res, _ = oracle.vertex_frame(P, allpos)
    assert res.n_combs == 0 and not res.keep
    # scale momenta up by 1.5: energy sum far outside any window
    big = [_vtrack_from_helix(v, 1.5 * m[0], +1), _vtrack_from_helix(v, 1.5 * m[1], +1),
           _vtrack_from_helix(v, 1.5 * m[2], -1)]
    res, _ = oracle.vertex_frame(P, big)
    assert res.n_combs == 0 and not res.keep
    res, _ = oracle.vertex_frame(P, vt)
    assert res.n_combs == 1


def test_comb_overflow(P, cfg):
    """Alg. 4: more than max_combs energy-compatible triples -> frame kept."""
    rng = np.random.default_rng(4)
    m = _signal_momenta(rng)
    v = (5.0, 5.0, 0.0)
    n_pos = 18  # 9 x 9 = 81 energy-compatible (m0-like, m1-like) pairs x 1 electron > 64
    tracks = [_vtrack_from_helix(v, m[i % 2] * (1 + 1e-4 * i), +1) for i in range(n_pos)]
    tracks.append(_vtrack_from_helix(v, m[2], -1))
    res, _ = oracle.vertex_frame(P, tracks)
    assert res.n_combs == cfg["max_combs"] + 1
    assert res.keep and res.reason == oracle.REASON_COMB_OVERFLOW


def test_noiseless_generated_signal_frames(P):
    """Generated mu->eee without scattering or smearing: whenever the three
    signal tracks are reconstructed, the frame is kept with the vertex at the
    generated decay point."""
    sc = synth.SynthConfig(fixed_signal=1, fixed_michel=0, noise_per_layer=0.0, ms_on=False,
                           sigma_pixel=0.0, seed=33)
    n = 150
    d = synth.generate(sc, n, truth=True)
    fr = oracle.Frames(d)
    checked = 0
    for f in range(n):
        parts = synth.particles(sc, f)
        if not all(p["layer_mask"] == 15 for p in parts):
            continue
        res, tracks = oracle.process_frame(P, fr, f)
        if res.n_tracks != 3:  # a true triplet outside the tuned cut windows (~1%)
            continue
        assert res.keep and res.reason == oracle.REASON_VERTEX, f
        assert (res.vertex.x, res.vertex.y, res.vertex.z) == pytest.approx(parts[0]["v"], abs=5e-3)
        assert res.vertex.p_total < 0.05
        checked += 1
    assert checked > 30


def _noisy_signal_tracks(seed):
    rng = np.random.default_rng(seed)
    m = _signal_momenta(rng)
    v = (6.0, -4.0, 12.0)
    kicks = rng.normal(size=(3, 3)) * 0.3
    return [_vtrack_from_helix(v, m[0] + kicks[0], +1), _vtrack_from_helix(v, m[1] + kicks[1], +1),
            _vtrack_from_helix(v, m[2] + kicks[2], -1)]


@pytest.mark.parametrize("seed", range(6))
def test_vertex_weights_scale_with_sigma_ms(cfg, seed):
    """Eq. 10 with sigma_pixel = 0: every sigma_i^2 is proportional to sigma_MS^2
    (Highland ~ sqrt(X)(1 + 0.038 ln X)); scaling X changes all weights by the same
    factor, so the vertex (Eq. 9, 11) is unchanged and chi2 (Eq. 12) scales by
    exactly 1 / (sigma ratio)^2 -- a wrong power of s or sigma in Eq. 10/12 fails."""
    vt = _noisy_signal_tracks(seed)
    base = dict(cfg, sigma_pixel=0.0, e_window=1e9, chi2_vertex_max=1e30, target_dist_max=1e9, p_total_max=1e9)
    X1, X2 = 0.00115, 0.0046
    r1, v1 = oracle.vertex_frame(oracle.make_params(dict(base, x_over_x0=X1)), vt)
    r2, v2 = oracle.vertex_frame(oracle.make_params(dict(base, x_over_x0=X2)), vt)
    assert v1 and len(v1) == len(v2)
    ratio = (oracle.highland(30.0, X2) / oracle.highland(30.0, X1)) ** 2
    for a, b in zip(v1, v2):
        assert (b.x, b.y, b.z) == pytest.approx((a.x, a.y, a.z), abs=1e-9)
        assert b.chi2 == pytest.approx(a.chi2 / ratio, rel=1e-9)


@pytest.mark.parametrize("seed", range(6))
def test_vertex_equal_weights_is_centroid(cfg, seed):
    """Eq. 9 with equal weights (sigma_MS -> 0, sigma_pixel dominant) reduces to
    the arithmetic mean: mu_t is the centroid of one choice of pairwise circle
    intersections, and mu_z the mean of the three Eq. 11 z values."""
    vt = _noisy_signal_tracks(seed)
    P = oracle.make_params(dict(cfg, x_over_x0=1e-30, sigma_pixel=1.0, e_window=1e9, chi2_vertex_max=1e30,
                                target_dist_max=1e9, p_total_max=1e9))
    res, verts = oracle.vertex_frame(P, vt)
    assert verts
    circles = []
    for t in vt:
        k = abs(t.kappa)
        rt = math.sqrt(1 - t.cos_theta01 ** 2) / k
        circles.append(((t.cx, t.cy), rt))
    pts = [oracle.circle_intersections(circles[i][0], circles[i][1], circles[j][0], circles[j][1])[0]
           for i, j in ((0, 1), (0, 2), (1, 2))]
    cents = [((a[0] + b[0] + c[0]) / 3, (a[1] + b[1] + c[1]) / 3) for a in pts[0] for b in pts[1] for c in pts[2]]
    v = verts[0]
    assert min(math.hypot(v.x - cx, v.y - cy) for cx, cy in cents) < 1e-9
