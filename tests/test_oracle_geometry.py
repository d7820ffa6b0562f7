"""Pins of the oracle's geometric primitives (Sec. IV-A Eq. 2-5,
Sec. IV-C circles, Fig. 5 arc relation, Fig. 3 target) against closed forms,
constructions and invariants."""
import math

import numpy as np
import pytest

import oracle
from helix import Helix, track_hits, kink


def test_tan_lambda_closed_forms():
    # 45 degree line, flat track (SPEC examples of Eq. 2)
    assert oracle.tan_lambda(0.0, 10.0, 20.0, 30.0) == pytest.approx(1.0, abs=1e-15)
    assert oracle.tan_lambda(5.0, 5.0, 20.0, 30.0) == 0.0
    # antisymmetric under exchanging the hits' z
    assert oracle.tan_lambda(3.0, -4.0, 23.3, 29.8) == -oracle.tan_lambda(-4.0, 3.0, 23.3, 29.8)


def test_cos_phi_closed_forms():
    assert oracle.cos_phi(1, 0, 0, 1, 1, 1) == 0.0
    assert oracle.cos_phi(2, 0, 5, 0, 2, 5) == 1.0
    assert oracle.cos_phi(1, 1, -1, 2, math.sqrt(2), math.sqrt(5)) == pytest.approx(1 / math.sqrt(10), rel=1e-14)
    # back to back
    assert oracle.cos_phi(3, 4, -3, -4, 5, 5) == pytest.approx(-1.0, rel=1e-15)


@pytest.mark.parametrize("R,cx,cy,angles", [(50.0, 0.0, 0.0, (0, 90, 180)),
                                            (81.4, 3.0, -7.0, (10, 40, 95)),
                                            (250.0, -20.0, 31.0, (3, 5, 9))])
def test_circle_radius_recovers_constructed_circle(R, cx, cy, angles):
    pts = [(cx + R * math.cos(math.radians(a)), cy + R * math.sin(math.radians(a)), 0.0) for a in angles]
    r_ccw = oracle.circle_radius(*pts)                      # counter-clockwise order
    r_cw = oracle.circle_radius(*pts[::-1])                 # clockwise order
    assert abs(r_ccw) == pytest.approx(R, rel=1e-9)
    # sign convention (reading R5): clockwise > 0, i.e. a positron in B along +z
    assert r_cw > 0 > r_ccw
    assert r_cw == pytest.approx(-r_ccw, rel=1e-12)


def test_circle_radius_collinear_is_infinite():
    assert math.isinf(oracle.circle_radius((0, 0, 0), (1, 0, 0), (2, 0, 0)))


def test_circle_radius_rotation_translation_invariant():
    rng = np.random.default_rng(1)
    for _ in range(50):
        p = rng.normal(size=(3, 2)) * 40
        r0 = oracle.circle_radius(*[(a, b, 0.0) for a, b in p])
        th = rng.uniform(0, 2 * math.pi)
        Rm = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
        q = p @ Rm.T + rng.normal(size=2) * 30
        r1 = oracle.circle_radius(*[(a, b, 5.0) for a, b in q])
        assert r1 == pytest.approx(r0, rel=1e-9)


def test_positron_track_has_positive_radius():
    """A positive charge in B along +z turns clockwise: Eq. 5 > 0 (reading R5)."""
    hits = track_hits((1.0, 2.0, 0.0), (20.0, 5.0, 3.0), +1, [23.3, 29.8, 73.9])
    hits_m = track_hits((1.0, 2.0, 0.0), (20.0, 5.0, 3.0), -1, [23.3, 29.8, 73.9])
    assert oracle.circle_radius(*hits) > 0
    assert oracle.circle_radius(*hits_m) < 0
    h = Helix((1.0, 2.0, 0.0), (20.0, 5.0, 3.0), +1)
    assert oracle.circle_radius(*hits) == pytest.approx(h.Rt, rel=1e-9)


@pytest.mark.parametrize("p,theta_deg", [(15.0, 40.0), (30.0, 75.0), (52.0, 110.0), (20.0, 150.0)])
def test_arc_relation_recovers_helix_bending(p, theta_deg):
    """Fig. 5 arc relation: for two points of a helix of 3D radius R the oracle's
    root Phi(d, z, 1/R) equals the transverse bending angle of the helix."""
    th = math.radians(theta_deg)
    mom = p * np.array([math.sin(th), 0.0, math.cos(th)])
    h = Helix((0.0, 0.0, 0.0), mom, +1)
    for t in (0.05, 0.4, 1.2, 2.5):
        a, b = h.at(0.0), h.at(t)
        d, z = math.hypot(*(b - a)[:2]), b[2] - a[2]
        assert oracle.arc_phi(d, z, 1.0 / h.R3) == pytest.approx(t, rel=1e-9, abs=1e-12)


def test_arc_relation_no_short_arc():
    # radius smaller than half the chord: no arc
    assert math.isnan(oracle.arc_phi(10.0, 0.0, 1.0 / 4.9))
    assert not math.isnan(oracle.arc_phi(10.0, 0.0, 1.0 / 5.1))


@pytest.mark.parametrize("q", [+1, -1])
@pytest.mark.parametrize("dtheta,dphi", [(0.0, 0.0), (0.01, 0.0), (0.0, 0.013), (-0.02, 0.007),
                                         (0.004, -0.03)])
def test_scattering_angles_recover_constructed_kink(q, dtheta, dphi):
    """Fig. 5: a track of fixed |p| kinked at the middle hit by (dtheta, dphi)
    has Theta_MS = dtheta and Phi_MS = dphi at its true 3D curvature."""
    v = (4.0, -3.0, 10.0)
    p = np.array([18.0, 11.0, 14.0])
    hits = track_hits(v, p, q, [23.3, 29.8, 73.9], kinks=[None, (dtheta, dphi)])
    k = 0.299792458 / np.linalg.norm(p)
    phi_ms, theta_ms = oracle.scattering_angles(*hits, q, k)
    assert phi_ms == pytest.approx(dphi, abs=1e-9)
    assert theta_ms == pytest.approx(dtheta, abs=1e-9)


def test_circle_intersections_closed_forms():
    pts, _ = oracle.circle_intersections((0, 0), 5.0, (8, 0), 5.0)
    assert sorted((round(x, 12), round(y, 12)) for x, y in pts) == [(4.0, -3.0), (4.0, 3.0)]
    assert oracle.circle_intersections((0, 0), 1.0, (10, 0), 1.0)[0] == []
    assert oracle.circle_intersections((0, 0), 1.0, (0, 0), 1.0)[0] == []     # concentric
    assert oracle.circle_intersections((0, 0), 5.0, (1, 0), 1.0)[0] == []     # nested
    pts, marg = oracle.circle_intersections((0, 0), 2.0, (4, 0), 2.0)        # tangent
    assert len(pts) == 2 and pts[0] == pytest.approx(pts[1], abs=1e-12) and marg


def test_circle_intersections_lie_on_both_circles():
    rng = np.random.default_rng(3)
    for _ in range(200):
        c1, c2 = rng.normal(size=2) * 30, rng.normal(size=2) * 30
        r1, r2 = rng.uniform(10, 80, size=2)
        pts, _ = oracle.circle_intersections(c1, r1, c2, r2)
        for x, y in pts:
            assert math.hypot(x - c1[0], y - c1[1]) == pytest.approx(r1, abs=1e-9)
            assert math.hypot(x - c2[0], y - c2[1]) == pytest.approx(r2, abs=1e-9)


def test_target_distance(P):
    # points on the double cone surface rho = 19 (1 - |z|/50)
    for z in (-50, -30, 0, 12.5, 49):
        rho = 19.0 * (1 - abs(z) / 50.0)
        for ph in (0.0, 1.0, 4.0):
            assert oracle.target_distance(P, rho * math.cos(ph), rho * math.sin(ph), z) == pytest.approx(0, abs=1e-12)
    # the origin: distance to the line through (0,-50) and (19,0) = 950 / sqrt(19^2 + 50^2)
    assert oracle.target_distance(P, 0, 0, 0) == pytest.approx(950 / math.hypot(19, 50), rel=1e-12)
    # beyond the tip: distance to the tip point
    assert oracle.target_distance(P, 0, 0, 60) == pytest.approx(10.0, rel=1e-12)
    # radially outside the rim
    assert oracle.target_distance(P, 0, 25, 0) == pytest.approx(6.0, rel=1e-12)


def test_highland_scaling():
    # sigma_MS ~ 1/p and ~ sqrt(x/X0)(1 + 0.038 ln x/X0) (PDG); doubling p halves it
    assert oracle.highland(20.0, 1e-3) == pytest.approx(2 * oracle.highland(40.0, 1e-3), rel=1e-14)
    # PDG: at x/X0 = 1 the log term vanishes: 13.6 MeV / p
    assert oracle.highland(13.6, 1.0) == pytest.approx(1.0, rel=1e-14)
