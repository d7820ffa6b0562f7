"""Test-side forward model of charged helices (independent of oracle/ and of the
CUDA path): exact helix points, cylinder crossings by numerical root finding,
and hand-built multiple-scattering kinks.  Used to pin the oracle."""
from __future__ import annotations

import math

import numpy as np
from scipy.optimize import brentq

PT_CONV = 0.299792458  # MeV/c per (T mm)


class Helix:
    """Helix of charge q (+1 turns clockwise seen from +z in B along +z)."""

    def __init__(self, v, p, q, b=1.0):
        self.v = np.asarray(v, dtype=float)
        p = np.asarray(p, dtype=float)
        self.q = q
        self.pt = math.hypot(p[0], p[1])
        self.pabs = float(np.linalg.norm(p))
        self.Rt = self.pt / (PT_CONV * b)
        self.R3 = self.pabs / (PT_CONV * b)
        self.psi0 = math.atan2(p[1], p[0])
        self.cot = p[2] / self.pt
        self.c = self.v[:2] + q * self.Rt * np.array([math.sin(self.psi0), -math.cos(self.psi0)])
        self.phi0 = math.atan2(self.v[1] - self.c[1], self.v[0] - self.c[0])

    def at(self, t):
        """position after turning by t (>= 0) radians"""
        ph = self.phi0 - self.q * t
        return np.array([self.c[0] + self.Rt * math.cos(ph), self.c[1] + self.Rt * math.sin(ph),
                         self.v[2] + self.Rt * self.cot * t])

    def direction(self, t):
        """unit momentum direction after turning by t"""
        psi = self.psi0 - self.q * t
        st = 1.0 / math.sqrt(1.0 + self.cot ** 2)
        return np.array([st * math.cos(psi), st * math.sin(psi), st * self.cot])

    def cross(self, rho, t_from=0.0):
        """first turning angle > t_from where the helix reaches transverse radius rho"""
        f = lambda t: math.hypot(*self.at(t)[:2]) - rho
        ts = np.linspace(t_from + 1e-9, t_from + math.pi, 4001)
        vals = [f(t) for t in ts]
        for i in range(len(ts) - 1):
            if vals[i] == 0:
                return ts[i]
            if vals[i] * vals[i + 1] < 0:
                return brentq(f, ts[i], ts[i + 1], xtol=1e-15, rtol=1e-15, maxiter=200)
        return None


def kink(direction, dtheta, dphi):
    """rotate a unit direction: polar angle += dtheta, azimuth += dphi (exact)."""
    d = np.asarray(direction, dtype=float)
    theta = math.acos(d[2] / np.linalg.norm(d)) + dtheta
    phi = math.atan2(d[1], d[0]) + dphi
    return np.array([math.sin(theta) * math.cos(phi), math.sin(theta) * math.sin(phi), math.cos(theta)])


def track_hits(v, p, q, radii, kinks=None, b=1.0):
    """Hits of a (possibly kinked) track on the given cylinder radii.
    kinks[i] = (dtheta, dphi) applied after the crossing of radii[i]."""
    hits = []
    pos, mom = np.asarray(v, float), np.asarray(p, float)
    pabs = float(np.linalg.norm(mom))
    for i, rho in enumerate(radii):
        h = Helix(pos, mom, q, b)
        t = h.cross(rho)
        if t is None:
            return None
        pos = h.at(t)
        hits.append(pos.copy())
        mom = pabs * h.direction(t)
        if kinks and i < len(kinks) and kinks[i] is not None:
            mom = pabs * kink(mom, *kinks[i])
    return hits
