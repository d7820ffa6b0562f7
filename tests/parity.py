"""Helpers shared by the GPU parity tests: run the oracle and the CUDA path on
the same generated frames and compare them with the tolerances of
BASELINE.json's north_star:
  * candidate sets, counts and accept/reject decisions bit-exact, except items
    whose cut variable lies within REL_BAND = 1e-5 (relative) of a threshold;
    those are listed and counted;
  * fitted curvatures and angles within 1e-4 relative.
"""
from __future__ import annotations

import math

import numpy as np

import oracle

REL_BAND = 1e-5
REL_KAPPA = 1e-4
# curvature floor of the relative tolerance: every track of a muon decay has
# p <= 52.83 MeV/c (kinematic endpoint), i.e. |kappa| >= 0.299792458 / 52.83 /mm
# in 1 T; those are compared at 1e-4 relative.  Stiffer (unphysical, near-straight
# fake) fits are compared at the absolute 1e-4 * KAPPA_FLOOR, the fp32 rounding
# floor of a curvature measured over ~50 mm chords.
KAPPA_FLOOR = 0.299792458 / 52.83
# fits with chi2_global above this are > 30 sigma inconsistent; the linearised
# model (Eq. 6, R6) is outside its domain there and only the reject decision is
# compared (measured fp32 agreement below it: <= 5e-6 relative on kappa)
CHI2_DOMAIN = 1000.0


def kappa_close(a, b):
    return abs(a - b) <= REL_KAPPA * max(abs(a), abs(b), KAPPA_FLOOR)


def near(v, thr, band=REL_BAND):
    return abs(v - thr) <= band * abs(thr)


def combo_is_marginal(P, fr, f, i0, i1, i2):
    """Does any cut variable of combination (i0,i1,i2) lie within the band of its
    threshold?  Evaluated with the oracle's own primitives (fp64)."""
    R = list(P.layer_r)
    h0, h1, h2 = fr.hit(f, 0, i0), fr.hit(f, 1, i1), fr.hit(f, 2, i2)
    dl = oracle.tan_lambda(h1[2], h2[2], R[1], R[2]) - oracle.tan_lambda(h0[2], h1[2], R[0], R[1])
    c01 = oracle.cos_phi(h0[0], h0[1], h1[0], h1[1], R[0], R[1])
    c12 = oracle.cos_phi(h1[0], h1[1], h2[0], h2[1], R[1], R[2])
    rt = abs(oracle.circle_radius(h0, h1, h2))
    return (near(abs(dl), P.dlambda_max) or near(c01, P.cos_phi01_min) or near(c12, P.cos_phi12_min)
            or near(rt, P.rt_min) or near(rt, P.rt_max))


def unpack(c):
    c = int(c)
    return c & 1023, (c >> 10) & 1023, (c >> 20) & 1023


def rel_close(a, b, rel=REL_KAPPA, abs_=0.0):
    return abs(a - b) <= rel * max(abs(a), abs(b)) + abs_
