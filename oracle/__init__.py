"""ctypes binding of the CPU oracle (m3e_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle_m3e.so")

c_double, c_int, c_int64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64


class Params(ctypes.Structure):
    _fields_ = [("layer_r", c_double * 4), ("b_field", c_double), ("target_r", c_double),
                ("target_half", c_double), ("dlambda_max", c_double), ("cos_phi01_min", c_double),
                ("cos_phi12_min", c_double), ("rt_min", c_double), ("rt_max", c_double),
                ("cuts_max", c_int), ("x_over_x0", c_double), ("chi2_max", c_double),
                ("max_tracks", c_int), ("e_window", c_double), ("xy_margin", c_double),
                ("sigma_pixel", c_double), ("chi2_vertex_max", c_double),
                ("target_dist_max", c_double), ("p_total_max", c_double), ("max_combs", c_int),
                ("rel_band", c_double)]


class Candidate(ctypes.Structure):
    _fields_ = [("i0", c_int), ("i1", c_int), ("i2", c_int), ("marginal", c_int), ("rtc", c_double)]


class TripletFit(ctypes.Structure):
    _fields_ = [("ok", c_int), ("q", c_int), ("rtc", c_double), ("phi_c", c_double * 2),
                ("k_c", c_double * 2), ("theta_c", c_double * 2), ("dphi", c_double * 2),
                ("dtheta", c_double * 2), ("a_phi", c_double), ("b_phi", c_double),
                ("a_theta", c_double), ("b_theta", c_double), ("sigma_ms", c_double),
                ("w_phi", c_double), ("w_theta", c_double), ("k_hat", c_double), ("kappa", c_double),
                ("var_kappa", c_double), ("chi2", c_double)]


class Track(ctypes.Structure):
    _fields_ = [("cand", c_int), ("hit", c_int * 4), ("status", c_int), ("accepted", c_int),
                ("marginal", c_int), ("q", c_int), ("pad", c_int), ("t1", TripletFit),
                ("t2", TripletFit), ("pred", c_double * 3), ("kappa", c_double),
                ("var_kappa", c_double), ("chi2", c_double), ("cos_theta01", c_double),
                ("cx", c_double), ("cy", c_double), ("rt", c_double), ("p", c_double),
                ("energy", c_double)]


class VTrack(ctypes.Structure):
    _fields_ = [("kappa", c_double), ("cos_theta01", c_double), ("cx", c_double), ("cy", c_double),
                ("h0", c_double * 3)]


class Vertex(ctypes.Structure):
    _fields_ = [("a", c_int), ("b", c_int), ("e", c_int), ("pass_", c_int), ("x", c_double),
                ("y", c_double), ("z", c_double), ("chi2", c_double), ("target_dist", c_double),
                ("p_total", c_double)]


class FrameResult(ctypes.Structure):
    _fields_ = [("reason", c_int), ("keep", c_int), ("n_cand", c_int), ("n_cand_marginal", c_int),
                ("funnel", c_int64 * 5), ("n_fit", c_int), ("n_tracks", c_int),
                ("n_fit_marginal", c_int), ("n_pos", c_int), ("n_neg", c_int), ("n_combs", c_int),
                ("n_vertex_marginal", c_int), ("has_vertex", c_int), ("vertex", Vertex)]


FIT_OK, FIT_DEGENERATE1, FIT_NO_REACH, FIT_LAYER3_EMPTY, FIT_DEGENERATE2, FIT_CHI2, FIT_DOMAIN = range(7)
REASON_NONE, REASON_TRIPLET_OVERFLOW, REASON_TRACK_OVERFLOW, REASON_COMB_OVERFLOW, REASON_VERTEX = range(5)

_lib = None
_P = ctypes.POINTER
_vp = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB)
        for i, T in enumerate([Params, Candidate, TripletFit, Track, VTrack, Vertex, FrameResult]):
            assert L.or_sizeof(i) == ctypes.sizeof(T), (T.__name__, L.or_sizeof(i), ctypes.sizeof(T))
        d3 = _P(c_double)
        L.or_tan_lambda.restype = c_double
        L.or_tan_lambda.argtypes = [c_double] * 4
        L.or_cos_phi.restype = c_double
        L.or_cos_phi.argtypes = [c_double] * 6
        L.or_circle_radius.restype = c_double
        L.or_circle_radius.argtypes = [d3, d3, d3]
        L.or_arc_phi.restype = c_double
        L.or_arc_phi.argtypes = [c_double] * 3
        L.or_highland.restype = c_double
        L.or_highland.argtypes = [c_double] * 2
        L.or_target_distance.restype = c_double
        L.or_target_distance.argtypes = [_P(Params), c_double, c_double, c_double]
        L.or_circle_intersections.argtypes = [c_double] * 6 + [d3, c_double, _P(ctypes.c_int)]
        L.or_scattering_angles.argtypes = [d3, d3, d3, ctypes.c_int, c_double, d3, d3]
        L.or_fit_triplet.argtypes = [_P(Params), d3, d3, d3, _P(TripletFit)]
        L.or_extrapolate.argtypes = [_P(Params), d3, d3, ctypes.c_int, c_double, d3]
        L.or_select.argtypes = [_P(Params), _vp, _vp, _vp, _vp, _P(Candidate), ctypes.c_int,
                                _P(FrameResult)]
        L.or_fit_candidate.argtypes = [_P(Params), _vp, _vp, _vp, _vp, _P(Candidate), _P(Track)]
        L.or_track_params.argtypes = [_P(Params), d3, d3, c_double, _P(Track)]
        L.or_vertex_frame.argtypes = [_P(Params), _P(VTrack), ctypes.c_int, _P(FrameResult),
                                      _P(Vertex), ctypes.c_int]
        L.or_process_frame.argtypes = [_P(Params), _vp, _vp, _vp, _vp, _P(FrameResult),
                                       _P(Candidate), _P(Track)]
        L.or_process_frames.restype = c_int64
        L.or_process_frames.argtypes = [_P(Params), _vp, _vp, _vp, _vp, c_int64, _P(FrameResult)]
        _lib = L
    return _lib


def make_params(cfg: dict) -> Params:
    """Build oracle parameters from the shared threshold configuration dict."""
    p = Params()
    for i in range(4):
        p.layer_r[i] = cfg["layer_r"][i]
    for k in ["b_field", "target_r", "target_half", "dlambda_max", "cos_phi01_min", "cos_phi12_min",
              "rt_min", "rt_max", "x_over_x0", "chi2_max", "e_window", "xy_margin", "sigma_pixel",
              "chi2_vertex_max", "target_dist_max", "p_total_max"]:
        setattr(p, k, float(cfg[k]))
    for k in ["cuts_max", "max_tracks", "max_combs"]:
        setattr(p, k, int(cfg[k]))
    p.rel_band = float(cfg.get("rel_band", 1e-5))
    return p


def _d3(v):
    return (c_double * 3)(*[float(t) for t in v])


# ---------------------------------------------------------------- primitives
def tan_lambda(zi, zj, ri, rj):
    return lib().or_tan_lambda(zi, zj, ri, rj)


def cos_phi(xi, yi, xj, yj, ri, rj):
    return lib().or_cos_phi(xi, yi, xj, yj, ri, rj)


def circle_radius(h0, h1, h2):
    return lib().or_circle_radius(_d3(h0), _d3(h1), _d3(h2))


def arc_phi(d, z, k):
    return lib().or_arc_phi(d, z, k)


def highland(p, x0):
    return lib().or_highland(p, x0)


def target_distance(P: Params, x, y, z):
    return lib().or_target_distance(ctypes.byref(P), x, y, z)


def circle_intersections(c1, r1, c2, r2, band=1e-5):
    out = (c_double * 4)()
    m = ctypes.c_int(0)
    n = lib().or_circle_intersections(c1[0], c1[1], r1, c2[0], c2[1], r2, out, band, ctypes.byref(m))
    pts = [(out[0], out[1]), (out[2], out[3])][:n]
    return pts, bool(m.value)


def scattering_angles(h0, h1, h2, q, k):
    a, b = (c_double * 1)(), (c_double * 1)()
    rc = lib().or_scattering_angles(_d3(h0), _d3(h1), _d3(h2), q, k, a, b)
    if rc != 0:
        return None
    return a[0], b[0]


def fit_triplet(P: Params, h0, h1, h2) -> TripletFit:
    o = TripletFit()
    lib().or_fit_triplet(ctypes.byref(P), _d3(h0), _d3(h1), _d3(h2), ctypes.byref(o))
    return o


def extrapolate(P: Params, h1, h2, q, k):
    o = (c_double * 3)()
    if lib().or_extrapolate(ctypes.byref(P), _d3(h1), _d3(h2), q, k, o) != 0:
        return None
    return tuple(o)


# ---------------------------------------------------------------- frames
class Frames:
    """Keeps the numpy arrays alive and exposes per-frame start pointers."""

    def __init__(self, d: dict):
        self.x = np.ascontiguousarray(d["x"], dtype=np.float32)
        self.y = np.ascontiguousarray(d["y"], dtype=np.float32)
        self.z = np.ascontiguousarray(d["z"], dtype=np.float32)
        self.offsets = np.ascontiguousarray(d["offsets"], dtype=np.uint32)
        self.n = (len(self.offsets) - 1) // 4

    def start_ptr(self, f):
        return self.offsets.ctypes.data + 16 * f

    def layer_counts(self, f):
        o = self.offsets[4 * f:4 * f + 5].astype(np.int64)
        return np.diff(o)

    def hit(self, f, layer, i):
        g = int(self.offsets[4 * f + layer]) + i
        return (float(self.x[g]), float(self.y[g]), float(self.z[g]))


def select(P: Params, fr: Frames, f: int, cap: int = None):
    cap = cap or P.cuts_max
    buf = (Candidate * max(cap, 1))()
    res = FrameResult()
    n = lib().or_select(ctypes.byref(P), fr.x.ctypes.data, fr.y.ctypes.data, fr.z.ctypes.data,
                        fr.start_ptr(f), buf, cap, ctypes.byref(res))
    return [buf[i] for i in range(n)], res


def fit_candidate(P: Params, fr: Frames, f: int, cand: Candidate) -> Track:
    o = Track()
    lib().or_fit_candidate(ctypes.byref(P), fr.x.ctypes.data, fr.y.ctypes.data, fr.z.ctypes.data,
                           fr.start_ptr(f), ctypes.byref(cand), ctypes.byref(o))
    return o


def track_params(P: Params, h0, h1, kappa: float):
    """Reading R11 at signed curvature kappa: a Track with q, cos_theta01, cx, cy,
    rt, p, energy set (None if no short arc of that curvature joins h0, h1)."""
    o = Track()
    o.kappa = kappa
    if lib().or_track_params(ctypes.byref(P), _d3(h0), _d3(h1), kappa, ctypes.byref(o)) != 0:
        return None
    return o


def vertex_frame(P: Params, vtracks, all_cap=256):
    n = len(vtracks)
    arr = (VTrack * max(n, 1))(*vtracks)
    res = FrameResult()
    out = (Vertex * all_cap)()
    nv = lib().or_vertex_frame(ctypes.byref(P), arr, n, ctypes.byref(res), out, all_cap)
    return res, [out[i] for i in range(min(nv, all_cap))]


def process_frame(P: Params, fr: Frames, f: int):
    res = FrameResult()
    cb = (Candidate * (P.cuts_max + 1))()
    tb = (Track * (P.max_tracks + 1))()
    lib().or_process_frame(ctypes.byref(P), fr.x.ctypes.data, fr.y.ctypes.data, fr.z.ctypes.data,
                           fr.start_ptr(f), ctypes.byref(res), cb, tb)
    ntr = min(res.n_tracks, P.max_tracks)
    return res, [tb[i] for i in range(ntr)]


def process_frames(P: Params, fr: Frames, first: int = 0, count: int = None):
    count = fr.n - first if count is None else count
    res = (FrameResult * max(count, 1))()
    lib().or_process_frames(ctypes.byref(P), fr.x.ctypes.data, fr.y.ctypes.data, fr.z.ctypes.data,
                            fr.start_ptr(first), count, res)
    return res


def results_to_numpy(res) -> dict:
    n = len(res)
    out = {k: np.zeros(n, dtype=np.int64) for k in
           ["reason", "keep", "n_cand", "n_cand_marginal", "n_fit", "n_tracks", "n_fit_marginal",
            "n_pos", "n_neg", "n_combs", "n_vertex_marginal", "has_vertex"]}
    out["funnel"] = np.zeros((n, 5), dtype=np.int64)
    for i, r in enumerate(res):
        for k in out:
            if k == "funnel":
                out[k][i] = list(r.funnel)
            else:
                out[k][i] = getattr(r, k)
    return out
