"""Seeded synthetic Mu3e frames (input synthesis only; see synth_core.h).

This module is the one thing the oracle side (tests, oracle/) and the CUDA side
(bench.py, GPU tests) share: it produces hit frames and truth.  It holds none of
the filter's arithmetic.

Frame layout produced (the layout the C-ABI consumes):
  x, y, z : float32[H]         hits, sorted by frame then layer
  offsets : uint32[4*F + 1]    offsets[4f+l] = first hit of layer l in frame f,
                               offsets[4F]   = H
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libm3e_synth.so")

# Frame length and rates: PAPER.md Sec. VI ("64 ns long frames"), Sec. III
# (1e8 mu/s phase I, 1e9 mu/s phase II).
FRAME_NS = 64.0
PHASE1_RATE = 1e8
PHASE2_RATE = 1e9
# One second of phase-I data at 64 ns frames = 1/64ns = 15.625e6 frames; the paper's
# 12-PC farm target is 1.302e6 frames/s per PC (Sec. VI) = 15.625e6 / 12.
FRAMES_PER_SECOND = int(round(1e9 / FRAME_NS))


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("muon_rate", ctypes.c_double),
        ("frame_ns", ctypes.c_double),
        ("signal_fraction", ctypes.c_double),
        ("fixed_michel", ctypes.c_int),
        ("fixed_signal", ctypes.c_int),
        ("noise_per_layer", ctypes.c_double),
        ("x_over_x0", ctypes.c_double),
        ("sigma_pixel", ctypes.c_double),
        ("ms_on", ctypes.c_int),
        ("normal_incidence", ctypes.c_int),
        ("seed", ctypes.c_uint64),
        ("layer_r", ctypes.c_double * 4),
        ("layer_half", ctypes.c_double * 4),
        ("b_field", ctypes.c_double),
        ("target_r", ctypes.c_double),
        ("target_half", ctypes.c_double),
    ]


class Particle(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("charge", ctypes.c_int),
        ("decay", ctypes.c_int),
        ("layer_mask", ctypes.c_int),
        ("p", ctypes.c_double * 3),
        ("v", ctypes.c_double * 3),
    ]


KIND_MICHEL, KIND_SIG_EPLUS, KIND_SIG_EMINUS = 0, 1, 2


@dataclasses.dataclass
class SynthConfig:
    """Generator configuration.  Geometry defaults: layer radii 23.3/29.8/73.9/86.3 mm
    and half lengths 60/60/170/180 mm read off PAPER.md Fig. 3 (axes of the
    transverse and longitudinal sketches); target cone radius 19 mm (Sec. IV-C),
    half length 50 mm (Fig. 3 target polygon); B = 1 T (Sec. III-B)."""

    muon_rate: float = PHASE1_RATE
    frame_ns: float = FRAME_NS
    signal_fraction: float = 0.0
    fixed_michel: int = -1
    fixed_signal: int = -1
    noise_per_layer: float = 0.25
    x_over_x0: float = 0.00115
    sigma_pixel: float = 0.080 / np.sqrt(12.0)
    ms_on: bool = True
    normal_incidence: bool = False
    seed: int = 20220623
    layer_r: tuple = (23.3, 29.8, 73.9, 86.3)
    layer_half: tuple = (60.0, 60.0, 170.0, 180.0)
    b_field: float = 1.0
    target_r: float = 19.0
    target_half: float = 50.0

    def _c(self) -> _Cfg:
        c = _Cfg()
        c.muon_rate = self.muon_rate
        c.frame_ns = self.frame_ns
        c.signal_fraction = self.signal_fraction
        c.fixed_michel = self.fixed_michel
        c.fixed_signal = self.fixed_signal
        c.noise_per_layer = self.noise_per_layer
        c.x_over_x0 = self.x_over_x0
        c.sigma_pixel = self.sigma_pixel
        c.ms_on = int(self.ms_on)
        c.normal_incidence = int(self.normal_incidence)
        c.seed = self.seed & ((1 << 64) - 1)
        for i in range(4):
            c.layer_r[i] = self.layer_r[i]
            c.layer_half[i] = self.layer_half[i]
        c.b_field = self.b_field
        c.target_r = self.target_r
        c.target_half = self.target_half
        return c


def preset(name: str, seed: int = 20220623) -> SynthConfig:
    """Configurations of BASELINE.json "configs"."""
    if name == "single_frame":  # configs[0]: one mu->eee + 5 Michel tracks
        return SynthConfig(fixed_signal=1, fixed_michel=5, seed=seed)
    if name == "phase1_bg":  # configs[1], configs[3]: 1e8 mu/s, Michel background only
        return SynthConfig(muon_rate=PHASE1_RATE, signal_fraction=0.0, seed=seed)
    if name == "phase1_sig":  # configs[2]: 1e8 mu/s, signal injected in 1% of frames
        return SynthConfig(muon_rate=PHASE1_RATE, signal_fraction=0.01, seed=seed)
    if name == "signal_only":  # every frame one signal decay, no background (efficiency studies)
        return SynthConfig(fixed_signal=1, fixed_michel=0, noise_per_layer=0.0, seed=seed)
    if name == "phase2_stress":  # configs[4]: 1e9 mu/s pile-up
        return SynthConfig(muon_rate=PHASE2_RATE, signal_fraction=0.0, seed=seed)
    raise KeyError(name)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB_PATH)
        L.synth_count.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_void_p, ctypes.c_int]
        L.synth_write.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.synth_particles.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint64,
                                      ctypes.POINTER(Particle), ctypes.c_int]
        assert L.synth_sizeof_cfg() == ctypes.sizeof(_Cfg)
        assert L.synth_sizeof_particle() == ctypes.sizeof(Particle)
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def generate(cfg: SynthConfig, n_frames: int, frame0: int = 0, truth: bool = False,
             threads: Optional[int] = None) -> dict:
    """Generate frames frame0 .. frame0+n_frames-1 (host, numpy arrays)."""
    L = lib()
    c = cfg._c()
    nt = threads or min(64, os.cpu_count() or 1)
    counts = np.zeros(4 * n_frames, dtype=np.uint32)
    if L.synth_count(ctypes.byref(c), frame0, n_frames, _ptr(counts), nt) != 0:
        raise RuntimeError("synth_count failed")
    offsets = np.zeros(4 * n_frames + 1, dtype=np.uint64)
    np.cumsum(counts, out=offsets[1:])
    if offsets[-1] >= 2**32:
        raise ValueError("more than 2^32 hits in one call; split the frame range")
    offsets = offsets.astype(np.uint32)
    H = int(offsets[-1])
    # +16 floats of slack so vector/bulk loads may round the end up (HBM layout)
    x = np.zeros(H + 16, dtype=np.float32)
    y = np.zeros(H + 16, dtype=np.float32)
    z = np.zeros(H + 16, dtype=np.float32)
    hp = np.zeros(H + 16, dtype=np.int32) if truth else None
    if L.synth_write(ctypes.byref(c), frame0, n_frames, _ptr(offsets), _ptr(x), _ptr(y), _ptr(z),
                     _ptr(hp), nt) != 0:
        raise RuntimeError("synth_write failed")
    out = {"x": x[:H], "y": y[:H], "z": z[:H], "offsets": offsets, "n_frames": n_frames,
           "frame0": frame0}
    if truth:
        out["hit_particle"] = hp[:H]
    return out


def particles(cfg: SynthConfig, frame_id: int) -> list:
    """Truth particle table of one frame (list of dicts)."""
    L = lib()
    c = cfg._c()
    buf = (Particle * 512)()
    n = L.synth_particles(ctypes.byref(c), frame_id, buf, 512)
    return [dict(kind=buf[i].kind, charge=buf[i].charge, decay=buf[i].decay,
                 layer_mask=buf[i].layer_mask, p=tuple(buf[i].p), v=tuple(buf[i].v))
            for i in range(n)]
