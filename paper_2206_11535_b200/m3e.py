"""Thin ctypes binding of libm3e.so (include/m3e.h).

Argument marshalling only: every step of the filter runs in the CUDA kernels of
csrc/.  Device buffers are torch tensors (PyTorch is used for device memory,
streams and process groups); host buffers are numpy arrays.  There is no CPU
fallback: if the shared library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# M3E_LIB: path of an alternative build (tuning experiments); default the in-tree build
LIB_PATH = os.environ.get("M3E_LIB") or os.path.join(_HERE, "lib", "libm3e.so")
ROOT = os.path.dirname(_HERE)
DEFAULT_CONFIG = os.path.join(ROOT, "config", "thresholds.json")

REASON_NONE, REASON_TRIPLET_OVERFLOW, REASON_TRACK_OVERFLOW, REASON_COMB_OVERFLOW, REASON_VERTEX, \
    REASON_INVALID = range(6)
REASON_NAMES = ["none", "triplet_overflow", "track_overflow", "comb_overflow", "vertex_found", "invalid"]

_d, _i32, _u64, _vp = ctypes.c_double, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p


class Params(ctypes.Structure):
    _fields_ = [("layer_r", _d * 4), ("b_field", _d), ("target_r", _d), ("target_half", _d),
                ("dlambda_max", _d), ("cos_phi01_min", _d), ("cos_phi12_min", _d), ("rt_min", _d),
                ("rt_max", _d), ("cuts_max", _i32), ("x_over_x0", _d), ("chi2_max", _d),
                ("max_tracks", _i32), ("e_window", _d), ("xy_margin", _d), ("sigma_pixel", _d),
                ("chi2_vertex_max", _d), ("target_dist_max", _d), ("p_total_max", _d),
                ("max_combs", _i32)]


class Outputs(ctypes.Structure):
    _fields_ = [("reason", _vp), ("frames", _vp), ("tracks", _vp), ("track_capacity", _u64),
                ("vertices", _vp), ("kept_frame", _vp), ("kept_offsets", _vp),
                ("kept_capacity", _u64), ("kept_x", _vp), ("kept_y", _vp), ("kept_z", _vp),
                ("kept_hit_capacity", _u64), ("summary", _vp)]


# numpy views of the output records (layouts of include/m3e.h)
FRAME_DTYPE = np.dtype([("n_cand", "<u2"), ("n_tracks", "<u2"), ("n_combs", "<u2"), ("reason", "u1"),
                        ("n_neg", "u1"), ("track_first", "<u4"), ("kept_index", "<u4")])
TRACK_DTYPE = np.dtype([("frame", "<u4"), ("hit", "<u2", (4,)), ("kappa", "<f4"), ("chi2", "<f4"),
                        ("cos_theta01", "<f4"), ("cx", "<f4"), ("cy", "<f4")])
VERTEX_DTYPE = np.dtype([("frame", "<u4"), ("track", "<u2", (3,)), ("pad", "<u2"), ("target_dist", "<f4"),
                         ("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("chi2", "<f8"), ("p_total", "<f4"),
                         ("pad2", "<u4")])
FIT_DTYPE = np.dtype([("status", "u1"), ("pad", "u1"), ("hit3", "<u2"), ("kappa1", "<f4"),
                      ("kappa2", "<f4"), ("var1", "<f4"), ("var2", "<f4"), ("kappa", "<f4"),
                      ("chi2", "<f4"), ("cos_theta01", "<f4"), ("cx", "<f4"), ("cy", "<f4")])
SUMMARY_DTYPE = np.dtype([("frames", "<u8"), ("kept_by_reason", "<u8", (6,)), ("candidates", "<u8"),
                          ("tracks", "<u8"), ("kept_hits", "<u8"), ("vertices", "<u8"),
                          ("overflow", "<u8"), ("track_slots", "<u8")])
assert FRAME_DTYPE.itemsize == 16 and TRACK_DTYPE.itemsize == 32 and VERTEX_DTYPE.itemsize == 56
assert FIT_DTYPE.itemsize == 40 and SUMMARY_DTYPE.itemsize == 104

_lib = None


def lib():
    """Load libm3e.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.m3e_version.restype = ctypes.c_char_p
        L.m3e_last_error.restype = ctypes.c_char_p
        L.m3e_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _u64, _u64]
        L.m3e_destroy.argtypes = [_vp]
        L.m3e_workspace_bytes.restype = _u64
        L.m3e_workspace_bytes.argtypes = [_vp]
        L.m3e_set_timing.argtypes = [_vp, ctypes.c_int]
        L.m3e_kernel_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_float)]
        L.m3e_debug_check.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint32)]
        P = ctypes.POINTER(Params)
        O = ctypes.POINTER(Outputs)
        L.m3e_filter.argtypes = [_vp, P, _vp, _vp, _vp, _vp, _u64, _u64, O, _vp]
        L.m3e_filter_host.argtypes = [_vp, P, _vp, _vp, _vp, _vp, _u64, O]
        L.m3e_select_triplets.argtypes = [_vp, P, _vp, _vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp]
        L.m3e_fit_tracks.argtypes = [_vp, P, _vp, _vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.m3e_vertex_select.argtypes = [_vp, P, _vp, _vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp, _vp]
        L.m3e_pack_frames.argtypes = [_vp, _vp, _vp, _vp, _vp, _u64, _u64, _vp, O, _vp]
        _lib = L
    return _lib


# names of every symbol include/m3e.h declares (checked by the CPU tests)
EXPORTED = ["m3e_version", "m3e_last_error", "m3e_create", "m3e_destroy", "m3e_workspace_bytes",
            "m3e_set_timing", "m3e_kernel_times", "m3e_debug_check",
            "m3e_filter", "m3e_filter_host", "m3e_select_triplets", "m3e_fit_tracks",
            "m3e_vertex_select", "m3e_pack_frames"]


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"libm3e error {rc}: {lib().m3e_last_error().decode()}")


def load_config(path: str = DEFAULT_CONFIG) -> dict:
    with open(path) as fh:
        return json.load(fh)


def make_params(cfg: dict) -> Params:
    p = Params()
    for i in range(4):
        p.layer_r[i] = cfg["layer_r"][i]
    for k in ["b_field", "target_r", "target_half", "dlambda_max", "cos_phi01_min", "cos_phi12_min",
              "rt_min", "rt_max", "x_over_x0", "chi2_max", "e_window", "xy_margin", "sigma_pixel",
              "chi2_vertex_max", "target_dist_max", "p_total_max"]:
        setattr(p, k, float(cfg[k]))
    for k in ["cuts_max", "max_tracks", "max_combs"]:
        setattr(p, k, int(cfg[k]))
    return p


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Context:
    """Device workspace + streams of libm3e (m3e_create / m3e_destroy)."""

    def __init__(self, device: int = 0, max_frames: int = 0, max_hits: int = 0):
        self._h = _vp()
        _check(lib().m3e_create(ctypes.byref(self._h), device, max_frames, max_hits))
        self.device = device

    def close(self):
        if self._h:
            lib().m3e_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def workspace_bytes(self) -> int:
        return int(lib().m3e_workspace_bytes(self._h))

    def set_timing(self, enable: bool = True):
        _check(lib().m3e_set_timing(self._h, int(enable)))

    def kernel_times(self):
        """Mean (selection, fit, tracks, vertex, finish, pack) kernel ms over the
        m3e_filter calls since the last reset (include/m3e.h m3e_kernel_times);
        the first four are 0 on the single-kernel (M3E_FUSED=1) path, where the
        filter kernel ("finish") runs every stage."""
        ms = (ctypes.c_float * 6)()
        _check(lib().m3e_kernel_times(self._h, ms))
        return tuple(float(v) for v in ms)

    def debug_check(self) -> int:
        """Source line of the first failed internal index check since the last
        call (0: none; 0xFFFFFFFF: the library was built without checks), see
        include/m3e.h m3e_debug_check."""
        line = ctypes.c_uint32(0)
        _check(lib().m3e_debug_check(self._h, ctypes.byref(line)))
        return int(line.value)


def make_outputs(**kw) -> Outputs:
    o = Outputs()
    for k, v in kw.items():
        if k.endswith("capacity"):
            setattr(o, k, int(v))
        else:
            setattr(o, k, _ptr(v))
    return o


def filter_device(ctx: Context, params: Params, x, y, z, offsets, n_frames: int, n_hits: int,
                  outputs: Outputs, stream=None):
    """m3e_filter: full hot path on device tensors (outputs: device tensors in `outputs`)."""
    _check(lib().m3e_filter(ctx.handle, ctypes.byref(params), _ptr(x), _ptr(y), _ptr(z), _ptr(offsets),
                            n_frames, n_hits, ctypes.byref(outputs), _stream(stream)))


def filter_host(ctx: Context, params: Params, x, y, z, offsets, n_frames: int, outputs: Outputs):
    """m3e_filter_host: host (numpy, preferably pinned) input and outputs; synchronous."""
    _check(lib().m3e_filter_host(ctx.handle, ctypes.byref(params), _ptr(x), _ptr(y), _ptr(z),
                                 _ptr(offsets), n_frames, ctypes.byref(outputs)))


def select_triplets(ctx, params, x, y, z, offsets, n_frames, n_hits, cand, cand_rt, frames, stream=None):
    _check(lib().m3e_select_triplets(ctx.handle, ctypes.byref(params), _ptr(x), _ptr(y), _ptr(z),
                                     _ptr(offsets), n_frames, n_hits, _ptr(cand), _ptr(cand_rt),
                                     _ptr(frames), _stream(stream)))


def fit_tracks(ctx, params, x, y, z, offsets, n_frames, n_hits, cand, cand_rt, n_cand, rec, tracks,
               frames, stream=None):
    _check(lib().m3e_fit_tracks(ctx.handle, ctypes.byref(params), _ptr(x), _ptr(y), _ptr(z), _ptr(offsets),
                                n_frames, n_hits, _ptr(cand), _ptr(cand_rt), _ptr(n_cand), _ptr(rec),
                                _ptr(tracks), _ptr(frames), _stream(stream)))


def vertex_select(ctx, params, x, y, z, offsets, n_frames, n_hits, tracks, n_tracks, frames, vertices,
                  stream=None):
    _check(lib().m3e_vertex_select(ctx.handle, ctypes.byref(params), _ptr(x), _ptr(y), _ptr(z),
                                   _ptr(offsets), n_frames, n_hits, _ptr(tracks), _ptr(n_tracks),
                                   _ptr(frames), _ptr(vertices), _stream(stream)))


def pack_frames(ctx, x, y, z, offsets, n_frames, n_hits, reason, outputs: Outputs, stream=None):
    _check(lib().m3e_pack_frames(ctx.handle, _ptr(x), _ptr(y), _ptr(z), _ptr(offsets), n_frames, n_hits,
                                 _ptr(reason), ctypes.byref(outputs), _stream(stream)))


# ------------------------------------------------------------ conveniences
class DeviceFrames:
    """Frames resident in HBM (SoA x/y/z with 16 B slack + offsets), torch tensors."""

    def __init__(self, d: dict, device="cuda"):
        import torch
        H = len(d["x"])
        self.n_frames = (len(d["offsets"]) - 1) // 4
        self.n_hits = H

        def f32(a):
            t = torch.zeros(H + 8, dtype=torch.float32, device=device)
            if H:
                t[:H] = torch.from_numpy(np.ascontiguousarray(a[:H], dtype=np.float32)).to(device)
            return t

        self.x, self.y, self.z = f32(d["x"]), f32(d["y"]), f32(d["z"])
        off = np.ascontiguousarray(d["offsets"], dtype=np.uint32).view(np.int32)
        self.offsets = torch.from_numpy(off.copy()).to(device)


class Result:
    """Device output buffers of one m3e_filter call and their host views."""

    def __init__(self, n_frames: int, n_hits: int, track_capacity: Optional[int] = None,
                 kept_capacity: Optional[int] = None, device="cuda"):
        import torch
        F = max(n_frames, 1)
        self.track_capacity = track_capacity if track_capacity is not None else 64 * F + 1024
        self.kept_capacity = kept_capacity if kept_capacity is not None else F
        kh = n_hits + 8 if kept_capacity is None else max(8, n_hits)
        u8 = dict(dtype=torch.uint8, device=device)
        self.reason = torch.zeros(F, **u8)
        self.frames = torch.zeros(F * 16, **u8)
        self.tracks = torch.zeros(self.track_capacity * 32, **u8)
        self.vertices = torch.zeros(self.kept_capacity * 56, **u8)
        self.kept_frame = torch.zeros(self.kept_capacity, dtype=torch.int32, device=device)
        self.kept_offsets = torch.zeros(4 * self.kept_capacity + 1, dtype=torch.int32, device=device)
        self.kept_x = torch.zeros(kh, dtype=torch.float32, device=device)
        self.kept_y = torch.zeros(kh, dtype=torch.float32, device=device)
        self.kept_z = torch.zeros(kh, dtype=torch.float32, device=device)
        self.summary = torch.zeros(SUMMARY_DTYPE.itemsize, **u8)
        self.outputs = make_outputs(reason=self.reason, frames=self.frames, tracks=self.tracks,
                                    track_capacity=self.track_capacity, vertices=self.vertices,
                                    kept_frame=self.kept_frame, kept_offsets=self.kept_offsets,
                                    kept_capacity=self.kept_capacity, kept_x=self.kept_x,
                                    kept_y=self.kept_y, kept_z=self.kept_z,
                                    kept_hit_capacity=kh, summary=self.summary)

    def summary_np(self):
        return self.summary.cpu().numpy().view(SUMMARY_DTYPE)[0]

    def frames_np(self, n_frames):
        return self.frames.cpu().numpy().view(FRAME_DTYPE)[:n_frames]

    def tracks_np(self, n):
        return self.tracks.cpu().numpy().view(TRACK_DTYPE)[:n]

    def vertices_np(self, n):
        return self.vertices.cpu().numpy().view(VERTEX_DTYPE)[:n]


def run_filter(ctx: Context, params: Params, fr: DeviceFrames, res: Optional[Result] = None, stream=None):
    res = res or Result(fr.n_frames, fr.n_hits)
    filter_device(ctx, params, fr.x, fr.y, fr.z, fr.offsets, fr.n_frames, fr.n_hits, res.outputs, stream)
    return res
