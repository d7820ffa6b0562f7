"""CPU-side check of the fit's fp32 arithmetic: the device code of the triplet fit
(paper_2206_11535_b200/csrc/m3e_device.cuh: fit_candidate, i.e. Eq. 5-8 and
Alg. 3 of PAPER.md Sec. IV-B) compiled for the host by tools/fit_numerics.cu and
compared, candidate by candidate, with the fp64 oracle on the oracle's own
Selection-Cut survivors, at north_star's bands (tests/parity.py): equal status
except for candidates the oracle marks marginal, equal layer-3 hit, kappa within
1e-4 relative, the Eq. 7 chi2 within 1e-3 of max(chi2, 1), cos theta_01 within
1e-4 (a 0.1% error in the fit's atan2 fails the chi2 check).  The GPU tests
(tests/test_gpu_parity.py) compare the kernels themselves; this pins the device
math on every CPU run, so a numerics change to the fit shows here before it
reaches a GPU box."""
import ctypes
import os
import shutil
import subprocess

import pytest

import oracle
import synth
from paper_2206_11535_b200 import m3e

from parity import REL_KAPPA, CHI2_DOMAIN

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHI2_REL = 1e-3   # |d chi2| / max(chi2, 1)


@pytest.fixture(scope="module")
def fitlib(tmp_path_factory):
    if shutil.which("nvcc") is None:
        pytest.skip("nvcc not available")
    so = str(tmp_path_factory.mktemp("fitnum") / "libfitnum.so")
    subprocess.check_call(["nvcc", "-std=c++17", "-O2", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-fPIC",
                           "-shared", "-I" + os.path.join(ROOT, "include"),
                           "-I" + os.path.join(ROOT, "paper_2206_11535_b200", "csrc"), "-o", so,
                           os.path.join(ROOT, "tools", "fit_numerics.cu")])
    L = ctypes.CDLL(so)
    vp = ctypes.c_void_p
    L.fit_numerics.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_float, vp]
    return L


@pytest.mark.parametrize("preset,n,seed", [("phase1_sig", 250, 77), ("signal_only", 150, 78)])
def test_fit_math_matches_oracle(fitlib, preset, n, seed):
    cfg = m3e.load_config()
    P, gp = oracle.make_params(cfg), m3e.make_params(cfg)
    d = synth.generate(synth.preset(preset, seed=seed), n)
    fr = oracle.Frames(d)
    out = (ctypes.c_float * 11)()
    ncand = nacc = excused = 0
    worst_k = worst_c = worst_x = 0.0
    for f in range(n):
        cands, _ = oracle.select(P, fr, f)
        for c in cands:
            o = oracle.fit_candidate(P, fr, f, c)
            ncand += 1
            fitlib.fit_numerics(ctypes.addressof(gp), fr.x.ctypes.data, fr.y.ctypes.data, fr.z.ctypes.data,
                                fr.offsets.ctypes.data + 16 * f, c.i0, c.i1, c.i2, c.rtc, ctypes.addressof(out))
            st = int(out[0])
            if st != o.status:
                assert o.marginal or c.marginal, (f, c.i0, c.i1, c.i2, st, o.status)
                excused += 1
                continue
            if o.status >= 2 and o.status != 3:
                assert int(out[1]) == o.hit[3], (f, c.i0, c.i1, c.i2)
            if o.status in (0, 5) and o.chi2 < CHI2_DOMAIN:
                dk = abs(out[6] - o.kappa) / abs(o.kappa)
                assert dk <= REL_KAPPA, (f, dk)
                worst_k = max(worst_k, dk)
                # Eq. 7 chi2 at kappa-bar: fp32 rounding only (measured <= 3e-5)
                dx = abs(out[7] - o.chi2) / max(o.chi2, 1.0)
                assert dx <= CHI2_REL, (f, dx)
                worst_x = max(worst_x, dx)
            if o.status == 0:
                nacc += 1
                dc = abs(out[8] - o.cos_theta01)
                assert dc <= 1e-4, (f, dc)
                worst_c = max(worst_c, dc)
    print(f"{preset}: {ncand} candidates, {nacc} accepted, {excused} marginal, "
          f"worst kappa {worst_k:.2e} rel, worst chi2 {worst_x:.2e}, worst cos theta01 {worst_c:.2e}")
    assert ncand > 100 and nacc > 50
