#!/usr/bin/env python3
"""Host study of the fp32 fit variants (tools/fit_numerics.cu built with each set of
-D flags) against the fp64 oracle: status / layer-3 hit mismatches and worst
kappa, chi2, cos theta deviations.  Usage: fit_numerics_study.py n_frames preset
"-DFLAG=.." ... ("" = default build).  Test infrastructure, not product."""
import ctypes, sys, subprocess, numpy as np
sys.path.insert(0, '/root/repo')
import oracle, synth
from paper_2206_11535_b200 import m3e
def build(tag, flags):
    so = f"/tmp/fitnum2_{tag}.so"
    subprocess.check_call(["nvcc", "-std=c++17", "-O2", "-Xcompiler", "-fPIC", "-shared", "-I/root/repo/include",
        "-I/root/repo/paper_2206_11535_b200/csrc", *flags, "-o", so, "/root/repo/tools/fit_numerics.cu"], stderr=subprocess.DEVNULL)
    L = ctypes.CDLL(so)
    vp = ctypes.c_void_p
    L.fit_numerics.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_float, vp]
    return L
cfg = m3e.load_config(); P = oracle.make_params(cfg); gp = m3e.make_params(cfg)
n = int(sys.argv[1]); preset = sys.argv[2]
variants = [(a, a.split()) if a else ("default", []) for a in sys.argv[3:]]
libs = [(t, build(str(i), fl)) for i, (t, fl) in enumerate(variants)]
d = synth.generate(synth.preset(preset, seed=77), n)
fr = oracle.Frames(d)
out = (ctypes.c_float * 11)()
stats = {t: [0, 0, 0.0, 0.0, 0.0] for t, _ in libs}
ncand = 0
for f in range(n):
    cands, res = oracle.select(P, fr, f)
    for c in cands:
        o = oracle.fit_candidate(P, fr, f, c)
        ncand += 1
        for t, L in libs:
            L.fit_numerics(ctypes.addressof(gp), fr.x.ctypes.data, fr.y.ctypes.data, fr.z.ctypes.data,
                           fr.offsets.ctypes.data + 16 * f, c.i0, c.i1, c.i2, c.rtc, ctypes.addressof(out))
            s = stats[t]
            if int(out[0]) != o.status:
                if not (o.marginal or c.marginal): s[0] += 1
                continue
            if o.status >= 2 and o.status != 3 and int(out[1]) != o.hit[3]: s[1] += 1
            if o.status in (0, 5) and o.chi2 < 1000:
                s[2] = max(s[2], abs(out[6] - o.kappa) / abs(o.kappa))
                s[4] = max(s[4], abs(out[7] - o.chi2) / max(o.chi2, 1.0))
            if o.status == 0: s[3] = max(s[3], abs(out[8] - o.cos_theta01))
for t, s in stats.items():
    print(f"{t}: {ncand} cands, status mismatches {s[0]}, hit3 mismatches {s[1]}, worst kappa {s[2]:.2e}, worst chi2 {s[4]:.2e}, worst cth {s[3]:.2e}")
