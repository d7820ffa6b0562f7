"""The check build of the CUDA path (lib/libm3e_check.so, -DM3E_CHECK: the
kernels bounds-check their shared-memory, candidate-store, staging-window and
output-slot indices and record the first failed check, include/m3e.h
m3e_debug_check) on every workload shape: no check fails, and its outputs are
byte-identical to the production library's."""
import hashlib
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_2206_11535_b200", "lib", "libm3e_check.so")

# (workload or muon rate, frames, seed, environment of m3e_create)
CASES = [("phase1_sig", 20000, 901, {}), ("signal_only", 2000, 902, {}), ("phase2_stress", 300, 903, {}),
         (1.2e9, 40, 904, {}), (1.7e9, 12, 905, {}), ("single_frame", 1, 906, {}),
         ("phase1_sig", 5000, 907, {"M3E_CAND_STORE": "2"}), ("phase1_sig", 3000, 908, {"M3E_FUSED": "1"}),
         ("phase2_stress", 80, 909, {"M3E_TRI_CAP": "5"})]

SCRIPT = r"""
import hashlib, json, os, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
import synth
from paper_2206_11535_b200 import m3e
w, n, seed, env = json.loads(sys.argv[1])
os.environ.update(env)
sc = synth.preset(w, seed=seed) if isinstance(w, str) else synth.SynthConfig(muon_rate=w, seed=seed)
d = synth.generate(sc, n)
ctx = m3e.Context(0)
res = m3e.run_filter(ctx, m3e.make_params(m3e.load_config()), m3e.DeviceFrames(d))
torch.cuda.synchronize()
sm = res.summary_np()
h = hashlib.sha256()
for a in (res.reason.cpu().numpy()[:n], res.frames_np(n), res.tracks_np(int(sm["track_slots"])),
          res.vertices_np(int(sum(sm["kept_by_reason"][1:])))):
    h.update(np.ascontiguousarray(a).tobytes())
print(json.dumps({"line": ctx.debug_check(), "hash": h.hexdigest(), "kept": [int(v) for v in sm["kept_by_reason"]],
                  "overflow": int(sm["overflow"])}))
"""


def _run(lib, case):
    env = dict(os.environ)
    if lib:
        env["M3E_LIB"] = lib
    else:
        env.pop("M3E_LIB", None)
    out = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}, json.dumps(case)], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-{'-'.join(c[3]) or 'split'}")
def test_check_build(case):
    assert os.path.exists(CHECK_LIB), "run __graft_entry__.build()"
    chk = _run(CHECK_LIB, case)
    prod = _run(None, case)
    print(case, chk)
    assert chk["line"] == 0, f"index check failed at m3e_kernels.cu line {chk['line']}"
    assert prod["line"] == 0xFFFFFFFF   # the production library has no checks compiled in
    assert chk["overflow"] == 0
    assert chk["hash"] == prod["hash"] and chk["kept"] == prod["kept"]
