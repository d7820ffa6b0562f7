#!/usr/bin/env python3
"""Small filter runs for compute-sanitizer (memcheck / racecheck / synccheck):
  compute-sanitizer --tool memcheck python tools/sanitize_run.py [split|fused]
Prints each workload's kept-by-reason counts (the run must also be correct)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "fused":
    os.environ["M3E_FUSED"] = "1"
if len(sys.argv) > 1 and sys.argv[1] == "spill":
    os.environ["M3E_CAND_STORE"] = "2"

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2206_11535_b200 import m3e  # noqa: E402

sizes = [("phase1_sig", 20000), ("signal_only", 3000), ("phase2_stress", 300), ("single_frame", 1)]
if len(sys.argv) > 2:
    sizes = [(w, int(n)) for w, n in (a.split(":") for a in sys.argv[2:])]
gp = m3e.make_params(m3e.load_config())
ctx = m3e.Context(0)
for name, n in sizes:
    d = synth.generate(synth.preset(name, seed=4321), n)
    res = m3e.run_filter(ctx, gp, m3e.DeviceFrames(d))
    torch.cuda.synchronize()
    print(name, n, np.array(res.summary_np()["kept_by_reason"]))
# the host path (chunks, two streams, device rebase)
d = synth.generate(synth.preset("phase1_sig", seed=4322), 5000)
small = m3e.Context(0, max_frames=1234)
H = len(d["x"])
keep = dict(reason=np.zeros(5000, np.uint8), frames=np.zeros(5000, m3e.FRAME_DTYPE),
            tracks=np.zeros(16 * 5000, m3e.TRACK_DTYPE), vertices=np.zeros(5000, m3e.VERTEX_DTYPE),
            kept_frame=np.zeros(5000, np.uint32), kept_offsets=np.zeros(4 * 5000 + 1, np.uint32),
            kept_x=np.zeros(H + 8, np.float32), kept_y=np.zeros(H + 8, np.float32),
            kept_z=np.zeros(H + 8, np.float32), summary=np.zeros(1, m3e.SUMMARY_DTYPE))   # alive during the call
out = m3e.make_outputs(track_capacity=16 * 5000, kept_capacity=5000, kept_hit_capacity=H + 8, **keep)
x, y, z = (np.concatenate([d[k], np.zeros(8, np.float32)]) for k in "xyz")
m3e.filter_host(small, gp, x, y, z, d["offsets"], 5000, out)
print("host path 5000", np.array(keep["summary"][0]["kept_by_reason"]))
small.close()
ctx.close()
