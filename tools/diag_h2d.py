"""Diagnostics: raw pinned H2D bandwidth and a timing breakdown of m3e_filter_host."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2206_11535_b200 import m3e

n = 4 << 20
a = torch.empty(n * 64, dtype=torch.uint8).pin_memory()
b = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); b.copy_(a, non_blocking=True); torch.cuda.synchronize()
    print(f"pinned H2D {a.numel()/1e9:.2f} GB: {a.numel()/(time.perf_counter()-t)/1e9:.1f} GB/s")
F = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
d = synth.generate(synth.preset("phase1_sig"), F, threads=os.cpu_count())
params = m3e.make_params(m3e.load_config())
pin = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().numpy()
hx, hy, hz = (pin(np.concatenate([d[k], np.zeros(8, np.float32)])) for k in "xyz")
hoff = pin(d["offsets"])
kc = max(1024, F // 20)
h_reason = pin(np.zeros(F, np.uint8)); h_s = np.zeros(1, m3e.SUMMARY_DTYPE)
for chunk in (1 << 18, 1 << 20, 1 << 22):
    ctx = m3e.Context(0, max_frames=chunk)
    out = m3e.make_outputs(reason=h_reason, summary=h_s)
    m3e.filter_host(ctx, params, hx, hy, hz, hoff, F, out)
    t = time.perf_counter(); m3e.filter_host(ctx, params, hx, hy, hz, hoff, F, out); dt = time.perf_counter() - t
    print(f"filter_host chunk {chunk}: {dt*1e3:.1f} ms for {F} frames ({F/dt/1e6:.1f} M frames/s)")
    ctx.close()
