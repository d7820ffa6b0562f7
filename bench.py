#!/usr/bin/env python3
"""Benchmark of the Mu3e online event selection hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one pass of the whole hot path (Selection Cuts -> triplet fit ->
vertex selection -> packer, one m3e_filter launch) over the workload:
BASELINE.json configs[3], one second of phase-I data = 15,625,000 frames of
64 ns at 1e8 mu/s (Michel background + 1% injected mu->eee signal), resident in
HBM.  N > 1: launched by torchrun, one rank per GPU; every rank filters its own
second of data (distinct frame ids), weak scaling; the only NCCL traffic is the
final reduction of counters (after the timed region).

Metric: input Gbps, Phase-I equivalent: the paper's 80 Gbps
is the phase-I stream at 1e8 mu/s = 15.625e6 frames/s (PAPER.md abstract,
Sec. VI), so Gbps_equiv = frames/s * 80 / 15.625e6.  hits/s, frames/s, the
bytes/s of the SoA hit stream the GPU actually reads, and the reduction factor
are reported beside it.

--impl reference times the CPU oracle (oracle/, fp64, one core) on a bounded
sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PHASE1_FRAMES_PER_S = 1e9 / 64.0      # 15.625e6 frames per second of phase-I data
PHASE1_GBPS = 80.0                     # PAPER.md abstract
METRIC = "input Gbps (Phase-I equivalent; hits/s, frames/s per B200), reduction factor"


def gbps_equiv(frames_per_s: float, muon_rate: float = 1e8) -> float:
    """Phase-I-equivalent input rate: 80 Gbps is 15.625e6 frames/s at 1e8 mu/s
    (PAPER.md abstract, Sec. VI); the detector data per frame scales with the muon
    rate, so a frame at rate R counts R / 1e8 phase-I frames."""
    return frames_per_s * PHASE1_GBPS / PHASE1_FRAMES_PER_S * (muon_rate / 1e8)


WORKLOAD_TEXT = {
    "phase1_sig": "configs[3]: 1 s of phase-I data per GPU = {F} frames of 64 ns at 1e8 mu/s "
                  "(Michel background + noise, 1% injected mu->eee)",
    "phase1_bg": "configs[1]-like: {F} frames of 64 ns at 1e8 mu/s (Michel background + noise only)",
    "phase2_stress": "configs[4]: {F} frames of 64 ns at 1e9 mu/s per GPU (phase-II pile-up, Michel + noise)",
}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed
    region (one `nvidia-smi -lms 50` process, started before and stopped after)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        import tempfile
        self._f = tempfile.TemporaryFile(mode="w+")
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "50"], stdout=self._f,
                                       stderr=subprocess.DEVNULL)
        except OSError:
            self._p = None
        time.sleep(0.3)   # nvidia-smi start-up before the timed region
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(5)
            except subprocess.TimeoutExpired:
                self._p.kill()
        self._f.seek(0)
        self.rows = [[c.strip() for c in l.split(",")] for l in self._f.read().splitlines() if l.strip()]
        self._f.close()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def kernel_source_hash() -> str:
    """sha256 (16 hex) of the CUDA sources: a committed ncu capture is used only if
    it was taken of these sources"""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2206_11535_b200", "csrc")
    for fn in sorted(os.listdir(csrc)):
        with open(os.path.join(csrc, fn), "rb") as fh:
            h.update(fn.encode() + fh.read())
    return h.hexdigest()[:16]


def load_profile(workload: str, frames: int, seed: int):
    """Per-kernel ncu counters (DRAM bytes, executed warp instructions, pipe
    utilisation per launch) of the committed capture of this exact configuration
    AND these kernel sources (profiles/*_bench_traffic.json): (kernels, file name),
    else ({}, None)."""
    import glob
    src = kernel_source_hash()
    for fn in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_bench_traffic.json")), reverse=True):
        try:
            t = json.load(open(fn))
        except Exception:
            continue
        if (t.get("workload") == workload and t.get("frames") == frames and t.get("seed") == seed
                and t.get("source_hash") == src):
            return t.get("kernels", {}), os.path.relpath(fn, ROOT)
    return {}, None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def generate(preset: str, n_frames: int, frame0: int, seed: int, world: int = 1):
    cfg = synth.preset(preset, seed=seed)
    t = time.time()
    # ranks of one node generate concurrently: share the host cores
    d = synth.generate(cfg, n_frames, frame0=frame0, threads=max(1, (os.cpu_count() or 1) // max(world, 1)))
    return d, time.time() - t


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def time_oracle(P, fr, first: int, count: int, threads: int) -> float:
    """Wall time of the CPU oracle (unchanged, fp64 C) over frames [first,
    first + count), split into `threads` contiguous slices run concurrently (frames
    are independent, Sec. V; ctypes releases the GIL during each call)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    cuts = [first + count * i // threads for i in range(threads + 1)]
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: oracle.process_frames(P, fr, first=cuts[i], count=cuts[i + 1] - cuts[i]),
                    range(threads)))
    return time.perf_counter() - t


def run_reference(a, rank, world):
    """Tier reference arm: the CPU oracle as it stands, on the host cores."""
    if rank != 0:
        return
    import oracle
    from paper_2206_11535_b200.m3e import load_config
    cfg = load_config()
    P = oracle.make_params(cfg)
    cores = host_cores()
    sample = a.ref_frames * cores
    d, _ = generate(a.workload, sample * (a.steps + a.warmup), 0, a.seed)
    fr = oracle.Frames(d)
    times = []
    for s in range(a.warmup + a.steps):
        dt = time_oracle(P, fr, s * sample, sample, cores)
        if s >= a.warmup:
            times.append(dt)
    fps = sample / statistics.mean(times)
    v = gbps_equiv(fps, synth.preset(a.workload).muon_rate)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "Gbps", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 * statistics.mean(times), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT.get(a.workload, a.workload).format(F=a.frames),
                       "sample_frames_per_step": sample, "parallelism": f"{cores} host threads"},
            "cpu_baseline": {"value": round(v, 6), "unit": "Gbps", "cores": cores, "kind": "oracle",
                             "sample": f"{sample} frames per step (consecutive frames of the workload), fp64 C "
                                       f"oracle, {cores} threads on contiguous frame slices",
                             "frames_per_s": round(fps, 1)},
            "e2e": {"value": round(v, 6), "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--frames", type=int, default=int(PHASE1_FRAMES_PER_S), help="frames per GPU per step")
    ap.add_argument("--workload", default="phase1_sig", help="synth preset (phase1_sig, phase1_bg, phase2_stress)")
    ap.add_argument("--seed", type=int, default=20220623)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-frames", type=int, default=4000, help="oracle sample per step and host core")
    ap.add_argument("--cpu-sample", type=int, default=15000, help="oracle sample for cpu_baseline, per host core")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-phys", action="store_true", help="skip the truth-based efficiency sample")
    ap.add_argument("--phys-frames", type=int, default=200000)
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3) if a.impl == "b200" else a.warmup
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (rendezvous on
        # 127.0.0.1), which sets RANK / LOCAL_RANK / WORLD_SIZE for every rank
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank, world, local = dist_env()
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")

    if a.impl == "reference":
        run_reference(a, rank, world)
        return

    import torch
    from paper_2206_11535_b200 import m3e

    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    params = m3e.make_params(m3e.load_config())
    rate = synth.preset(a.workload).muon_rate

    # ---- this rank's second of phase-I data (distinct frame ids per rank)
    F = a.frames
    d, t_gen = generate(a.workload, F, rank * F, a.seed, world)
    H = len(d["x"])
    frames = m3e.DeviceFrames(d, device=dev)
    ctx = m3e.Context(local)
    trk_cap = (64 if a.workload.startswith("phase2") else 12) * F
    kept_cap = F if a.workload.startswith("phase2") else max(1024, F // 20)
    res = m3e.Result(F, H, track_capacity=trk_cap, kept_capacity=kept_cap, device=dev)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream(dev))   # inputs and output buffers were filled there
    in_bytes = 12 * H + 16 * F + 4

    def step():
        m3e.filter_device(ctx, params, frames.x, frames.y, frames.z, frames.offsets, F, H, res.outputs, stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    ctx.set_timing(True)   # CUDA events around each kernel of the path, on the launch stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = [s.elapsed_time(e) for s, e in ev]
    ms_step = statistics.mean(ms)
    ms_select, ms_fit, ms_tracks, ms_vertex, ms_filter, ms_pack = ctx.kernel_times()
    sm = res.summary_np()
    kept = int(sum(sm["kept_by_reason"][1:]))
    assert int(sm["frames"]) == F and not int(sm["overflow"]), "output capacity exceeded"
    out_bytes = (F * (1 + 16) + int(sm["tracks"]) * 32 + kept * (56 + 4 + 16) + int(sm["kept_hits"]) * 12)
    from paper_2206_11535_b200 import dist as m3dist
    counters = torch.tensor([F, H, kept, int(sm["tracks"]), int(sm["kept_hits"]), 0.0] +
                            [int(v) for v in sm["kept_by_reason"]], dtype=torch.float64, device=dev)
    # the only collectives (after the timed region): counters (sum), slowest rank's
    # step time (max), accepted global frame ids (gather)
    counters, t_max = m3dist.reduce_counters(counters, ms_step / 1e3)
    counters[5] = t_max * 1e6
    kept_ids = m3dist.gather_kept(res.kept_frame[:kept], rank * F)
    assert kept_ids.numel() == int(counters[2])
    tot_frames, tot_hits, tot_kept = float(counters[0]), float(counters[1]), float(counters[2])
    ms_max = float(counters[5]) / 1e3
    fps = tot_frames / (ms_max / 1e3)

    # ---- end to end through the public host API (H2D + filter + D2H per step)
    e2e = None
    if not a.no_e2e:
        pin = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().numpy()
        hx, hy, hz = (pin(np.concatenate([d[k], np.zeros(8, np.float32)])) for k in "xyz")
        hoff = pin(d["offsets"])
        # kept-frame capacities: ~0.4% of frames at phase I, most frames at phase II
        kc = F if a.workload.startswith("phase2") else max(1024, F // 20)
        kh = H + 8 if a.workload.startswith("phase2") else kc * 64
        h_reason = pin(np.zeros(F, np.uint8))
        h_kf = pin(np.zeros(kc, np.uint32))
        h_ko = pin(np.zeros(4 * kc + 1, np.uint32))
        h_kx, h_ky, h_kz = (pin(np.zeros(kh, np.float32)) for _ in range(3))
        h_v = pin(np.zeros(kc * 56, np.uint8))
        h_s = np.zeros(1, m3e.SUMMARY_DTYPE)
        hout = m3e.make_outputs(reason=h_reason, vertices=h_v, kept_frame=h_kf, kept_offsets=h_ko,
                                kept_capacity=kc, kept_x=h_kx, kept_y=h_ky, kept_z=h_kz,
                                kept_hit_capacity=kh, summary=h_s)
        hctx = m3e.Context(local, max_frames=1 << 20)
        m3e.filter_host(hctx, params, hx, hy, hz, hoff, F, hout)  # warm-up (allocations)
        tt = []
        for _ in range(a.e2e_steps):
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            m3e.filter_host(hctx, params, hx, hy, hz, hoff, F, hout)
            tt.append(time.perf_counter() - t)
        t_e2e = statistics.mean(tt)
        if world > 1:
            tm = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            t_e2e = float(tm)
        hkept = int(sum(h_s[0]["kept_by_reason"][1:]))
        assert hkept == kept, "host path disagrees with the device path"
        d2h = F + 96 + hkept * (4 + 16 + 56) + int(h_s[0]["kept_hits"]) * 12
        e2e = {"value": round(gbps_equiv(world * F / t_e2e, rate), 3), "unit": "Gbps", "h2d_bytes_per_step": in_bytes,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(1e3 * t_e2e, 3),
               "frames_per_s": round(world * F / t_e2e, 1)}
        hctx.close()

    # ---- physics figures on a sample with truth (rank 0; outside the timed region):
    # signal-track / signal-event efficiency of the CUDA path (synth/truth.py)
    phys = None
    if rank == 0 and not a.no_phys:
        from synth.truth import signal_efficiency
        n_e = min(F, a.phys_frames)
        de = synth.generate(synth.preset(a.workload, seed=a.seed), n_e, frame0=0, truth=True)
        re_ = m3e.run_filter(ctx, params, m3e.DeviceFrames(de, device=dev))
        torch.cuda.synchronize(dev)
        sme = re_.summary_np()
        phys = signal_efficiency(synth.preset(a.workload, seed=a.seed), de, re_.frames_np(n_e),
                                 re_.tracks_np(int(sme["track_slots"])), params.max_tracks)
        phys["sample_frames"] = n_e
        del re_, de

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        import oracle
        P = oracle.make_params(m3e.load_config())
        fr = oracle.Frames(d)
        cores = host_cores()
        n = min(a.cpu_sample * cores, F)
        dt = time_oracle(P, fr, 0, n, cores)
        cpu = {"value": round(gbps_equiv(n / dt, rate), 6), "unit": "Gbps", "cores": cores, "kind": "oracle",
               "sample": f"first {n} frames of the workload, fp64 C oracle, {cores} threads on contiguous "
                         f"frame slices",
               "frames_per_s": round(n / dt, 1)}

    if rank == 0:
        peak, peak_kind = load_peaks()
        clocks = clk.summary()
        prof, prof_file = load_profile(a.workload, F, a.seed)
        # instruction-issue peak: 148 SMs x 4 schedulers x 1 warp instruction per cycle at
        # the SM clock sampled during the timed region
        sm_mhz = clocks.get("sm_mhz") or 1965.0
        issue_peak = 148 * 4 * sm_mhz * 1e6 / 1e9   # G warp-instructions/s
        # the method's own bytes: hit stream in, final outputs out
        tracks = int(sm["tracks"])
        split = ms_select > 0
        big = H > 60 * F
        if split:
            names = [("select", "m3e::filter_kernel<SELECT_C, BIG=false>", ms_select, in_bytes),
                     ("fit", "m3e::fit_kernel", ms_fit, in_bytes + 32 * tracks),
                     ("vertex", "m3e::vertex_kernel+triple_kernel+vpost_kernel", ms_vertex, 0),
                     ("fused_spilled", "m3e::filter_kernel<FULL, BIG=false>", ms_filter, 0),
                     ("pack", "m3e::pack_kernel+kept_kernel", ms_pack, out_bytes - 32 * tracks)]   # (the fit writes the tracks)
        else:
            names = [("filter", "m3e::filter_kernel<FULL, BIG=%s>" % ("true" if big else "false"), ms_filter,
                      in_bytes + out_bytes), ("pack", "m3e::pack_kernel+kept_kernel", ms_pack, out_bytes)]
        per = {}
        for key, kn, kt, alg in names:
            e = {"ms": round(kt, 4), "share": round(kt / ms_step, 4), "method_bytes": int(alg)}
            kp = {}
            parts = kn.split("+")
            for part in parts:
                part = part if part.startswith("m3e::") else "m3e::" + part
                for k2, v2 in prof.get(part, {}).items():
                    if len(parts) == 1 or k2 in ("dram_read_bytes", "dram_write_bytes", "inst_executed"):
                        kp[k2] = kp.get(k2, 0) + v2
            if kp and kt > 0:
                e["dram_bytes"] = int(kp["dram_read_bytes"] + kp["dram_write_bytes"])
                e["dram_frac"] = round(e["dram_bytes"] / (kt / 1e3) / 1e9 / peak, 4)
                e["issue_frac"] = round(kp["inst_executed"] / (kt / 1e3) / 1e9 / issue_peak, 4)
                for pipe in ("alu", "fma", "xu", "lsu"):
                    if f"pipe_{pipe}_pct" in kp:
                        e[f"pipe_{pipe}_pct"] = round(kp[f"pipe_{pipe}_pct"], 1)
            if alg and kt > 0:
                e["method_frac"] = round(alg / (kt / 1e3) / 1e9 / peak, 4)
            per[key] = e
        # dominant kernel: the one taking the largest share of the step
        dom = max(names, key=lambda k: k[2])
        kname, kms, alg_bytes = dom[1], dom[2], dom[3]
        kp = prof.get(kname, {})
        traffic = (kp["dram_read_bytes"] + kp["dram_write_bytes"]) if "dram_read_bytes" in kp else None
        ie = kp.get("inst_executed")
        if ie:
            # bound by instruction issue (DRAM well below peak: see roofline.kernels)
            roof = {"bound": "issue", "achieved": round(ie / (kms / 1e3) / 1e9, 2), "peak": round(issue_peak, 2),
                    "unit": "G warp-inst/s", "frac": round(ie / (kms / 1e3) / 1e9 / issue_peak, 4),
                    "warp_inst_per_launch": int(ie)}
        else:
            roof = {"bound": "hbm", "achieved": round(alg_bytes / (kms / 1e3) / 1e9, 2), "peak": peak,
                    "unit": "GB/s", "frac": round(alg_bytes / (kms / 1e3) / 1e9 / peak, 4)}
        step_bytes = in_bytes + out_bytes
        roof.update({
            "traffic": traffic, "kernel": kname, "kernel_ms": round(kms, 4), "share_of_step": round(kms / ms_step, 4),
            "algorithmic_bytes_per_launch": int(alg_bytes),
            "hbm_frac_of_kernel": round(alg_bytes / (kms / 1e3) / 1e9 / peak, 4),
            "hbm_peak": peak, "peak_kind": peak_kind, "profile": prof_file,
            "step_hbm": {"method_bytes": int(step_bytes), "achieved": round(step_bytes / (ms_step / 1e3) / 1e9, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(step_bytes / (ms_step / 1e3) / 1e9 / peak, 4),
                         "dram_bytes_ncu": int(sum(v.get("dram_bytes", 0) for v in per.values())) if prof else None},
            "kernels": per, "candidates_per_frame": round(int(sm["candidates"]) / F, 3)})
        line = {
            "metric": METRIC, "value": round(gbps_equiv(fps, rate), 3), "unit": "Gbps", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT.get(a.workload, a.workload).format(F=F),
                       # headline: frames/s and the real-time factor (64 ns frames arrive at
                       # 15.625e6 frames/s); value = the same rate as Phase-I-equivalent Gbps
                       "realtime_factor": round(fps / PHASE1_FRAMES_PER_S, 3),
                       "realtime_factor_per_gpu": round(fps / (world * PHASE1_FRAMES_PER_S), 3),
                       "frames_per_s": round(fps, 1), "hits_per_s": round(tot_hits / ms_max * 1e3, 1),
                       "value_definition": "frames/s x 80 Gbps / 15.625e6 frames/s x (muon rate / 1e8): the "
                                           "paper's 80 Gbps Phase-I stream scaled by the real-time factor",
                       "hit_stream_gbps": round(8 * in_bytes * world / ms_max / 1e9 * 1e3, 3),
                       "frames": int(tot_frames), "hits": int(tot_hits),
                       "kept_frames": int(tot_kept),
                       "reduction_factor": round(tot_frames / tot_kept, 2) if tot_kept else None,
                       "kept_by_reason": {m3e.REASON_NAMES[i]: int(counters[6 + i]) for i in range(1, 6)},
                       "muon_rate": rate,
                       "l2": "inputs (%.2f GB) >> 126 MB L2, no flush needed" % (in_bytes / 1e9),
                       "parallelism": f"frame-sharded dp{world}", "generation_s": round(t_gen, 1),
                       "physics": phys},
            "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": (9 if split else 3) * a.steps, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
