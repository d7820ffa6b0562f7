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


def load_profile(workload: str, frames: int, seed: int):
    """Per-kernel ncu counters (DRAM bytes, executed warp instructions per launch)
    of the committed capture of this exact configuration
    (profiles/*_bench_traffic.json), else {}."""
    import glob
    for fn in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_bench_traffic.json")), reverse=True):
        try:
            t = json.load(open(fn))
        except Exception:
            continue
        if t.get("workload") == workload and t.get("frames") == frames and t.get("seed") == seed:
            return t.get("kernels", {})
    return {}


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


def run_reference(a, rank, world):
    """Tier reference arm: the CPU oracle as it stands, on the host cores."""
    if rank != 0:
        return
    import oracle
    from paper_2206_11535_b200.m3e import load_config
    cfg = load_config()
    P = oracle.make_params(cfg)
    sample = a.ref_frames
    d, _ = generate(a.workload, sample * (a.steps + a.warmup), 0, a.seed)
    fr = oracle.Frames(d)
    times = []
    for s in range(a.warmup + a.steps):
        t = time.perf_counter()
        oracle.process_frames(P, fr, first=s * sample, count=sample)
        dt = time.perf_counter() - t
        if s >= a.warmup:
            times.append(dt)
    fps = sample / statistics.mean(times)
    v = gbps_equiv(fps, synth.preset(a.workload).muon_rate)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "Gbps", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 * statistics.mean(times), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT.get(a.workload, a.workload).format(F=a.frames),
                       "sample_frames_per_step": sample, "parallelism": "single core"},
            "cpu_baseline": {"value": round(v, 6), "unit": "Gbps", "cores": 1, "kind": "oracle",
                             "sample": f"{sample} frames per step, single-threaded fp64 C oracle",
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
    ap.add_argument("--ref-frames", type=int, default=4000, help="oracle sample per step")
    ap.add_argument("--cpu-sample", type=int, default=15000, help="oracle sample for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-phys", action="store_true", help="skip the truth-based efficiency sample")
    ap.add_argument("--phys-frames", type=int, default=200000)
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3) if a.impl == "b200" else a.warmup
    rank, world, local = dist_env()

    if a.impl == "reference":
        run_reference(a, rank, world)
        return

    import torch
    from paper_2206_11535_b200 import m3e

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
        kc = max(1024, F // 20)
        h_reason = pin(np.zeros(F, np.uint8))
        h_kf = pin(np.zeros(kc, np.uint32))
        h_ko = pin(np.zeros(4 * kc + 1, np.uint32))
        h_kx, h_ky, h_kz = (pin(np.zeros(kc * 64, np.float32)) for _ in range(3))
        h_v = pin(np.zeros(kc * 56, np.uint8))
        h_s = np.zeros(1, m3e.SUMMARY_DTYPE)
        hout = m3e.make_outputs(reason=h_reason, vertices=h_v, kept_frame=h_kf, kept_offsets=h_ko,
                                kept_capacity=kc, kept_x=h_kx, kept_y=h_ky, kept_z=h_kz,
                                kept_hit_capacity=kc * 64, summary=h_s)
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
                                 re_.tracks_np(int(sme["tracks"])), params.max_tracks)
        phys["sample_frames"] = n_e
        del re_, de

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        import oracle
        P = oracle.make_params(m3e.load_config())
        fr = oracle.Frames(d)
        n = min(a.cpu_sample, F)
        t = time.perf_counter()
        oracle.process_frames(P, fr, first=0, count=n)
        dt = time.perf_counter() - t
        cpu = {"value": round(gbps_equiv(n / dt, rate), 6), "unit": "Gbps", "cores": 1, "kind": "oracle",
               "sample": f"first {n} frames of the workload, single-threaded fp64 C oracle",
               "frames_per_s": round(n / dt, 1)}

    if rank == 0:
        peak, peak_kind = load_peaks()
        # algorithmic bytes per launch:
        #   selection kernel: hit stream in, selection words (4 B/frame) + store entries (16 B) out
        #   fit kernel: store entries + the candidates' frames (hit stream) in, fit records (32 B) out
        #   tracks kernel: selection words + code bytes (1 B per entry) in, track words out
        #   vertex kernel: the listed frames' fit records + hits in (~1% of frames), small
        #   finish kernel (+ the fused kernel over spilled warp-batches, ~0): selection
        #   and track words in, per-frame outputs, kept records out
        #   (fused path: one kernel, hit stream in + outputs)
        split = ms_select > 0
        cand = int(sm["candidates"])
        big = H > 60 * F
        if split:
            kernels = [("m3e::filter_kernel<SELECT_C, BIG=false>", ms_select, in_bytes + 4 * F + 16 * cand),
                       ("m3e::fit_kernel", ms_fit, in_bytes + 16 * cand + 32 * cand),
                       ("m3e::tracks_kernel", ms_tracks, 4 * F + cand + 4 * F),
                       ("m3e::finish_kernel", ms_filter, 8 * F + F * (1 + 16) + kept * 64)]
        else:
            kernels = [("m3e::filter_kernel<FULL, BIG=%s>" % ("true" if big else "false"), ms_filter,
                        in_bytes + out_bytes)]
        kname, kms, alg_bytes = max(kernels, key=lambda k: k[1])
        achieved = alg_bytes / (kms / 1e3) / 1e9
        clocks = clk.summary()
        prof = load_profile(a.workload, F, a.seed)
        kp = prof.get(kname, {})
        traffic = (kp["dram_read_bytes"] + kp["dram_write_bytes"]) if "dram_read_bytes" in kp else None
        # instruction-issue roofline of the two issue-bound kernels:
        # warp instructions per launch (ncu, committed capture of this configuration) over
        # the live kernel time, against 148 SMs x 4 schedulers x 1 warp-instruction/cycle
        # at the sampled SM clock
        sm_mhz = clocks.get("sm_mhz") or 1965.0
        issue_peak = 148 * 4 * sm_mhz * 1e6 / 1e9   # G warp-instructions/s
        issue = {}
        for key, kn, kt in (("select", "m3e::filter_kernel<SELECT_C, BIG=false>", ms_select),
                            ("fit", "m3e::fit_kernel", ms_fit)):
            ie = prof.get(kn, {}).get("inst_executed")
            if ie and kt > 0:
                ach = ie / (kt / 1e3) / 1e9
                issue[key] = {"warp_inst_per_launch": int(ie), "achieved": round(ach, 1), "peak": round(issue_peak, 1),
                              "unit": "G warp-inst/s", "frac": round(ach / issue_peak, 4)}
        line = {
            "metric": METRIC, "value": round(gbps_equiv(fps, rate), 3), "unit": "Gbps", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT.get(a.workload, a.workload).format(F=F),
                       "frames": int(tot_frames), "hits": int(tot_hits),
                       "frames_per_s": round(fps, 1), "hits_per_s": round(tot_hits / ms_max * 1e3, 1),
                       "hit_stream_gbps": round(8 * in_bytes * world / ms_max / 1e9 * 1e3, 3),
                       "kept_frames": int(tot_kept),
                       "reduction_factor": round(tot_frames / tot_kept, 2) if tot_kept else None,
                       "kept_by_reason": {m3e.REASON_NAMES[i]: int(counters[6 + i]) for i in range(1, 6)},
                       "realtime_factor": round(fps / (world * PHASE1_FRAMES_PER_S), 3),
                       "muon_rate": rate,
                       "l2": "inputs (%.2f GB) >> 126 MB L2, no flush needed" % (in_bytes / 1e9),
                       "parallelism": f"frame-sharded dp{world}", "generation_s": round(t_gen, 1),
                       "physics": phys},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": traffic, "peak_kind": peak_kind, "issue": issue or None,
                         "kernel": kname, "kernel_ms": round(kms, 4), "share_of_step": round(kms / ms_step, 4),
                         "algorithmic_bytes_per_launch": int(alg_bytes),
                         "kernels_ms": {"select": round(ms_select, 4), "fit": round(ms_fit, 4),
                                        "tracks": round(ms_tracks, 4), "vertex": round(ms_vertex, 4),
                                        "finish": round(ms_filter, 4), "pack": round(ms_pack, 4)},
                         "candidates_per_frame": round(cand / F, 3)},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": (9 if split else 2) * a.steps, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
