"""Parity at BASELINE.json's full size, in the launch configuration bench.py
times: configs[3] (one second of phase-I data, 15 625 000 frames, the bench's
seed), checked against the oracle on sampled frames (uniform sample + every kept
frame) and by properties that hold at any size; and configs[4] (1e9 mu/s)."""
import numpy as np
import pytest

import oracle
import synth
from parity import check_track_layout, compare_outputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2206_11535_b200 import m3e  # noqa: E402

BENCH_SEED = 20220623   # bench.py --seed default
FRAMES_1S = 15_625_000  # one second of 64 ns frames


def _check_frames(P, fr, res, frames_np, tracks_np, sample, name):
    """sampled frames against the oracle, item by item (tests/parity.py)"""
    K = int(np.count_nonzero(frames_np["reason"]))
    tally = compare_outputs(P, fr, frames_np, tracks_np, res.vertices_np(K), sample)
    print(tally.report(f"{name}: {len(sample)} sampled frames"))
    return tally


def _run(ctx, gp, d, track_cap, kept_cap):
    df = m3e.DeviceFrames(d)
    res = m3e.Result(df.n_frames, df.n_hits, track_capacity=track_cap, kept_capacity=kept_cap)
    m3e.run_filter(ctx, gp, df, res)
    torch.cuda.synchronize()
    return df, res


@pytest.mark.slow
def test_fullsize_phase1_second(cfg):
    gp, P = m3e.make_params(cfg), oracle.make_params(cfg)
    d = synth.generate(synth.preset("phase1_sig", seed=BENCH_SEED), FRAMES_1S)
    F, H = FRAMES_1S, len(d["x"])
    ctx = m3e.Context(0)
    df, res = _run(ctx, gp, d, 12 * F, max(1024, F // 20))   # bench.py's capacities
    sm = res.summary_np()
    assert int(sm["frames"]) == F and not int(sm["overflow"])
    reason = res.reason.cpu().numpy()
    frames_np = res.frames_np(F)
    T = int(sm["tracks"])
    tracks_np = res.tracks_np(int(sm["track_slots"]))
    # properties at any size
    assert np.array_equal(reason, frames_np["reason"])
    assert np.array_equal(np.bincount(reason, minlength=6), sm["kept_by_reason"])
    ntr = np.minimum(frames_np["n_tracks"].astype(np.int64), P.max_tracks)
    ntr[frames_np["reason"] == m3e.REASON_TRIPLET_OVERFLOW] = 0
    assert int(ntr.sum()) == T
    check_track_layout(P, frames_np, tracks_np, sm)
    kept = np.nonzero(reason)[0]
    K = len(kept)
    assert np.array_equal(res.kept_frame[:K].cpu().numpy().view(np.uint32).astype(np.int64), kept)
    kf = frames_np["kept_index"]
    assert np.array_equal(kf[kept], np.arange(K, dtype=np.uint32))
    assert F / K > 100   # reduction factor (paper: > 100)
    # sampled parity: 2500 uniform frames + 1500 kept frames
    rng = np.random.default_rng(1)
    sample = np.unique(np.concatenate([rng.integers(0, F, 2500), rng.choice(kept, min(K, 1500), replace=False)]))
    fr = oracle.Frames(d)
    tally = _check_frames(P, fr, res, frames_np, tracks_np, sample, "configs[3] full size")
    assert len(tally.frames) <= max(2, 2e-3 * len(sample))
    assert tally.counts().get("_vertex_compared", 0) > 100
    # packed kept frames: verbatim hits of sampled kept frames
    koff = res.kept_offsets[:4 * K + 1].cpu().numpy().view(np.uint32).astype(np.int64)
    kz = res.kept_z.cpu().numpy()
    off = d["offsets"].astype(np.int64)
    for k in rng.choice(K, min(K, 200), replace=False):
        f = kept[k]
        n = off[4 * f + 4] - off[4 * f]
        assert np.array_equal(kz[koff[4 * k]:koff[4 * k] + n], d["z"][off[4 * f]:off[4 * f + 4]])
    ctx.close()


def test_phase2_sampled(cfg):
    """configs[4] (1e9 mu/s, ~223 hits per frame: warp-batches of one frame,
    staging windows overflow into HBM reads) on 20 000 frames, 400 sampled."""
    gp, P = m3e.make_params(cfg), oracle.make_params(cfg)
    n = 20000
    d = synth.generate(synth.preset("phase2_stress", seed=777), n)
    ctx = m3e.Context(0)
    df, res = _run(ctx, gp, d, 64 * n, n)
    sm = res.summary_np()
    assert not int(sm["overflow"])
    frames_np = res.frames_np(n)
    tracks_np = res.tracks_np(int(sm["track_slots"]))
    sample = np.random.default_rng(2).choice(n, 400, replace=False)
    tally = _check_frames(P, oracle.Frames(d), res, frames_np, tracks_np, sample, "configs[4]")
    assert len(tally.frames) <= max(2, 5e-3 * len(sample))
    ctx.close()
