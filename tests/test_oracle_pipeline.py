"""Pins of the oracle's frame pipeline (Alg. 1-4, Sec. V-B, Sec. VI):
brute-force enumeration on tiny frames, overflow rules, funnel invariants, and
the paper's printed efficiencies / rejection reproduced as toy-data bands."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _frames(hits_by_frame):
    xs, ys, zs, off = [], [], [], [0]
    for frame in hits_by_frame:
        for layer in frame:
            for h in layer:
                xs.append(h[0]); ys.append(h[1]); zs.append(h[2])
            off.append(len(xs))
    return oracle.Frames({"x": np.array(xs, np.float32), "y": np.array(ys, np.float32),
                          "z": np.array(zs, np.float32), "offsets": np.array(off, np.uint32)})


def test_paper_constants_in_config(cfg):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_constants.json")))
    assert cfg["cuts_max"] == g["cuts_max"]["value"]
    assert cfg["chi2_max"] == g["chi2_max"]["value"]
    assert cfg["target_r"] == g["target_r_mm"]["value"]
    assert cfg["b_field"] == g["b_field_T"]["value"]
    assert len(cfg["layer_r"]) == g["n_layers"]["value"]
    # 1 s of data at 64 ns frames over the 12-PC farm = 1.302e6 frames/s per PC
    per_pc = 1e9 / g["frame_ns"]["value"] / g["farm_pcs"]["value"]
    assert per_pc == pytest.approx(g["farm_frames_per_s_per_pc"]["value"], rel=1e-3)


@pytest.mark.parametrize("seed", range(20))
def test_selection_equals_brute_force_on_tiny_frames(P, cfg, seed):
    """Alg. 2: the survivor list is exactly the row-major list of combinations
    passing all four cuts (brute force over itertools.product with the cut
    predicates evaluated from the Eq. 2-5 definitions in numpy)."""
    rng = np.random.default_rng(seed)
    R = cfg["layer_r"]
    frame = []
    for layer in range(3):
        n = int(rng.integers(0, 6))
        ph = rng.uniform(-0.4, 0.4, size=n) + 1.0
        zz = rng.uniform(-30, 30, size=n)
        frame.append([(R[layer] * math.cos(a), R[layer] * math.sin(a), c) for a, c in zip(ph, zz)])
    frame.append([])
    fr = _frames([frame])
    cands, res = oracle.select(P, fr, 0)
    want = []
    for (i, a), (j, b), (k, c) in itertools.product(*[list(enumerate(frame[l])) for l in range(3)]):
        a, b, c = (np.array(fr.hit(0, l, ix)) for l, ix in ((0, i), (1, j), (2, k)))
        dl = (c[2] - b[2]) / (R[2] - R[1]) - (b[2] - a[2]) / (R[1] - R[0])
        c01 = a[:2] @ b[:2] / (R[0] * R[1])
        c12 = b[:2] @ c[:2] / (R[1] * R[2])
        m = np.array([[a[0], a[1], 1], [b[0], b[1], 1], [c[0], c[1], 1]])
        area2 = np.linalg.det(m)  # twice the signed area, = -cross_z of Eq. 5
        rt = abs(np.linalg.norm(a[:2] - b[:2]) * np.linalg.norm(b[:2] - c[:2]) *
                 np.linalg.norm(c[:2] - a[:2]) / (2 * area2)) if area2 != 0 else math.inf
        if (abs(dl) <= cfg["dlambda_max"] and c01 >= cfg["cos_phi01_min"] and c12 >= cfg["cos_phi12_min"]
                and cfg["rt_min"] <= rt <= cfg["rt_max"]):
            want.append((i, j, k))
    assert [(c.i0, c.i1, c.i2) for c in cands] == want
    n_all = len(frame[0]) * len(frame[1]) * len(frame[2])
    assert res.funnel[0] == n_all
    assert res.n_cand == len(want)


def test_funnel_and_stage_invariants(P):
    """Each cut passes at most what the previous one passed (Fig. 4), and any
    frame kept by a later step passed every earlier step."""
    d = synth.generate(synth.preset("phase1_sig", seed=4), 3000)
    fr = oracle.Frames(d)
    r = oracle.results_to_numpy(oracle.process_frames(P, fr))
    f = r["funnel"]
    assert np.all(f[:, :-1] >= f[:, 1:])
    assert np.all(r["n_cand"] == f[:, 4])
    assert np.all(r["n_fit"] == np.minimum(r["n_cand"], P.cuts_max))
    assert np.all(r["n_tracks"] <= r["n_fit"])
    v = r["reason"] == oracle.REASON_VERTEX
    assert v.sum() > 0
    assert np.all(r["n_cand"][v] >= 3) and np.all(r["n_tracks"][v] >= 3)
    assert np.all(r["n_pos"][v] >= 2) and np.all(r["n_neg"][v] >= 1) and np.all(r["n_combs"][v] >= 1)
    assert np.all(r["keep"] == (r["reason"] != oracle.REASON_NONE))
    # exactly once: reasons + discards = frames
    assert np.bincount(r["reason"], minlength=5).sum() == fr.n


def test_empty_and_degenerate_frames(P):
    one = [(23.3, 0.0, 0.0)]
    frames = [[[], [], [], []],                         # empty frame
              [one, [], [(73.9, 0, 0)], [(86.3, 0, 0)]],  # empty layer 1
              [one, [(29.8, 0, 0)], [(73.9, 0, 0)], []]]  # collinear triplet (r_tc infinite)
    fr = _frames(frames)
    for f in range(3):
        res, tracks = oracle.process_frame(P, fr, f)
        assert res.reason == oracle.REASON_NONE and not res.keep
        assert res.n_cand == 0 and tracks == []


def test_triplet_overflow(P, cfg):
    """Sec. VI: more than 768 surviving hit triplets -> frame kept, rest skipped;
    the enumeration stops at 769 (reading R3)."""
    rng = np.random.default_rng(1)
    R = cfg["layer_r"]
    # a dense bundle of curved tracks: 12 x 12 x 12 = 1728 combinations, most passing
    frame = []
    for layer in range(4):
        pts = []
        for _ in range(12):
            ph = 0.3 + (R[layer] / (2 * 80.0)) + rng.normal() * 1e-3
            pts.append((R[layer] * math.cos(ph), R[layer] * math.sin(ph), rng.normal() * 0.5))
        frame.append(pts)
    fr = _frames([frame])
    res, tracks = oracle.process_frame(P, fr, 0)
    assert res.n_cand == cfg["cuts_max"] + 1
    assert res.reason == oracle.REASON_TRIPLET_OVERFLOW and res.keep and tracks == []
    assert res.n_fit == 0


def test_determinism(P):
    d1 = synth.generate(synth.preset("phase1_sig", seed=77), 500)
    d2 = synth.generate(synth.preset("phase1_sig", seed=77), 500, threads=3)
    for k in ("x", "y", "z", "offsets"):
        assert np.array_equal(d1[k], d2[k])
    r1 = oracle.results_to_numpy(oracle.process_frames(P, oracle.Frames(d1)))
    r2 = oracle.results_to_numpy(oracle.process_frames(P, oracle.Frames(d2)))
    for k in r1:
        assert np.array_equal(r1[k], r2[k])


def _true_hits(d, f):
    out = {}
    hp, off = d["hit_particle"], d["offsets"]
    for layer in range(4):
        for g in range(int(off[4 * f + layer]), int(off[4 * f + layer + 1])):
            if hp[g] >= 0:
                out.setdefault(int(hp[g]), {})[layer] = g - int(off[4 * f + layer])
    return out


@pytest.mark.slow
def test_paper_selection_figures(P):
    """Sec. IV-A / Fig. 4 on toy data (fresh seed, not the tuning sample):
    > 98.5% of true (reconstructible) triplets kept, > 95% of combinations
    removed, first cut (Delta lambda) alone removes > 80%."""
    d = synth.generate(synth.preset("phase1_bg", seed=424242), 2500, truth=True)
    fr = oracle.Frames(d)
    funnel = np.zeros(5)
    n_true = kept = 0
    for f in range(fr.n):
        cands, res = oracle.select(P, fr, f)
        funnel += np.array(list(res.funnel), float)
        want = {(l[0], l[1], l[2]) for l in _true_hits(d, f).values() if len(l) == 4}
        got = {(c.i0, c.i1, c.i2) for c in cands}
        n_true += len(want)
        kept += len(want & got)
    assert kept / n_true > 0.985
    assert funnel[4] / funnel[0] < 0.05
    assert funnel[1] / funnel[0] < 0.20


@pytest.mark.slow
def test_paper_track_and_signal_efficiency(P):
    """Sec. VI-A on toy data: > 97% of reconstructible signal tracks are found
    (paper: "over 97% of tracks from signal particles").  Frames whose three
    signal particles are reconstructible are identified in > 88% of cases on the
    toy (paper: > 94% on Geant4); the gap is the paper's own rule "If two circles
    do not intersect, the track triplet is skipped"."""
    sc = synth.preset("signal_only", seed=515)
    n = 2500
    d = synth.generate(sc, n, truth=True)
    fr = oracle.Frames(d)
    trk_tot = trk_ok = frm_tot = frm_ok = 0
    for f in range(n):
        parts = synth.particles(sc, f)
        th = _true_hits(d, f)
        res, tracks = oracle.process_frame(P, fr, f)
        found = {(t.hit[0], t.hit[1], t.hit[2], t.hit[3]): t for t in tracks}
        allrec = True
        for pid, p in enumerate(parts):
            if p["layer_mask"] != 15:
                allrec = False
                continue
            trk_tot += 1
            h = th[pid]
            t = found.get((h[0], h[1], h[2], h[3]))
            if t is not None and (t.kappa > 0) == (p["charge"] > 0):
                trk_ok += 1
        if allrec:
            frm_tot += 1
            frm_ok += int(res.keep and res.reason == oracle.REASON_VERTEX)
    assert trk_ok / trk_tot > 0.97
    assert frm_ok / frm_tot > 0.88


@pytest.mark.slow
def test_paper_reduction_factor(P):
    """Abstract / Sec. VI-B: at 1e8 mu/s the data rate is reduced by > 100
    (frames kept < 1%), with signal injected in 1% of frames."""
    d = synth.generate(synth.preset("phase1_sig", seed=616), 6000)
    r = oracle.results_to_numpy(oracle.process_frames(P, oracle.Frames(d)))
    assert r["keep"].mean() < 0.01


def test_signal_event_loss_attribution(P):
    """Known gap, attributed: north_star asks for >= 94%
    of signal events; the oracle keeps ~90.5% of frames whose three mu->eee
    daughters are reconstructible.  tools/efficiency_study.py follows the TRUE
    triple through Alg. 2-4: ~5% of frames are lost to the paper's rule "If two
    circles do not intersect, the track triplet is skipped" (Sec. IV-C; the
    daughters' circles miss by ~0.2 mm after layer-0 scattering), and lifting
    that one rule (the two circles made tangent, everything else the oracle's)
    brings the same frames to >= 93.5%."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "efficiency_study", os.path.join(ROOT, "tools", "efficiency_study.py"))
    es = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(es)
    sc = synth.preset("signal_only", seed=9101)
    n = 8000
    d = synth.generate(sc, n, truth=True)
    fr = oracle.Frames(d)
    tot = kept = lifted = no_int = 0
    for f in range(n):
        r = es.classify(P, fr, d, sc, f)
        if r is None:
            continue
        tot += 1
        (cause, det), _, tracks, tri = r
        kept += cause == "kept"
        if cause == "no_intersect":
            no_int += 1
            lifted += es.lift_no_intersect(P, fr, f, tracks, tri)
    assert 0.87 <= kept / tot <= 0.93
    assert 0.03 <= no_int / tot <= 0.07
    assert (kept + lifted) / tot >= 0.935
