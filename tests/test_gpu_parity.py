"""GPU parity of the CUDA path (libm3e.so, called through its C ABI) against the
fp64 CPU oracle on the same seeded frames.  Stage-isolated
tests feed both sides identical inputs; the end-to-end test compares whole
frames and explains every difference by a near-threshold decision."""
import math

import numpy as np
import pytest

import oracle
import synth
from parity import (CHI2_DOMAIN, check_track_layout, REL_KAPPA, Tally, chi2_marginal, combo_is_marginal, compare_outputs, layer3_tie,
                    near, rel_close, unpack)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2206_11535_b200 import m3e  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = m3e.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def gp(cfg):
    return m3e.make_params(cfg)


def _gen(name, n, seed):
    d = synth.generate(synth.preset(name, seed=seed), n)
    return d, oracle.Frames(d), m3e.DeviceFrames(d)


# ------------------------------------------------------------------ selection
@pytest.mark.parametrize("name,n,seed", [("phase1_sig", 3000, 101), ("phase2_stress", 120, 102),
                                         ("single_frame", 1, 103), ("phase1_bg", 65, 104)])
def test_selection_parity(ctx, gp, P, name, n, seed):
    d, fr, df = _gen(name, n, seed)
    C = P.cuts_max
    cand = torch.zeros(n * C, dtype=torch.int32, device="cuda")
    crt = torch.zeros(n * C, dtype=torch.float32, device="cuda")
    frames = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    m3e.select_triplets(ctx, gp, df.x, df.y, df.z, df.offsets, n, df.n_hits, cand, crt, frames)
    torch.cuda.synchronize()
    fo = frames.cpu().numpy().view(m3e.FRAME_DTYPE)
    cand, crt = cand.cpu().numpy(), crt.cpu().numpy()
    n_marg = n_cmp = 0
    Pbig = oracle.make_params(dict(m3e.load_config(), cuts_max=1 << 30))
    for f in range(n):
        oc, res = oracle.select(P, fr, f)
        ncg = int(fo["n_cand"][f])
        if res.n_cand > C or ncg > C:  # overflow frames store nothing: only the decision is compared
            if (res.n_cand > C) != (ncg > C):
                # the flip needs marginal combinations across the cap: N survivors in all,
                # m of all combinations within the band of a cut threshold
                _, full = oracle.select(Pbig, fr, f, cap=1)
                N, m = full.n_cand, full.n_cand_marginal
                assert (N - m <= C) if N > C else (N + m > C), (f, N, m, ncg)
                n_marg += 1
            continue
        g = [unpack(c) for c in cand[f * C:f * C + min(ncg, C)]]
        o = [(c.i0, c.i1, c.i2) for c in oc]
        if g != o:
            for t in set(g) ^ set(o):
                assert combo_is_marginal(P, fr, f, *t), (f, t)
                n_marg += 1
            assert [t for t in g if t in set(o)] == [t for t in o if t in set(g)]  # order kept
        else:
            assert ncg == res.n_cand
            for k, c in enumerate(oc):  # cached r_tc (Eq. 5)
                assert rel_close(float(crt[f * C + k]), c.rtc, 1e-5), (f, k)
        n_cmp += len(o)
    print(f"{name}: {n_cmp} candidates compared, {n_marg} near-threshold items")
    assert n_marg <= max(2, 1e-3 * n_cmp)


# ------------------------------------------------------------------------ fit
@pytest.mark.parametrize("name,n,seed", [("phase1_sig", 2000, 201), ("signal_only", 800, 202),
                                         ("phase2_stress", 40, 203)])
def test_fit_parity(ctx, gp, P, name, n, seed):
    """Stage (d) on the ORACLE's candidates: every fit matches the oracle's
    (curvatures within 1e-4 relative, decisions exact unless near a threshold)."""
    d, fr, df = _gen(name, n, seed)
    C, T = P.cuts_max, P.max_tracks
    cand = np.zeros(n * C, np.uint32)
    crt = np.zeros(n * C, np.float32)
    ncand = np.zeros(n, np.uint16)
    ocands = []
    for f in range(n):
        oc, res = oracle.select(P, fr, f)
        ocands.append(oc)
        ncand[f] = min(res.n_cand, C + 1)
        for k, c in enumerate(oc):
            cand[f * C + k] = c.i0 | (c.i1 << 10) | (c.i2 << 20)
            crt[f * C + k] = c.rtc
    dev = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda()
    rec = torch.zeros(n * C * 40, dtype=torch.uint8, device="cuda")
    trk = torch.zeros(n * T * 32, dtype=torch.uint8, device="cuda")
    frames = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    nc_t = torch.from_numpy(ncand.view(np.int16)).cuda()
    m3e.fit_tracks(ctx, gp, df.x, df.y, df.z, df.offsets, n, df.n_hits, dev(cand), dev(crt), nc_t, rec, trk,
                   frames)
    torch.cuda.synchronize()
    rec = rec.cpu().numpy().view(m3e.FIT_DTYPE)
    n_fit = 0
    tally = Tally()
    worst = 0.0
    chi2_dev = []
    for f in range(n):
        if ncand[f] > C:
            continue
        for k, c in enumerate(ocands[f]):
            o = oracle.fit_candidate(P, fr, f, c)
            g = rec[f * C + k]
            n_fit += 1
            gs = int(g["status"])
            # layer-3 hit (R10) of every fit that reached the search: equal unless the
            # oracle's closest and second-closest hits are within the band
            if o.status not in (oracle.FIT_DEGENERATE1, oracle.FIT_NO_REACH, oracle.FIT_LAYER3_EMPTY) and \
                    gs not in (oracle.FIT_DEGENERATE1, oracle.FIT_NO_REACH, oracle.FIT_LAYER3_EMPTY):
                if int(g["hit3"]) != o.hit[3]:
                    assert layer3_tie(P, fr, f, o), (f, k, int(g["hit3"]), o.hit[3])
                    tally.add(f, "hit3_tie", k)
                    continue
            if o.status in (oracle.FIT_OK, oracle.FIT_CHI2) and 10.0 <= o.chi2 <= 100.0 and \
                    gs in (oracle.FIT_OK, oracle.FIT_CHI2):
                chi2_dev.append(abs(float(g["chi2"]) - o.chi2) / o.chi2)
            if gs != o.status:
                assert chi2_marginal(P, o) and {gs, o.status} == {oracle.FIT_OK, oracle.FIT_CHI2}, \
                    (f, k, gs, o.status, float(g["chi2"]), o.chi2)
                tally.add(f, "chi2", k)
                continue
            # curvatures / chi2 compared wherever the linearised model is in its domain:
            # chi2_global < 1000 (every fit the chi2 < 32 cut could accept, with a 30x
            # margin); beyond, only the reject decision is compared
            if o.status in (oracle.FIT_OK, oracle.FIT_CHI2) and o.chi2 < CHI2_DOMAIN:
                for a, b in [(g["kappa1"], o.t1.kappa), (g["kappa2"], o.t2.kappa), (g["kappa"], o.kappa)]:
                    worst = max(worst, abs(a - b) / abs(b))
                    assert rel_close(float(a), b, REL_KAPPA), (f, k, float(a), b, o.chi2)
                assert rel_close(float(g["var1"]), o.t1.var_kappa, 1e-3)
                assert abs(float(g["chi2"]) - o.chi2) <= 1e-3 * max(o.chi2, 1.0), (f, k, float(g["chi2"]), o.chi2)
            if o.status == oracle.FIT_OK:
                assert abs(float(g["cos_theta01"]) - o.cos_theta01) <= 1e-4
                assert math.hypot(float(g["cx"]) - o.cx, float(g["cy"]) - o.cy) <= 1e-4 * o.rt
    assert n_fit > 0
    chi2_dev = np.array(chi2_dev) if chi2_dev else np.zeros(1)
    print(f"{name}: {n_fit} fits, worst kappa rel diff {worst:.2e}, chi2 in [10, 100]: rel diff max "
          f"{chi2_dev.max():.2e} p99 {np.quantile(chi2_dev, 0.99):.2e}; {tally.report()}")
    assert len(tally) <= max(2, 1e-3 * n_fit)


# --------------------------------------------------------------------- vertex
def _float_tracks(P, fr, f, tracks):
    """oracle tracks rounded to the float32 fields of m3e_track"""
    out = []
    for t in tracks:
        out.append(dict(kappa=np.float32(t.kappa), cos_theta01=np.float32(t.cos_theta01),
                        cx=np.float32(t.cx), cy=np.float32(t.cy), hit=list(t.hit), chi2=np.float32(t.chi2)))
    return out


@pytest.mark.parametrize("name,n,seed", [("signal_only", 1500, 301), ("phase1_sig", 3000, 302)])
def test_vertex_parity(ctx, gp, P, name, n, seed):
    """Stage (e) on identical (float32) tracks: fp64 on both sides, so decisions
    and vertices agree to rounding."""
    d, fr, df = _gen(name, n, seed)
    T = P.max_tracks
    trk = np.zeros(n * T, m3e.TRACK_DTYPE)
    ntrk = np.zeros(n, np.uint16)
    want = []
    for f in range(n):
        res, tracks = oracle.process_frame(P, fr, f)
        if res.n_tracks > T or res.reason in (oracle.REASON_TRIPLET_OVERFLOW, oracle.REASON_TRACK_OVERFLOW):
            want.append(None)
            continue
        ft = _float_tracks(P, fr, f, tracks)
        ntrk[f] = len(ft)
        vt = []
        for k, t in enumerate(ft):
            i = f * T + k
            trk["frame"][i] = f
            trk["hit"][i] = t["hit"]
            for key in ("kappa", "chi2", "cos_theta01", "cx", "cy"):
                trk[key][i] = t[key]
            vt.append(oracle.VTrack(float(t["kappa"]), float(t["cos_theta01"]), float(t["cx"]), float(t["cy"]),
                                    fr.hit(f, 0, t["hit"][0])))
        want.append(oracle.vertex_frame(P, vt)[0])
    g_trk = torch.from_numpy(trk.view(np.uint8)).cuda()
    g_n = torch.from_numpy(ntrk.view(np.int16)).cuda()
    frames = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    vtx = torch.zeros(n * 56, dtype=torch.uint8, device="cuda")
    m3e.vertex_select(ctx, gp, df.x, df.y, df.z, df.offsets, n, df.n_hits, g_trk, g_n, frames, vtx)
    torch.cuda.synchronize()
    fo = frames.cpu().numpy().view(m3e.FRAME_DTYPE)
    vo = vtx.cpu().numpy().view(m3e.VERTEX_DTYPE)
    n_v = 0
    for f in range(n):
        w = want[f]
        if w is None:
            continue
        assert int(fo["n_combs"][f]) == w.n_combs, f
        # fp64 on both sides on identical float32 tracks: decisions exact
        assert int(fo["reason"][f]) == (w.reason if w.keep else 0), (f, int(fo["reason"][f]), w.reason)
        if w.reason == oracle.REASON_VERTEX and int(fo["reason"][f]) == w.reason:
            v = vo[f]
            n_v += 1
            assert (int(v["track"][0]), int(v["track"][1]), int(v["track"][2])) == (w.vertex.a, w.vertex.b, w.vertex.e)
            for a, b in [(v["x"], w.vertex.x), (v["y"], w.vertex.y), (v["z"], w.vertex.z)]:
                assert abs(float(a) - b) <= 1e-9 * max(1.0, abs(b))
            assert rel_close(float(v["chi2"]), w.vertex.chi2, 1e-9, 1e-12)
    assert n_v > 0


# ---------------------------------------------------------------- end to end
def _compare_full(P, fr, res, n, name=""):
    """every frame of one m3e_filter call against the oracle, item by item
    (tests/parity.py); returns the tally of near-threshold items"""
    sm = res.summary_np()
    K = int(sum(sm["kept_by_reason"][1:]))
    check_track_layout(P, res.frames_np(n), res.tracks_np(int(sm["track_slots"])), sm)
    tally = compare_outputs(P, fr, res.frames_np(n), res.tracks_np(int(sm["track_slots"])), res.vertices_np(K),
                            range(n))
    print(tally.report(name))
    return tally


@pytest.mark.parametrize("name,n,seed", [("phase1_sig", 4000, 401), ("signal_only", 1000, 402),
                                         ("phase2_stress", 150, 403), ("single_frame", 1, 404),
                                         ("phase1_bg", 129, 405)])
def test_full_parity(ctx, gp, P, name, n, seed):
    d, fr, df = _gen(name, n, seed)
    res = m3e.run_filter(ctx, gp, df)
    torch.cuda.synchronize()
    sm = res.summary_np()
    assert int(sm["overflow"]) == 0
    frames_np = res.frames_np(n)
    tracks_np = res.tracks_np(int(sm["track_slots"]))
    tally = _compare_full(P, fr, res, n, name)
    assert len(tally.frames) <= max(1, 2e-3 * n)
    if name in ("phase1_sig", "signal_only"):
        assert tally.counts().get("_vertex_compared", 0) > 0
    # summary consistency and the reason bytes
    reason = res.reason.cpu().numpy()[:n]
    assert np.array_equal(reason, frames_np["reason"])
    assert int(sm["frames"]) == n
    assert np.array_equal(np.bincount(reason, minlength=6), sm["kept_by_reason"])
    # packed kept frames are the input frames, verbatim and in order
    kept = np.nonzero(reason)[0]
    K = len(kept)
    assert np.array_equal(res.kept_frame.cpu().numpy()[:K], kept)
    koff = res.kept_offsets.cpu().numpy()[:4 * K + 1].astype(np.int64)
    kx = res.kept_x.cpu().numpy()
    off = d["offsets"].astype(np.int64)
    assert koff[4 * K] == int(sm["kept_hits"]) if K else True
    for k, f in enumerate(kept):
        lo, hi = off[4 * f], off[4 * f + 4]
        assert np.array_equal(koff[4 * k:4 * k + 4] - koff[4 * k], off[4 * f:4 * f + 4] - lo)
        assert np.array_equal(kx[koff[4 * k]:koff[4 * k] + (hi - lo)], d["x"][lo:hi])
    # frame-ordered tracks with unused slots (m3e.h m3e_outputs.tracks)
    check_track_layout(P, frames_np, tracks_np, sm)


@pytest.mark.parametrize("fused", ["0", "1"])
def test_track_overflow_parity(cfg, monkeypatch, fused):
    """max_tracks = 2: most frames with tracks overflow (R3), so the capped
    track lists go through the staged path of the finish and pack kernels."""
    c2 = dict(cfg, max_tracks=2)
    gp2, P2 = m3e.make_params(c2), oracle.make_params(c2)
    monkeypatch.setenv("M3E_FUSED", fused)
    c = m3e.Context(0)
    n = 3000
    d, fr, df = _gen("phase1_sig", n, 801)
    res = m3e.run_filter(c, gp2, df)
    torch.cuda.synchronize()
    sm = res.summary_np()
    assert int(sm["overflow"]) == 0
    frames_np = res.frames_np(n)
    assert int(np.count_nonzero(frames_np["reason"] == m3e.REASON_TRACK_OVERFLOW)) > n // 4
    tally = _compare_full(P2, fr, res, n, "max_tracks=2")
    assert len(tally.frames) <= max(1, 2e-3 * n)
    c.close()


def _outputs(res, n):
    sm = res.summary_np()
    T, K = int(sm["track_slots"]), int(sum(sm["kept_by_reason"][1:]))
    return (res.reason.cpu().numpy()[:n].copy(), res.frames_np(n).copy(), res.tracks_np(T).copy(),
            res.kept_frame.cpu().numpy()[:K].copy(), res.vertices_np(K).copy(), sm.copy())


def test_phase2_split_and_fused_agree(gp, monkeypatch):
    """Phase-II frames (~220 hits) take the split path too (the mask-factorised
    selection walk, store sized for ~330 candidates per frame, a triple list of up
    to 32 per frame): byte-identical to the fused kernel (pair-list walk), also
    with a store that forces spills.  Every walk evaluates each cut with the same
    fp32 expression (cos_sep, pair_u), so the candidate lists agree exactly."""
    n = 80
    d, fr, df = _gen("phase2_stress", n, 731)
    outs = []
    for env in [{}, {"M3E_CAND_STORE": "100"}, {"M3E_FUSED": "1"}]:
        for k in ["M3E_CAND_STORE", "M3E_FUSED"]:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c = m3e.Context(0)
        res = m3e.run_filter(c, gp, df)
        torch.cuda.synchronize()
        outs.append(_outputs(res, n))
        c.close()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


def test_dense_frames_mask_walks(gp, P, monkeypatch):
    """Frames denser than phase II (1.2e9 and 1.7e9 mu/s: ~67 / ~95 hits per layer)
    drive the selection kernel's mask walks with 64-bit (n1, n2 <= 64) and 128-bit
    (<= 96) masks and the pair-list walk beyond: item by item against the oracle,
    and byte-identical to the fused kernel, which takes the pair-list walk for
    every big frame."""
    for rate, n, seed in ((1.2e9, 40, 741), (1.7e9, 12, 742)):
        sc = synth.SynthConfig(muon_rate=rate, seed=seed)
        d = synth.generate(sc, n)
        fr, df = oracle.Frames(d), m3e.DeviceFrames(d)
        cnt = np.diff(d["offsets"].astype(np.int64)).reshape(-1, 4)
        m = np.maximum(cnt[:, 1], cnt[:, 2])
        print(f"rate {rate:.2g}: frames with max(n1, n2) <= 64 / <= 96 / > 96:",
              int((m <= 64).sum()), int(((m > 64) & (m <= 96)).sum()), int((m > 96).sum()))
        outs = []
        for env in [{}, {"M3E_FUSED": "1"}]:
            monkeypatch.delenv("M3E_FUSED", raising=False)
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            c = m3e.Context(0)
            res = m3e.run_filter(c, gp, df)
            torch.cuda.synchronize()
            if not env:
                tally = _compare_full(P, fr, res, n, f"dense {rate:.2g}")
                assert len(tally.frames) <= 1
            outs.append(_outputs(res, n))
            c.close()
        for a, b in zip(outs[0], outs[1]):
            assert np.array_equal(a, b)
        if rate < 1.5e9:
            assert ((m > 64) & (m <= 96)).sum() >= n // 4 and (m <= 64).sum() >= 2
        else:
            assert (m > 96).sum() >= 1


def test_vertex_triple_list_full(gp, monkeypatch):
    """The split path's vertex stage lists e+e+e- triples for a dense phase-2
    kernel; frames whose triples do not fit the list (M3E_TRI_CAP, read at
    m3e_create) run the whole vertex selection in place.  Both must give the
    fused kernel's outputs byte for byte."""
    n = 3000
    d, fr, df = _gen("signal_only", n, 711)
    outs = []
    for env in [{}, {"M3E_TRI_CAP": "40"}, {"M3E_FUSED": "1"}]:
        for k in ["M3E_TRI_CAP", "M3E_FUSED"]:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c = m3e.Context(0)
        res = m3e.run_filter(c, gp, df)
        torch.cuda.synchronize()
        outs.append(_outputs(res, n))
        c.close()
    assert int(np.count_nonzero(outs[0][0] == m3e.REASON_VERTEX)) > n // 10
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("store", ["0", "2"])
def test_split_spill_and_fused_agree(gp, monkeypatch, store):
    """The production path runs the Selection Cuts in their own kernel and
    hands candidates to the fit kernel through a bounded store; warp-batches
    that do not fit are re-selected inside the fit kernel.  Forcing spills
    (M3E_CAND_STORE entries per frame, read at m3e_create) and the single fused
    kernel (M3E_FUSED=1) must give byte-identical outputs."""
    n = 6000
    d, fr, df = _gen("signal_only", n, 701)   # ~30 candidates per frame: store of 2/frame spills
    outs = []
    for env in [{}, {"M3E_CAND_STORE": store}, {"M3E_FUSED": "1"}]:
        for k in ["M3E_CAND_STORE", "M3E_FUSED"]:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c = m3e.Context(0)
        res = m3e.run_filter(c, gp, df)
        torch.cuda.synchronize()
        outs.append(_outputs(res, n))
        c.close()
    assert int(outs[0][5]["overflow"]) == 0
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("cuts_max", [3, 8, 40])
def test_flat_selection_cap(cfg, monkeypatch, cuts_max):
    """The production selection walks each warp-batch flat across frames and caps
    survivors per frame (R3).  With a small cuts_max many phase-I frames overflow
    inside one warp-batch, next to frames that do not: outputs must be
    byte-identical to the fused kernel's frame-by-frame walk and match the oracle
    run with the same cap."""
    c2 = dict(cfg, cuts_max=cuts_max)
    gp2, P2 = m3e.make_params(c2), oracle.make_params(c2)
    n = 4000
    d, fr, df = _gen("phase1_sig", n, 900 + cuts_max)
    outs = []
    for fused in ("0", "1"):
        monkeypatch.setenv("M3E_FUSED", fused)
        c = m3e.Context(0)
        res = m3e.run_filter(c, gp2, df)
        torch.cuda.synchronize()
        outs.append(_outputs(res, n))
        if fused == "0":
            sm = res.summary_np()
            frames_np = res.frames_np(n)
            n_ov = int(np.count_nonzero(frames_np["reason"] == m3e.REASON_TRIPLET_OVERFLOW))
            if cuts_max < 10:
                assert n_ov > n // 20
            assert np.all(frames_np["n_cand"] <= cuts_max + 1)
            tally = _compare_full(P2, fr, res, n, f"cuts_max={cuts_max}")
            assert len(tally.frames) <= max(1, 2e-3 * n)
        c.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_flat_selection_dense_frame(ctx, gp, P, cfg):
    """A dense frame (11 hits per layer on one helix bundle: > cuts_max survivors
    among <= 4096 combinations) inside a warp-batch of ordinary frames: the flat
    walk marks it TRIPLET_OVERFLOW, keeps n_cand = cuts_max + 1 and leaves the
    neighbours' candidates untouched."""
    n = 48
    d = synth.generate(synth.preset("phase1_sig", seed=931), n)
    R = cfg["layer_r"]
    rng = np.random.default_rng(5)
    off = d["offsets"].astype(np.int64)
    xs, ys, zs, noff = [], [], [], [0]
    for f in range(n):
        for layer in range(4):
            lo, hi = off[4 * f + layer], off[4 * f + layer + 1]
            if f == 7:
                for _ in range(11):
                    a = 0.3 + R[layer] / 160 + rng.normal() * 1e-3
                    xs.append(R[layer] * math.cos(a)); ys.append(R[layer] * math.sin(a)); zs.append(rng.normal() * 0.5)
            else:
                xs.extend(d["x"][lo:hi]); ys.extend(d["y"][lo:hi]); zs.extend(d["z"][lo:hi])
            noff.append(len(xs))
    d2 = {"x": np.array(xs, np.float32), "y": np.array(ys, np.float32), "z": np.array(zs, np.float32),
          "offsets": np.array(noff, np.uint32)}
    res = m3e.run_filter(ctx, gp, m3e.DeviceFrames(d2))
    torch.cuda.synchronize()
    fo = res.frames_np(n)
    assert int(fo["reason"][7]) == m3e.REASON_TRIPLET_OVERFLOW
    assert int(fo["n_cand"][7]) == P.cuts_max + 1
    fr2 = oracle.Frames(d2)
    tally = _compare_full(P, fr2, res, n, "dense frame")
    assert len(tally.frames) <= 1


def test_host_path_matches_device(ctx, gp, P):
    """m3e_filter_host (chunked, two streams) == m3e_filter on the same frames."""
    n = 5000
    d, fr, df = _gen("phase1_sig", n, 501)
    res = m3e.run_filter(ctx, gp, df)
    torch.cuda.synchronize()
    small = m3e.Context(0, max_frames=1234)  # forces 5 chunks
    H = len(d["x"])
    reason = np.zeros(n, np.uint8)
    frames = np.zeros(n, m3e.FRAME_DTYPE)
    tracks = np.zeros(16 * n, m3e.TRACK_DTYPE)
    kept_frame = np.zeros(n, np.uint32)
    kept_off = np.zeros(4 * n + 1, np.uint32)
    kx, ky, kz = (np.zeros(H + 8, np.float32) for _ in range(3))
    vert = np.zeros(n, m3e.VERTEX_DTYPE)
    summ = np.zeros(1, m3e.SUMMARY_DTYPE)
    x, y, z = (np.concatenate([d[k], np.zeros(8, np.float32)]) for k in "xyz")
    out = m3e.make_outputs(reason=reason, frames=frames, tracks=tracks, track_capacity=len(tracks),
                           vertices=vert, kept_frame=kept_frame, kept_offsets=kept_off, kept_capacity=n,
                           kept_x=kx, kept_y=ky, kept_z=kz, kept_hit_capacity=H + 8, summary=summ)
    m3e.filter_host(small, gp, x, y, z, d["offsets"], n, out)
    small.close()
    sm = res.summary_np()
    assert np.array_equal(reason, res.reason.cpu().numpy()[:n])
    # the track array's slot layout follows each call's warp-batches (chunks of 1234
    # frames split warp-batches differently than one call): every frame field but
    # track_first equal, each frame's tracks equal, both layouts valid
    fd = res.frames_np(n)
    for k in m3e.FRAME_DTYPE.names:
        if k != "track_first":
            assert np.array_equal(frames[k], fd[k]), k
    T, Th = int(sm["track_slots"]), int(summ[0]["track_slots"])
    assert int(summ[0]["tracks"]) == int(sm["tracks"])
    td = res.tracks_np(T)
    check_track_layout(P, frames, tracks[:Th], summ[0])
    check_track_layout(P, fd, td, sm)
    nt = np.where((fd["reason"] != 1) & (fd["reason"] != 5),
                  np.minimum(fd["n_tracks"].astype(np.int64), gp.max_tracks), 0)
    ih = np.repeat(frames["track_first"].astype(np.int64), nt) + np.arange(int(nt.sum())) - \
        np.repeat(np.cumsum(nt) - nt, nt)
    idv = np.repeat(fd["track_first"].astype(np.int64), nt) + np.arange(int(nt.sum())) - \
        np.repeat(np.cumsum(nt) - nt, nt)
    assert np.array_equal(tracks[ih], td[idv])
    K = int(np.count_nonzero(reason))
    assert np.array_equal(kept_frame[:K], res.kept_frame.cpu().numpy()[:K].view(np.uint32))
    assert np.array_equal(kept_off[:4 * K + 1], res.kept_offsets.cpu().numpy()[:4 * K + 1].view(np.uint32))
    assert np.array_equal(vert[:K], res.vertices_np(K))


def test_pack_frames(ctx):
    n = 777
    d, fr, df = _gen("phase1_bg", n, 601)
    rng = np.random.default_rng(0)
    reason = rng.choice([0, 0, 0, 1, 4], size=n).astype(np.uint8)
    res = m3e.Result(n, df.n_hits)
    m3e.pack_frames(ctx, df.x, df.y, df.z, df.offsets, n, df.n_hits, torch.from_numpy(reason).cuda(), res.outputs)
    torch.cuda.synchronize()
    kept = np.nonzero(reason)[0]
    K = len(kept)
    assert np.array_equal(res.kept_frame.cpu().numpy()[:K], kept)
    koff = res.kept_offsets.cpu().numpy()[:4 * K + 1].astype(np.int64)
    off = d["offsets"].astype(np.int64)
    want = np.concatenate([d["z"][off[4 * f]:off[4 * f + 4]] for f in kept])
    assert koff[-1] == len(want)
    assert np.array_equal(res.kept_z.cpu().numpy()[:len(want)], want)
    assert int(res.summary_np()["kept_hits"]) == len(want)


def test_edge_cases(ctx, gp, P, cfg):
    """empty call, empty frames/layers, a frame with > 1024 hits in a layer
    (M3E_REASON_INVALID), a triplet-overflow frame, ragged batch boundaries."""
    # F = 0
    res = m3e.Result(0, 0)
    empty = m3e.DeviceFrames({"x": np.zeros(0, np.float32), "y": np.zeros(0, np.float32),
                              "z": np.zeros(0, np.float32), "offsets": np.zeros(1, np.uint32)})
    m3e.run_filter(ctx, gp, empty, res)
    torch.cuda.synchronize()
    assert int(res.summary_np()["frames"]) == 0
    # hand-built frames
    R = cfg["layer_r"]
    frames = [[[], [], [], []], [[(R[0], 0, 0)], [], [(R[2], 0, 0)], [(R[3], 0, 0)]]]
    rng = np.random.default_rng(3)
    dense = []
    for layer in range(4):
        dense.append([(R[layer] * math.cos(0.3 + R[layer] / 160 + rng.normal() * 1e-3),
                       R[layer] * math.sin(0.3 + R[layer] / 160 + rng.normal() * 1e-3), rng.normal() * 0.5)
                      for _ in range(12)])
    frames.append(dense)
    big = [[(R[0] * math.cos(a), R[0] * math.sin(a), 0.0) for a in np.linspace(0, 6, 1100)], [], [], []]
    frames.append(big)
    xs, ys, zs, off = [], [], [], [0]
    for fr_ in frames:
        for layer in fr_:
            for h in layer:
                xs.append(h[0]); ys.append(h[1]); zs.append(h[2])
            off.append(len(xs))
    d = {"x": np.array(xs, np.float32), "y": np.array(ys, np.float32), "z": np.array(zs, np.float32),
         "offsets": np.array(off, np.uint32)}
    df = m3e.DeviceFrames(d)
    res = m3e.run_filter(ctx, gp, df)
    torch.cuda.synchronize()
    fo = res.frames_np(4)
    assert list(fo["reason"]) == [0, 0, m3e.REASON_TRIPLET_OVERFLOW, m3e.REASON_INVALID]
    assert int(fo["n_cand"][2]) == P.cuts_max + 1
    # ragged sizes around the batch size
    for n in (63, 64, 65, 130):
        d2 = synth.generate(synth.preset("phase1_sig", seed=700 + n), n)
        fr2 = oracle.Frames(d2)
        res2 = m3e.run_filter(ctx, gp, m3e.DeviceFrames(d2))
        torch.cuda.synchronize()
        tally = _compare_full(P, fr2, res2, n, f"ragged {n}")
        assert len(tally.frames) <= 1
