"""CPU test of the GPU parity harness (tests/parity.py): outputs in the C-ABI
layouts built from the oracle's own results, rounded to the float32 fields of
m3e_track (the vertex stage then re-run on those float32 tracks, as the CUDA
path does), must pass item by item; a plausible bug injected anywhere (a dropped
or extra track, a kappa off by 2e-4, a flipped vertex decision, a moved
vertex, a miscounted candidate list) must fail."""
import copy

import numpy as np
import pytest

import oracle
import synth
from paper_2206_11535_b200.m3e import FRAME_DTYPE, TRACK_DTYPE, VERTEX_DTYPE
from parity import Tally, compare_outputs, vtracks_gpu


def _fake_outputs(P, fr, n):
    frames = np.zeros(n, FRAME_DTYPE)
    tracks, verts = [], []
    for f in range(n):
        o, otr = oracle.process_frame(P, fr, f)
        g = frames[f]
        g["n_cand"], g["n_tracks"], g["reason"] = o.n_cand, o.n_tracks, o.reason
        g["track_first"] = len(tracks)
        g["kept_index"] = 0xFFFFFFFF
        ft = []
        if o.reason != oracle.REASON_TRIPLET_OVERFLOW:
            for t in otr:
                r = np.zeros(1, TRACK_DTYPE)[0]
                r["frame"], r["hit"] = f, t.hit
                for k in ("kappa", "chi2", "cos_theta01", "cx", "cy"):
                    r[k] = getattr(t, k)
                ft.append(r)
        tracks.extend(ft)
        reason, ncomb, vx = o.reason, 0, None
        if o.reason not in (oracle.REASON_TRIPLET_OVERFLOW, oracle.REASON_TRACK_OVERFLOW):
            w, _ = oracle.vertex_frame(P, vtracks_gpu(fr, f, ft))
            reason, ncomb = (w.reason if w.keep else 0), w.n_combs
            if reason == oracle.REASON_VERTEX:
                vx = w.vertex
        g["reason"], g["n_combs"] = reason, ncomb
        if reason:
            g["kept_index"] = len(verts)
            v = np.zeros(1, VERTEX_DTYPE)[0]
            v["frame"] = f if vx is not None else 0xFFFFFFFF
            if vx is not None:
                v["track"] = (vx.a, vx.b, vx.e)
                v["x"], v["y"], v["z"], v["chi2"] = vx.x, vx.y, vx.z, vx.chi2
            verts.append(v)
    return frames, np.array(tracks, TRACK_DTYPE), np.array(verts, VERTEX_DTYPE)


@pytest.fixture(scope="module")
def data(P):
    out = {}
    for name, n, seed in (("phase1_sig", 500, 1501), ("signal_only", 300, 1502)):
        d = synth.generate(synth.preset(name, seed=seed), n)
        fr = oracle.Frames(d)
        out[name] = (fr, n) + _fake_outputs(P, fr, n)
    return out


def test_float32_outputs_pass(P, data):
    for name, (fr, n, fo, tr, vx) in data.items():
        tally = compare_outputs(P, fr, fo, tr, vx, range(n))
        assert len(tally.frames) <= 2, tally.report(name)
        if name == "signal_only":
            assert tally.counts().get("_vertex_compared", 0) > 50


def _frame_with(fo, tr, pred):
    for f in range(len(fo)):
        nt = min(int(fo["n_tracks"][f]), 64)
        if int(fo["reason"][f]) != 1 and pred(f, nt):
            return f
    raise AssertionError("no such frame")


@pytest.mark.parametrize("bug", ["drop_track", "kappa", "cos_theta", "centre", "n_cand", "reason", "n_combs",
                                 "vertex_xyz", "hit3"])
def test_injected_bugs_fail(P, data, bug):
    fr, n, fo, tr, vx = copy.deepcopy(data["signal_only"])
    if bug == "drop_track":   # a track vanishes, the list and counts stay consistent
        f = _frame_with(fo, tr, lambda f, nt: nt >= 2 and int(fo["reason"][f]) == 0)
        i = int(fo["track_first"][f])
        tr = np.delete(tr, i)
        fo["n_tracks"][f] -= 1
        fo["track_first"][f + 1:] -= 1
    elif bug in ("kappa", "cos_theta", "centre", "hit3"):
        f = _frame_with(fo, tr, lambda f, nt: nt >= 1)
        i = int(fo["track_first"][f])
        if bug == "kappa":
            tr["kappa"][i] *= 1 + 2e-4
        elif bug == "cos_theta":
            tr["cos_theta01"][i] += 3e-4
        elif bug == "centre":
            tr["cx"][i] += 0.05
        else:
            n3 = int(fr.layer_counts(f)[3])
            tr["hit"][i][3] = (int(tr["hit"][i][3]) + 1) % max(n3, 2)
    elif bug == "n_cand":
        f = _frame_with(fo, tr, lambda f, nt: oracle.process_frame(P, fr, f)[0].n_cand_marginal == 0
                        and int(fo["n_cand"][f]) > 0)
        fo["n_cand"][f] += 1
    elif bug == "reason":
        f = _frame_with(fo, tr, lambda f, nt: int(fo["reason"][f]) == oracle.REASON_VERTEX)
        fo["reason"][f] = 0
    elif bug == "n_combs":
        f = _frame_with(fo, tr, lambda f, nt: int(fo["n_combs"][f]) > 0)
        fo["n_combs"][f] += 1
    elif bug == "vertex_xyz":
        f = _frame_with(fo, tr, lambda f, nt: int(fo["reason"][f]) == oracle.REASON_VERTEX)
        vx["z"][int(fo["kept_index"][f])] += 1e-6
    with pytest.raises(AssertionError):
        compare_outputs(P, fr, fo, tr, vx, range(n), Tally())


def _gapped(P, fo, tr, fb=8):
    """the fake outputs re-laid out as the CUDA path lays out its track array:
    warp-batches of fb frames, each owning sum min(n_cand, max_tracks) slots,
    its tracks at the front, the rest marked unused"""
    fo = fo.copy()
    live = (fo["reason"] != 1) & (fo["reason"] != 5)
    nt = np.where(live, np.minimum(fo["n_tracks"].astype(np.int64), P.max_tracks), 0)
    ns = np.where(live, np.minimum(fo["n_cand"].astype(np.int64), P.max_tracks), 0)
    out, pos = [], 0
    for b0 in range(0, len(fo), fb):
        slots = int(ns[b0:b0 + fb].sum())
        batch = []
        for f in range(b0, min(len(fo), b0 + fb)):
            fo["track_first"][f] = pos + len(batch)
            i = int(fo["track_first"][f]) - pos
            src = tr[int(np.cumsum(nt)[f] - nt[f]):int(np.cumsum(nt)[f])]
            batch.extend(src)
            assert i + len(src) == len(batch)
        mark = np.zeros(1, TRACK_DTYPE)[0]
        mark["frame"] = 0xFFFFFFFF
        batch.extend([mark] * (slots - len(batch)))
        out.extend(batch)
        pos += slots
    sm = {"track_slots": pos, "tracks": int(nt.sum())}
    return fo, np.array(out, TRACK_DTYPE), sm


@pytest.mark.parametrize("bug", [None, "marker", "frame", "extent", "order"])
def test_track_layout_check(P, data, bug):
    """check_track_layout accepts the gapped frame-ordered layout and rejects a
    dirty unused slot, a track filed under the wrong frame, a wrong extent, or
    frames out of order"""
    from parity import check_track_layout
    fr, n, fo, tr, vx = data["phase1_sig"]
    fo, tg, sm = _gapped(P, fo, tr)
    assert len(tg) > sm["tracks"]   # the layout really has unused slots
    if bug is None:
        check_track_layout(P, fo, tg, sm)
        tally = compare_outputs(P, fr, fo, tg, vx, range(n))
        assert len(tally.frames) <= 2
        return
    if bug == "marker":
        i = int(np.nonzero(tg["frame"] == 0xFFFFFFFF)[0][0])
        tg["kappa"][i] = 1.0
    elif bug == "frame":
        i = int(np.nonzero(tg["frame"] != 0xFFFFFFFF)[0][3])
        tg["frame"][i] += 1
    elif bug == "extent":
        sm = dict(sm, track_slots=sm["track_slots"] + 1)
    elif bug == "order":
        f = int(np.nonzero(fo["n_tracks"] > 0)[0][1])
        fo["track_first"][f] = 0
    with pytest.raises(AssertionError):
        check_track_layout(P, fo, tg, sm)
