"""Tracker: init_tracker / track_frame / track_sequence, Algorithm 2
(/root/reference/SPEC.md:437-498).

CPU tests check the oracle restatement (oracle/gs_oracle.cpp, pins T1-T5) against the SPEC's
examples on synthetic fixtures with known trajectories; GPU tests require gs_track_init /
gs_track_sequence to equal the oracle BIT-EXACTLY (windows, lost flags, inner iterations).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2206_02200_b200 import configs as CF
from paper_2206_02200_b200 import gridshift as G

RED, BLUE = (220, 20, 20), (20, 20, 200)


def square_seq(T=8, H=96, W=128, s=16, start=(30, 30), v=(5, 0), remove_at=None, bg=BLUE):
    fr = np.empty((T, H, W, 3), np.uint8)
    fr[...] = bg
    centres = []
    for t in range(T):
        x0, y0 = start[0] + v[0] * t, start[1] + v[1] * t
        if remove_at is None or t < remove_at:
            fr[t, y0:y0 + s, x0:x0 + s] = RED
        centres.append((x0 + (s - 1) / 2, y0 + (s - 1) / 2))
    return fr, np.array(centres)


def win_at(c, size=20.0):
    # the 16-px square must dominate the window: top_1 selects the largest cluster
    return [c[0], c[1], size, size]


# ------------------------------------------------------------------ oracle (CPU)
def test_shifted_square_centre_within_eta():
    fr, c = square_seq(T=6, v=(5, 0))
    r = O.track(fr, win_at(c[0]), h=0.1, eta=1.0)
    assert not r["lost"].any()
    for t in range(1, 6):
        assert np.hypot(*(r["windows"][t - 1, :2] - c[t])) <= 1.0


def test_zero_matching_pixels_grow_and_lost():
    fr, c = square_seq(T=3, remove_at=1)
    r = O.track(fr, win_at(c[0]), h=0.1, max_inner=7)
    assert r["lost"].all()
    # after k inner iterations the window dims are x1.1^k
    l = 20.0
    for t in range(2):
        for _ in range(7):
            l = l * 1.1
        assert r["windows"][t, 2] == l and r["windows"][t, 3] == l
    assert (r["inner"] == 7).all()


def test_stationary_target_shrinks():
    fr, c = square_seq(T=4, v=(0, 0))
    r = O.track(fr, win_at(c[0]), h=0.1)
    # matched extent 15 < 20 on both axes: x0.99 per convergence pass
    w = 20.0
    for t in range(3):
        for _ in range(int(r["inner"][t])):
            w = w * 0.99
        assert r["windows"][t, 2] == w and r["windows"][t, 3] == w
        assert np.allclose(r["windows"][t, :2], c[0])


def test_linear_motion_30_frames():
    # SPEC.md:477 claims <= 2 px per frame over 30 frames.  Under the literal size rule the
    # matched extent inside the window is always < l, so the window shrinks 1 % per inner
    # iteration and the centre lags the target more as it shrinks (6 px by frame 30 at 5 px per
    # frame, DESIGN.md §"Tracker"): the claim holds for the first 10 frames; the target is never
    # lost over the 30.
    fr, c = square_seq(T=31, H=120, W=220, v=(5, 2), start=(10, 20))
    r = O.track(fr, win_at(c[0]), h=0.1)
    err = np.hypot(*(r["windows"][:, :2] - c[1:]).T)
    assert err[:10].max() <= 2.0 and err.max() <= 8.0 and not r["lost"].any()


def test_target_removed_lost_onward():
    fr, c = square_seq(T=14, v=(2, 0), remove_at=10)
    r = O.track(fr, win_at(c[0]), h=0.1, max_inner=5)
    assert not r["lost"][:9].any() and r["lost"][9:].all()
    assert np.all(np.diff(r["windows"][8:, 2]) > 0)  # windows keep growing


def test_oracle_errors():
    fr, c = square_seq(T=2)
    with pytest.raises(O.OracleError) as e:
        O.track(fr, [500.0, 500.0, 10.0, 10.0], h=0.1)
    assert e.value.status == 13  # InvalidWindowError
    with pytest.raises(O.OracleError) as e:
        O.track(fr, win_at(c[0]), h=0.1, ids=[7])
    assert e.value.status == 14  # SelectionError
    with pytest.raises(O.OracleError) as e:
        O.track(fr, win_at(c[0]), h=0.0)
    assert e.value.status == 2


# ------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def tracker():
    t = G.Tracker(0)
    yield t
    t.close()


def gpu_track(tracker, frames, window, **kw):
    cfg = G.TrackerConfig(h=kw.pop("h"), f=kw.pop("f", 1.0), eta=kw.pop("eta", 1.0),
                          max_inner_iters=kw.pop("max_inner", 20), top_k=kw.pop("top_k", 1),
                          ids=kw.pop("ids", None))
    assert not kw
    tracker.init(frames[0], window, cfg)
    return tracker.track_sequence(frames[1:])


def assert_same(gpu, ora):
    win, lost, inner = gpu
    assert np.array_equal(win.view(np.int64), ora["windows"].view(np.int64)), (win, ora["windows"])
    assert np.array_equal(lost, ora["lost"])
    assert np.array_equal(inner, ora["inner"])


CASES = [
    ("shift", dict(T=6, v=(5, 0)), 20.0, dict(h=0.1)),
    ("lost", dict(T=4, remove_at=1), 20.0, dict(h=0.1, max_inner=7)),
    ("stationary", dict(T=4, v=(0, 0)), 20.0, dict(h=0.1)),
    ("linear30", dict(T=31, H=120, W=220, v=(5, 2), start=(10, 20)), 20.0, dict(h=0.1)),
    ("removed", dict(T=14, v=(2, 0), remove_at=10), 20.0, dict(h=0.1, max_inner=5)),
    ("f2", dict(T=8, v=(3, 1)), 30.0, dict(h=0.08, f=1.5, eta=0.5)),
    ("background", dict(T=5, v=(4, 4)), 40.0, dict(h=0.1, top_k=2)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,seq,size,kw", CASES, ids=[c[0] for c in CASES])
def test_gpu_track_matches_oracle(tracker, name, seq, size, kw):
    fr, c = square_seq(**seq)
    w = win_at(c[0], size)
    ora = O.track(fr, w, **kw)
    assert_same(gpu_track(tracker, fr, w, **dict(kw)), ora)


@pytest.mark.gpu
def test_gpu_track_ellipse_frames(tracker):
    X = CF.ellipse_frames(nf=12)  # cfg4 frames (features in [0,1]) -> 8-bit pixels
    fr = np.clip(np.rint(X.astype(np.float64) * 255.0), 0, 255).astype(np.uint8)
    fr = fr.reshape(12, 480, 640, 3)
    for win in ([320.0, 240.0, 120.0, 90.0], [150.0, 100.0, 60.0, 60.0]):
        for kw in (dict(h=0.08), dict(h=0.08, top_k=2), dict(h=0.12, f=1.5, eta=0.5)):
            ora = O.track(fr, win, **kw)
            assert_same(gpu_track(tracker, fr, win, **dict(kw)), ora)


@pytest.mark.gpu
def test_gpu_track_errors(tracker):
    fr, c = square_seq(T=2)
    with pytest.raises(G.InvalidWindowError):
        gpu_track(tracker, fr, [500.0, 500.0, 10.0, 10.0], h=0.1)
    with pytest.raises(G.SelectionError):
        gpu_track(tracker, fr, win_at(c[0]), h=0.1, ids=[7])
    with pytest.raises(G.InvalidBandwidthError):
        gpu_track(tracker, fr, win_at(c[0]), h=0.0)
