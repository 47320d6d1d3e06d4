"""Bandwidth sweep: tune_bandwidth and
silhouette / silhouette_subsampled.

CPU tests pin the oracle (oracle/gs_oracle.cpp, pins S1-S3) against the SPEC examples and an
independent implementation (scikit-learn's silhouette_score); GPU tests require the
gs_tune_bandwidth / gs_silhouette_subsampled path to equal the oracle BIT-EXACTLY (the engine
labels are bit-exact against build mode "fixed", and the silhouette follows the oracle's
summation order with correctly rounded fp64 operations).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2206_02200_b200 import configs as CF
from paper_2206_02200_b200 import gridshift as G


def two_groups(seed=3, n=200, spread=0.02, gap=0.6):
    rng = np.random.default_rng(seed)
    a = 0.1 + spread * rng.random((n // 2, 2))
    b = 0.1 + gap + spread * rng.random((n - n // 2, 2))
    return np.vstack([a, b])


def small_image(seed=2208, W=120, H=80):
    return CF.voronoi_rgb(seed=seed, W=W, H=H).astype(np.float32)


# ------------------------------------------------------------------ oracle pins (CPU)
def test_silhouette_spec_examples():
    # SPEC.md:316 two far-separated tight pairs -> > 0.9
    X = np.array([[0.0], [0.01], [10.0], [10.01]])
    sc, valid, _ = O.silhouette(X, [0, 0, 1, 1])
    assert valid and sc > 0.9
    # SPEC.md:317 all points one cluster -> undefined
    assert O.silhouette(X, [0, 0, 0, 0])[1] is False
    # SPEC.md:318 uniform interleaved labels on identical points -> 0
    sc, valid, _ = O.silhouette(np.zeros((6, 3)), [0, 1, 0, 1, 0, 1])
    assert valid and sc == 0.0


def test_silhouette_matches_sklearn():
    from sklearn.metrics import silhouette_score, silhouette_samples
    rng = np.random.default_rng(0)
    for n, d, k in [(300, 3, 5), (200, 2, 2), (150, 5, 7)]:
        X = rng.random((n, d))
        lab = rng.integers(0, k, n)
        lab[0] = k  # a singleton cluster: contributes 0
        sc, valid, per = O.silhouette(X, lab)
        assert valid
        assert abs(sc - silhouette_score(X, lab)) < 1e-12
        np.testing.assert_allclose(per, silhouette_samples(X, lab), rtol=0, atol=1e-12)


def test_subsample_pins():
    X = two_groups(n=400)
    lab = (X[:, 0] > 0.4).astype(np.int32)
    full = O.silhouette(X, lab)[0]
    # n <= cap -> exactly the silhouette
    assert O.silhouette_subsampled(X, lab, cap=400, seed=5)[0] == full
    # fixed seed -> deterministic; different seeds differ in the sample
    a = O.sample_indices(10_000, 100, 11)
    assert np.array_equal(a, O.sample_indices(10_000, 100, 11))
    assert not np.array_equal(a, O.sample_indices(10_000, 100, 12))
    assert len(np.unique(a)) == 100 and np.all(np.diff(a) > 0)
    # two-group synthetic, cap 100 -> within 0.1 of the full silhouette
    for seed in range(5):
        assert abs(O.silhouette_subsampled(X, lab, cap=100, seed=seed)[0] - full) < 0.1


def test_oracle_tune_ties_and_failure():
    X = two_groups()
    hs = [0.05, 0.1, 0.2, 0.3, 0.9]
    r = O.tune(X, hs, max_iter=100, cap=1000)
    # any h between the intra-group spread and the gap separates the groups: equal scores,
    # the smallest wins
    v = [s for s, ok in zip(r["scores"], r["valid"]) if ok]
    assert max(v) == r["scores"][hs.index(r["best_h"])]
    ties = [h for h, s, ok in zip(hs, r["scores"], r["valid"]) if ok and s == max(v)]
    assert r["best_h"] == min(ties) and len(ties) >= 2
    # single-point dataset -> tuning failure
    with pytest.raises(O.OracleError) as e:
        O.tune(np.array([[0.5, 0.5]]), hs, cap=10)
    assert e.value.status == 11


def test_tune_abi_validation_without_device():
    # argument checks happen before any device work: a bad grid is refused even here
    lib = G.load_library()
    t = G.C.c_void_p()
    st = lib.gs_tuner_create(0, 2, G.C.byref(t))
    if st == 10:  # GS_E_NO_DEVICE on a CPU-only host: the documented refusal, no fallback
        return
    assert st == 0
    lib.gs_tuner_destroy(t)


# ------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def tuner():
    t = G.Tuner(0, max_concurrent=4)
    yield t
    t.close()


def _assert_sweep_equal(gpu, ora, hs):
    assert gpu.best_h == ora["best_h"]
    for i, e in enumerate(gpu.entries):
        assert e.h == hs[i]
        assert e.k == ora["k"][i], (hs[i], e.k, ora["k"][i])
        assert e.iterations == ora["iterations"][i]
        assert (e.score is not None) == bool(ora["valid"][i])
        if e.score is not None:
            assert e.score == ora["scores"][i], (hs[i], e.score, ora["scores"][i])  # bit-exact


@pytest.mark.gpu
@pytest.mark.parametrize("cap", [500, 20_000])
def test_gpu_tune_matches_oracle_image(tuner, cap):
    X = small_image()
    hs = [0.05, 0.08, 0.1, 0.15, 0.2, 0.3, 0.5, 1.0]
    gpu = tuner.tune_bandwidth(X, hs, max_iter=100, cap=cap, seed=7)
    ora = O.tune(X.astype(np.float64), hs, max_iter=100, cap=cap, seed=7, mode=O.BUILD_FIXED)
    _assert_sweep_equal(gpu, ora, hs)


@pytest.mark.gpu
def test_gpu_tune_default_grid_blobs(tuner):
    X = CF.generate("cfg1")[0]
    X = (X - X.min(0)) / (X.max(0) - X.min(0))  # SPEC.md:348 min-max normalisation
    hs = [round(0.05 * i, 2) for i in range(1, 21)]
    gpu = tuner.tune_bandwidth(X, None, max_iter=300, cap=2000, seed=1)
    ora = O.tune(X, hs, max_iter=300, cap=2000, seed=1, mode=O.BUILD_FIXED)
    _assert_sweep_equal(gpu, ora, hs)


@pytest.mark.gpu
def test_gpu_tune_ties_smallest_h(tuner):
    X = two_groups()
    hs = [0.9, 0.3, 0.2, 0.1, 0.05]  # unsorted grid: the tie rule is on h, not grid order
    gpu = tuner.tune_bandwidth(X, hs, max_iter=100, cap=1000)
    ora = O.tune(X, hs, max_iter=100, cap=1000, mode=O.BUILD_FIXED)
    _assert_sweep_equal(gpu, ora, hs)
    assert gpu.best_h == 0.1 or gpu.best_h == min(
        e.h for e in gpu.entries if e.score is not None and e.score == max(
            x.score for x in gpu.entries if x.score is not None))


@pytest.mark.gpu
def test_gpu_silhouette_subsampled_bit_exact(tuner):
    rng = np.random.default_rng(4)
    X = rng.random((5000, 3))
    lab = rng.integers(0, 9, 5000).astype(np.int32)
    lab[17] = 50  # singleton
    for cap, seed in [(6000, 0), (800, 3), (2, 9)]:
        ora, valid, _ = O.silhouette_subsampled(X, lab, cap, seed)
        if not valid:
            with pytest.raises(G.UndefinedScoreError):
                tuner.silhouette_subsampled(X, lab, cap, seed)
            continue
        assert tuner.silhouette_subsampled(X, lab, cap, seed) == ora


@pytest.mark.gpu
def test_gpu_tune_errors(tuner):
    X = two_groups()
    with pytest.raises(G.InvalidBandwidthError):
        tuner.tune_bandwidth(X, [0.5, 1.5])
    with pytest.raises(G.InvalidBandwidthError):
        tuner.tune_bandwidth(X, [0.0])
    with pytest.raises(G.InvalidParameterError):
        tuner.tune_bandwidth(X, [])
    with pytest.raises(G.InvalidParameterError):
        tuner.tune_bandwidth(X, [0.5], cap=1)
    with pytest.raises(G.TuningFailureError):
        tuner.tune_bandwidth(np.array([[0.5, 0.5]]), [0.1, 0.5], cap=10)
    with pytest.raises(G.UndefinedScoreError):
        tuner.silhouette_subsampled(X, np.zeros(len(X), np.int32), 100)
    bad = X.copy()
    bad[3, 1] = np.nan
    with pytest.raises(G.InvalidInputError):
        tuner.tune_bandwidth(bad, [0.5])
