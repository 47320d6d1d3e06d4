"""MS++ baseline: mspp_run, parallel (Jacobi) grid mean shift
(ledger :242-246).

CPU tests check the oracle restatement (oracle/gs_oracle.cpp, pins M1-M5) against the SPEC's
examples; GPU tests require gs_mspp_run to equal the oracle BIT-EXACTLY (labels, centroids,
iterations, convergence flag, per-iteration displacement).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2206_02200_b200 import configs as CF
from paper_2206_02200_b200 import gridshift as G
from tests.parity_util import matched_agreement


def two_groups(seed=5, n=300, h=0.5):
    rng = np.random.default_rng(seed)
    a = rng.normal(0.0, 0.3, (n // 2, 2))
    b = rng.normal(0.0, 0.3, (n - n // 2, 2)) + np.array([10.0, 10.0])  # gap >> 3h
    return np.vstack([a, b])


# ------------------------------------------------------------------ oracle (CPU)
def test_spec_single_point():
    r = O.mspp(np.array([[0.3, 0.7]]), 0.5)
    assert r["k"] == 1 and r["converged"] and np.array_equal(r["centroids"], [[0.3, 0.7]])


def test_spec_parallel_update_example():
    # cells [0]:(0.4, count 3), [1]:(0.6, count 1), h = 0.5: BOTH move to 0.45
    # (old neighbour centroids), unlike the engine's sequential sweep (0.4875)
    X = np.array([[0.4], [0.4], [0.4], [0.6]])
    r = O.mspp(X, 0.5, max_iter=1)
    assert r["disp"][0] == pytest.approx(0.15, abs=1e-15)
    assert r["k"] == 1 and r["centroids"][0, 0] == pytest.approx(0.45, abs=1e-15)
    e = O.run(X, 0.5, 1, O.BUILD_FIXED)
    assert abs(e["centroids"][0, 0] - 0.45) > 1e-3  # 0.459375


def test_spec_separated_groups_match_engine():
    # groups separated by > 3h -> the same 2 clusters as engine.run
    X = two_groups()
    r = O.mspp(X, 0.5)
    e = O.run(X, 0.5, 300, O.BUILD_FIXED)
    assert r["converged"]
    assert matched_agreement(r["labels"], e["labels"])[0] == 1.0


def test_oracle_errors():
    with pytest.raises(O.OracleError):
        O.mspp(np.array([[0.0]]), 0.0)
    with pytest.raises(O.OracleError):
        O.mspp(np.array([[0.0]]), 0.5, tol=0.0)
    with pytest.raises(O.OracleError):
        O.mspp(np.array([[np.nan]]), 0.5)


# ------------------------------------------------------------------ GPU parity
def _same(gpu, ora):
    assert np.array_equal(gpu.labels, ora["labels"])
    assert gpu.iterations == ora["iterations"]
    assert gpu.converged == ora["converged"]
    assert np.array_equal(gpu.centroids.view(np.int64), ora["centroids"].view(np.int64))
    disp = np.array([v for _, v in gpu.history])
    assert np.array_equal(disp.view(np.int64), ora["disp"].view(np.int64))


CASES = [
    ("cfg1", lambda: CF.generate("cfg1")[0], 0.5, {}),
    ("cfg2", lambda: CF.generate("cfg2")[0], 0.08, {}),
    ("groups", two_groups, 0.5, {}),
    ("single", lambda: np.array([[0.3, 0.7]]), 0.5, {}),
    ("d1", lambda: np.random.default_rng(1).normal(0, 1, (2000, 1)), 0.3, {}),
    ("d4", lambda: np.random.default_rng(2).random((3000, 4)), 0.25, {}),
    ("d5", lambda: np.random.default_rng(3).random((3000, 5)), 0.3, {}),
    ("maxiter1", lambda: CF.generate("cfg1")[0], 0.5, dict(max_iter=1)),
    ("maxiter2", lambda: CF.generate("cfg2")[0], 0.08, dict(max_iter=2)),
    ("bigtol", lambda: CF.generate("cfg1")[0], 0.5, dict(tol=10.0)),
    ("cells1700", lambda: np.random.default_rng(6).random((20000, 3)), 0.09, {}),
    # first grids beyond one CTA (r2): the later iterations run on all SMs
    ("cells8000", lambda: np.random.default_rng(7).random((50000, 3)), 0.05, {}),
    ("cfg5_small", lambda: CF.generate("cfg5", scale=1 / 64)[0], 1.0, {}),
    ("cfg3_small", lambda: CF.generate("cfg3", scale=0.05)[0], 0.06, {}),
    ("big_maxiter3", lambda: np.random.default_rng(8).random((60000, 2)), 0.01, dict(max_iter=3)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,gen,h,kw", CASES, ids=[c[0] for c in CASES])
def test_gpu_mspp_matches_oracle(engine, name, gen, h, kw):
    X = gen()
    ora = O.mspp(X.astype(np.float64), h, **kw)
    _same(engine.mspp(X, h, **kw), ora)


@pytest.mark.gpu
def test_gpu_mspp_then_engine_run(engine):
    # the MS++ call leaves the context's dense grid clean: an engine run afterwards is exact
    X = CF.generate("cfg2")[0]
    engine.mspp(X, 0.08)
    r = engine.run(X, G.EngineConfig(0.08, 100))
    o = O.run(X.astype(np.float64), 0.08, 100, O.BUILD_FIXED)
    assert np.array_equal(r.labels, o["labels"])


@pytest.mark.gpu
def test_gpu_mspp_errors(engine):
    with pytest.raises(G.InvalidBandwidthError):
        engine.mspp(np.zeros((4, 2)), 0.0)
    with pytest.raises(G.InvalidParameterError):
        engine.mspp(np.zeros((4, 2)), 0.5, tol=0.0)
    bad = np.zeros((4, 2))
    bad[1, 1] = np.inf
    with pytest.raises(G.InvalidInputError):
        engine.mspp(bad, 0.5)
    # a first grid beyond one CTA runs on all SMs and leaves the context's grid clean for the
    # next engine run
    engine.mspp(np.random.default_rng(7).random((50000, 3)), 0.05)
    X = CF.generate("cfg2")[0]
    r = engine.run(X, G.EngineConfig(0.08, 100))
    assert np.array_equal(r.labels, O.run(X.astype(np.float64), 0.08, 100, O.BUILD_FIXED)["labels"])
