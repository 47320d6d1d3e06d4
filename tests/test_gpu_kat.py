"""SPEC known-answer examples through the C-ABI on the GPU (golden: tests/golden/spec_kats.json)."""
import math

import numpy as np
import pytest

from paper_2206_02200_b200 import gridshift as G

pytestmark = pytest.mark.gpu


def test_grid_index(engine, kats):
    for case in kats["grid_index"]:
        keys, counts, cent, slot = engine.debug_build(np.array([case["x"]]), case["h"])
        assert keys.tolist() == [case["key"]], case["src"]
        assert counts.tolist() == [1]


def test_build(engine, kats):
    from oracle import oracle as O
    for case in kats["build"]:
        X = np.array(case["X"], np.float64)
        keys, counts, cent, slot = engine.debug_build(X, case["h"])
        assert keys.tolist() == case["keys"], case["src"]
        assert counts.tolist() == case["counts"]
        np.testing.assert_allclose(cent, case["centroids"], rtol=case["tol"])
        assert len(slot) == len(X)
        # fp32 inputs are widened exactly; 0.9f/0.1 floors to 8, not 9, so compare with the
        # oracle on the widened values rather than with the fp64 example
        X32 = X.astype(np.float32)
        g = engine.debug_build(X32, case["h"])
        o = O.build_grid(X32.astype(np.float64), case["h"], O.BUILD_FIXED)
        assert g[0].tolist() == o[0].tolist() and g[1].tolist() == o[1].tolist()
        assert g[2].tobytes() == o[2].tobytes()


def test_merge(engine, kats):
    for case in kats["merge"]:
        r = engine.debug_iterate_once(np.array(case["keys"]), np.array(case["counts"]),
                                      np.array(case["centroids"]), case["h"])
        assert r["keys"].tolist() == case["out_keys"], case["src"]
        assert r["counts"].tolist() == case["out_counts"]
        np.testing.assert_allclose(r["centroids"], case["out_centroids"], rtol=case["tol"])
        assert r["parent"].tolist() == [0] * len(case["keys"])


def test_iterate_once(engine, kats):
    for case in kats["iterate_once"]:
        r = engine.debug_iterate_once(np.array(case["keys"]), np.array(case["counts"]),
                                      np.array(case["centroids"]), case["h"])
        if case["tol"] == 0.0:
            assert r["swept"].tolist() == case["swept"], case["src"]
            assert r["centroids"].tolist() == case["out_centroids"]
        else:
            np.testing.assert_allclose(r["swept"], case["swept"], rtol=case["tol"])
            np.testing.assert_allclose(r["centroids"], case["out_centroids"], rtol=case["tol"])
        assert r["keys"].tolist() == case["out_keys"]
        assert r["counts"].tolist() == case["out_counts"]
        assert r["changed"] == case["changed"]


def test_spec_123_bit_exact(engine):
    r = engine.debug_iterate_once(np.array([[0], [1]]), np.array([3, 1]),
                                  np.array([[0.4], [0.6]]), 0.5)
    s0 = (3 * 0.4 + 1 * 0.6) / 4
    s1 = (3 * s0 + 1 * 0.6) / 4
    assert r["swept"][:, 0].tolist() == [s0, s1]
    assert r["centroids"][0, 0] == (3 * s0 + 1 * s1) / 4


def test_jacobi_contrast(engine, kats):
    c = kats["jacobi_contrast"][0]
    r = engine.debug_iterate_once(np.array(c["keys"]), np.array(c["counts"]),
                                  np.array(c["centroids"]), c["h"])
    assert math.isclose(r["swept"][1, 0], c["engine_cell1"], rel_tol=1e-15)
    assert abs(r["swept"][1, 0] - c["jacobi_cell1"]) > 0.03


def test_run(engine, kats):
    for case in kats["run"]:
        r = engine.run(np.array(case["X"]), G.EngineConfig(case["h"], 1000))
        assert r.labels.tolist() == case["labels"], case["src"]
        assert len(r.centroids) == case["k"]
        if "iterations" in case:
            assert r.iterations == case["iterations"]
        np.testing.assert_allclose(r.centroids, case["centroids"], rtol=case["tol"])
        assert r.converged


def test_run_traced(engine, kats):
    for case in kats["run_traced"]:
        r = engine.run(np.array(case["X"]), G.EngineConfig(case["h"], 1000, record_history=True))
        assert len(r.history) == case["snapshots"], case["src"]


def test_errors(engine):
    X = np.array([[0.1, 0.2], [0.3, 0.4]])
    with pytest.raises(G.InvalidBandwidthError):
        engine.run(X, G.EngineConfig(0.0))
    with pytest.raises(G.InvalidBandwidthError):
        engine.run(X, G.EngineConfig(-1.0))
    with pytest.raises(G.EmptyInputError):
        engine.run(np.zeros((0, 2)), G.EngineConfig(0.5))
    with pytest.raises(G.InvalidInputError):
        engine.run(np.array([[0.1, np.nan]]), G.EngineConfig(0.5))
    with pytest.raises(G.InvalidInputError):
        engine.run(np.array([[0.1, np.inf]], np.float32), G.EngineConfig(0.5))
    with pytest.raises(G.InvalidParameterError):
        engine.run(X, G.EngineConfig(0.5, max_iterations=0))
    # the context stays usable after an error
    r = engine.run(X, G.EngineConfig(0.5))
    assert r.labels.tolist() == [0, 0]


def test_max_iter_warning_flag(engine):
    # a long chain of adjacent cells cannot finish in one iteration: partial result + flag
    X = np.arange(0, 40, 0.25)[:, None]
    r = engine.run(X, G.EngineConfig(1.0, max_iterations=1))
    assert r.iterations == 1 and not r.converged
    assert r.labels.shape == (len(X),)
