"""Pins the CPU oracle against every known-answer example of the reference spec.

The reference has no tests, fixtures or golden files; these SPEC examples are
the only published answers for the path, transcribed into tests/golden/spec_kats.json.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O


def test_grid_index(kats):
    # grid_index via build of a single point: the cell key is floor(x/h)
    for case in kats["grid_index"]:
        keys, counts, cent, _ = O.build_grid(np.array([case["x"]]), case["h"], O.BUILD_SPEC)
        assert keys.tolist() == [case["key"]], case["src"]


def test_neighborhood(kats):
    # neighborhood: a cell surrounded by all 3^d neighbours sees them all
    for case in kats["neighborhood"]:
        d = case["d"]
        j = np.array(case["j"])
        offs = np.array(np.meshgrid(*[[-1, 0, 1]] * d, indexing="ij")).reshape(d, -1).T
        keys = j + offs  # lexicographic order in v
        assert len(keys) == 3 ** d
        if "expect" in case:
            assert keys.tolist() == case["expect"], case["src"]
        assert not O.has_converged(keys)
        assert O.has_converged(j[None])


def test_build(kats):
    for case in kats["build"]:
        for mode in (O.BUILD_SPEC, O.BUILD_FIXED):
            keys, counts, cent, slot = O.build_grid(np.array(case["X"]), case["h"], mode)
            assert keys.tolist() == case["keys"], case["src"]
            assert counts.tolist() == case["counts"]
            np.testing.assert_allclose(cent, case["centroids"], rtol=case["tol"], atol=1e-15)
            if mode == O.BUILD_SPEC and case["src"] == "SPEC.md:64":
                # incremental mean of 0.1, 0.2 is exactly (1*0.1+0.2)/2
                assert cent[0, 0] == (1 * 0.1 + 0.2) / 2


def test_merge(kats):
    for case in kats["merge"]:
        r = O.iterate_once(case["keys"], case["counts"], case["centroids"], case["h"])
        assert r["keys"].tolist() == case["out_keys"], case["src"]
        assert r["counts"].tolist() == case["out_counts"]
        np.testing.assert_allclose(r["centroids"], case["out_centroids"], rtol=case["tol"])
        assert r["parent"].tolist() == [0] * len(case["keys"])
        # merge conservation: Σcount and Σcount*centroid preserved
        c_in = np.array(case["counts"], float)
        s_in = np.array(case["centroids"])[:, 0]
        assert r["counts"].sum() == c_in.sum()
        assert math.isclose(float((r["counts"] * r["centroids"][:, 0]).sum()),
                            float((c_in * s_in).sum()), rel_tol=1e-14)


def test_iterate_once(kats):
    for case in kats["iterate_once"]:
        r = O.iterate_once(case["keys"], case["counts"], case["centroids"], case["h"])
        if case["tol"] == 0.0:
            assert r["swept"].tolist() == case["swept"], case["src"]
            assert r["centroids"].tolist() == case["out_centroids"]
        else:
            np.testing.assert_allclose(r["swept"], case["swept"], rtol=case["tol"])
            np.testing.assert_allclose(r["centroids"], case["out_centroids"], rtol=case["tol"])
        assert r["keys"].tolist() == case["out_keys"]
        assert r["counts"].tolist() == case["out_counts"]
        assert r["changed"] == case["changed"]


def test_spec_123_exact_values():
    # the SPEC.md:123 hand trace holds to the last bit in fp64
    r = O.iterate_once([[0], [1]], [3, 1], [[0.4], [0.6]], 0.5)
    assert r["swept"][0, 0] == (3 * 0.4 + 1 * 0.6) / 4
    assert r["swept"][1, 0] == (3 * r["swept"][0, 0] + 1 * 0.6) / 4
    assert r["centroids"][0, 0] == (3 * r["swept"][0, 0] + 1 * r["swept"][1, 0]) / 4


def test_has_converged(kats):
    for case in kats["has_converged"]:
        assert O.has_converged(np.array(case["keys"])) == case["expect"], case["src"]


def test_run(kats):
    for case in kats["run"]:
        for mode in (O.BUILD_SPEC, O.BUILD_FIXED):
            r = O.run(np.array(case["X"]), case["h"], 1000, mode)
            assert r["k"] == case["k"], case["src"]
            assert r["labels"].tolist() == case["labels"]
            if "iterations" in case:
                assert r["iterations"] == case["iterations"]
            np.testing.assert_allclose(r["centroids"], case["centroids"], rtol=case["tol"])
            assert r["converged"]


def test_run_traced(kats):
    for case in kats["run_traced"]:
        r = O.run(np.array(case["X"]), case["h"])
        assert len(r["history"]) == case["snapshots"], case["src"]


def test_jacobi_contrast(kats):
    c = kats["jacobi_contrast"][0]
    r = O.iterate_once(c["keys"], c["counts"], c["centroids"], c["h"])
    # fp64 gives 0.48750000000000004 for the SPEC's exact 0.4875
    assert math.isclose(r["swept"][1, 0], c["engine_cell1"], rel_tol=1e-15)
    assert abs(r["swept"][1, 0] - c["jacobi_cell1"]) > 0.03


def test_errors(kats):
    X = np.array([[0.1, 0.2]])
    with pytest.raises(O.OracleError) as e:
        O.run(X, 0.0)
    assert e.value.status == 2
    with pytest.raises(O.OracleError) as e:
        O.run(X, -1.0)
    assert e.value.status == 2
    with pytest.raises(O.OracleError) as e:
        O.run(np.zeros((0, 2)), 0.5)
    assert e.value.status == 3
    with pytest.raises(O.OracleError) as e:
        O.run(np.array([[0.1, np.nan]]), 0.5)
    assert e.value.status == 1


def test_invariants_random():
    # partition / conservation / non-increasing m / bounding box
    rng = np.random.default_rng(7)
    for trial in range(20):
        d = int(rng.integers(1, 5))
        n = int(rng.integers(1, 400))
        X = rng.normal(size=(n, d)) * rng.uniform(0.2, 3)
        h = float(rng.uniform(0.1, 1.5))
        r = O.run(X, h, 200, O.BUILD_SPEC)
        assert set(np.unique(r["labels"])) == set(range(r["k"]))
        ms = [m for m, _ in r["history"]]
        assert all(a >= b for a, b in zip(ms, ms[1:]))
        lo, hi = X.min(0), X.max(0)
        assert np.all(r["centroids"] >= lo - 1e-9) and np.all(r["centroids"] <= hi + 1e-9)
        r2 = O.run(X, h, 200, O.BUILD_SPEC)  # determinism SPEC.md:159
        assert np.array_equal(r["labels"], r2["labels"])
        assert np.array_equal(r["centroids"], r2["centroids"])


def test_fixed_mode_matches_spec_mode_on_small_configs():
    from paper_2206_02200_b200 import configs as CF
    for name in ("cfg1", "cfg2"):
        cfg = CF.CONFIGS[name]
        X = CF.generate(name)[0]
        a = O.run(X, cfg.h, cfg.max_iter, O.BUILD_SPEC)
        b = O.run(X, cfg.h, cfg.max_iter, O.BUILD_FIXED)
        assert a["k"] == b["k"] and a["iterations"] == b["iterations"]
        assert np.array_equal(a["labels"], b["labels"])
        np.testing.assert_allclose(a["centroids"], b["centroids"], rtol=1e-12)
