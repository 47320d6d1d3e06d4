"""Randomised GPU parity: seeded mixtures over d = 1..6, point counts, bandwidths, dtypes and
batches, on the default schedule (K8 after the global path), on the global path only (the
16-CTA cluster sweep for d <= 3, the dataflow sweep for d > 3), and as batched frames (the K2
table replicas).  Every case must equal the fixed-point-build oracle bit for bit."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2206_02200_b200 import gridshift as G

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def _mixture(rng, n, d):
    # (the key box must stay within the dense grid's 2^28 cells: a smaller span for d >= 5)
    k = int(rng.integers(1, 9))
    centres = rng.uniform(0.0, 4.0 if d <= 4 else 2.0, (k, d))
    sig = rng.uniform(0.05, 0.6, (k, 1))
    lab = rng.integers(0, k, n)
    return centres[lab] + sig[lab] * rng.standard_normal((n, d))


def _cases():
    out = []
    for seed in range(64):
        rng = np.random.default_rng(1000 + seed)
        d = int(rng.integers(1, 7))
        n = int(rng.integers(50, 6000 if d <= 3 else 2500))
        h = float(rng.uniform(0.15, 0.6) if d <= 4 else rng.uniform(0.35, 0.6))
        f32 = bool(rng.integers(0, 2))
        out.append((f"s{seed}-d{d}-n{n}", seed, d, n, h, f32))
    return out


def _check(engine, X, h, flags, name):
    g = engine.run(X, G.EngineConfig(h, 300, record_history=True, debug_flags=flags))
    o = O.run(X.astype(np.float64), h, 300, O.BUILD_FIXED)
    assert g.iterations == o["iterations"], name
    assert np.array_equal(g.labels, o["labels"]), f"{name}: labels"
    assert np.array_equal(_bits(g.centroids), _bits(o["centroids"])), f"{name}: centroids"
    assert g.history == o["history"], f"{name}: history"


@pytest.mark.parametrize("name,seed,d,n,h,f32", _cases(), ids=[c[0] for c in _cases()])
def test_fuzz_default_and_global(engine, name, seed, d, n, h, f32):
    rng = np.random.default_rng(seed)
    X = _mixture(rng, n, d).astype(np.float32 if f32 else np.float64)
    _check(engine, X, h, 0, name)
    _check(engine, X, h, G.GS_DEBUG_GLOBAL_PATH, name + "-global")


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_batched_frames(engine, seed):
    rng = np.random.default_rng(500 + seed)
    B, n, d = int(rng.integers(2, 6)), int(rng.integers(200, 3000)), 3
    h = float(rng.uniform(0.2, 0.5))
    X = np.stack([_mixture(rng, n, d) for _ in range(B)]).astype(np.float32)
    rb = engine.run_batch(X, G.EngineConfig(h, 300))
    for f in range(B):
        o = O.run(X[f].astype(np.float64), h, 300, O.BUILD_FIXED)
        assert np.array_equal(rb.labels[f], o["labels"]), f"frame {f}"
        assert rb.iterations[f] == o["iterations"]
        assert np.array_equal(_bits(rb.centroids[f]), _bits(o["centroids"])), f"frame {f}"


@pytest.mark.parametrize("d", [2, 5])
def test_fuzz_batched_frames_global_path(engine, d):
    """Batched frames on the forced global path (cluster sweep d <= 3, dataflow sweep d > 3),
    frames finishing at different iterations (frozen frames' cells stay in the sweep)."""
    rng = np.random.default_rng(900 + d)
    B, n = 4, 1500
    frames = [_mixture(rng, n, d) for _ in range(B - 1)] + [np.full((n, d), 0.25)]
    X = np.stack(frames).astype(np.float64)
    h = 0.45
    rb = engine.run_batch(X, G.EngineConfig(h, 300, debug_flags=G.GS_DEBUG_GLOBAL_PATH))
    for f in range(B):
        o = O.run(X[f], h, 300, O.BUILD_FIXED)
        assert rb.iterations[f] == o["iterations"], f
        assert np.array_equal(rb.labels[f], o["labels"]), f
        assert np.array_equal(_bits(rb.centroids[f]), _bits(o["centroids"])), f


def _high_d_cases():
    """d = 7..12 (SPEC.md:96's documented limit): the dense cell grid holds the key box (apron 2
    per side), so the data spans few cells per dimension -- 3 (d 7), 2 (d 8-10), 2 in one
    dimension (d 11), one cell (d 12: 5^12 cells)."""
    out = []
    for d, span, seeds in ((7, 3, 3), (8, 2, 3), (9, 2, 2), (10, 2, 2), (11, 1, 1), (12, 0, 1)):
        for s in range(seeds):
            out.append((f"d{d}-s{s}", d, span, 700 + 10 * d + s))
    return out


@pytest.mark.parametrize("name,d,span,seed", _high_d_cases(), ids=[c[0] for c in _high_d_cases()])
def test_fuzz_high_dimensions(engine, name, d, span, seed):
    """K2/K3/K8/K7 and the global path's census/scan/Kahn sweep (d >= 7) bit-exact vs the oracle."""
    rng = np.random.default_rng(seed)
    h = 1.0
    n = 600
    k = 3
    centres = rng.uniform(0.3, 0.7, (k, d))
    if span >= 2:
        centres[:, :] = rng.uniform(0.3, span - 0.3, (k, d))
    elif span == 1:
        centres[:, 0] = rng.uniform(0.3, 1.7, k)
    lab = rng.integers(0, k, n)
    X = centres[lab] + 0.08 * rng.standard_normal((n, d))
    lo = 0.01
    hi = np.full(d, 0.99) if span == 0 else np.full(d, max(span, 1) - 0.01)
    if span == 1:
        hi[:] = 0.99
        hi[0] = 1.99
    X = np.clip(X, lo, hi)
    _check(engine, X, h, 0, name)
    _check(engine, X, h, G.GS_DEBUG_GLOBAL_PATH, name + "-global")


def test_high_dimension_key_range_refused(engine):
    """A d = 12 dataset whose key box exceeds the dense grid is refused loudly (KEY_RANGE ->
    InvalidParameterError), never approximated."""
    rng = np.random.default_rng(5)
    X = rng.uniform(0.0, 3.0, (200, 12))
    with pytest.raises(G.InvalidParameterError):
        engine.run(X, G.EngineConfig(1.0, 50))


@pytest.mark.parametrize("flags", ["flow", "levels", "single"])
@pytest.mark.parametrize("d", [2, 3, 5])
def test_fuzz_sweep_schedules(engine, d, flags):
    """Every global-path sweep variant (dataflow cluster sweep, level-synchronous cluster sweep,
    single-CTA sweep) on the same inputs, bit-exact vs the oracle."""
    fl = {"flow": G.GS_DEBUG_SWEEP_FLOW, "levels": G.GS_DEBUG_SWEEP_LEVELS,
          "single": G.GS_DEBUG_SWEEP_SINGLE}[flags]
    for seed in range(3):
        rng = np.random.default_rng(4000 + 10 * d + seed)
        n = 4000 if d <= 3 else 2000
        X = _mixture(rng, n, d).astype(np.float32)
        h = 0.3 if d <= 3 else 0.5
        _check(engine, X, h, G.GS_DEBUG_GLOBAL_PATH | fl, f"d{d}-{flags}-{seed}")
