"""GPU engine vs the CPU oracle on identical seeded inputs.

Two oracles (oracle/gs_oracle.cpp):
  * build mode "fixed" shares the engine's fixed-point binning definition; everything after
    binning is the SPEC's sweep/merge/termination.  The GPU must match it BIT-EXACTLY:
    keys, counts, centroids, parent structure, iterations, labels.
  * build mode "spec" is the literal SPEC (incremental-mean binning).  The GPU must match it
    within north_star's tolerances: centroids <= 1e-5 relative, labels >= 99.9 % after an
    optimal permutation match.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2206_02200_b200 import configs as CF
from paper_2206_02200_b200 import gridshift as G
from tests.parity_util import matched_agreement, oracle_states

pytestmark = pytest.mark.gpu

CENTROID_RTOL = 1e-5      # north_star: centroids within 1e-5 relative
LABEL_AGREEMENT = 0.999   # north_star: >= 99.9 % after optimal permutation match


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def assert_state_equal(gpu, ora, what=""):
    assert np.array_equal(gpu[0], ora[0]), f"{what}: keys differ"
    assert np.array_equal(gpu[1], ora[1]), f"{what}: counts differ"
    assert np.array_equal(_bits(gpu[2]), _bits(ora[2])), f"{what}: centroids differ (bits)"


def small_inputs():
    """(name, X, h) small cases: configs at reduced size plus adversarial ones."""
    out = []
    out.append(("cfg1", CF.generate("cfg1")[0], 0.5))
    out.append(("cfg2", CF.generate("cfg2")[0], 0.08))
    out.append(("cfg3_small", CF.generate("cfg3", scale=0.05)[0], 0.06))
    out.append(("cfg4_frame", CF.generate("cfg4", scale=0.25, frames=1)[0], 0.08))
    out.append(("cfg5_small", CF.generate("cfg5", scale=1 / 256)[0], 1.0))
    rng = np.random.default_rng(1)
    # boundary points: exact multiples of h, negatives, duplicates
    g = np.repeat(np.arange(-6, 7, dtype=np.float64) * 0.25, 3)
    out.append(("boundaries", np.stack([g, g[::-1]], 1), 0.25))
    out.append(("negative", rng.normal(-50.0, 3.0, size=(3000, 3)), 1.5))
    out.append(("duplicates", np.repeat(rng.uniform(0, 1, size=(20, 2)), 50, 0), 0.1))
    out.append(("d1", rng.normal(0, 1, size=(5000, 1)), 0.2))
    out.append(("d4", rng.normal(0, 1, size=(4000, 4)), 0.6))
    out.append(("d6", rng.normal(0, 1, size=(3000, 6)), 0.9))
    out.append(("single", np.array([[1.0, 2.0, 3.0]]), 0.3))
    # fp32 corner cases of the fast key path: signed zeros, exact multiples of h and their
    # fp32 neighbours, values whose x/h lands within an ulp of an integer
    z = np.array([-0.0, 0.0, -0.0, 0.0], np.float32)
    m = (np.arange(-40, 41) * np.float32(0.08)).astype(np.float32)
    near = np.concatenate([m, np.nextafter(m, np.float32(1e9)), np.nextafter(m, np.float32(-1e9))])
    g3 = np.stack([np.resize(np.concatenate([z, near]), 400)] * 3, 1)
    g3[:, 1] = g3[::-1, 1]
    out.append(("f32_corners", np.ascontiguousarray(g3.astype(np.float32)), 0.08))
    return out


@pytest.mark.parametrize("case", small_inputs(), ids=lambda c: c[0])
def test_build_bit_exact(engine, case):
    name, X, h = case
    g = engine.debug_build(X, h)
    o = O.build_grid(X.astype(np.float64), h, O.BUILD_FIXED)
    assert_state_equal(g[:3], o[:3], name)
    assert np.array_equal(g[3], o[3]), "point -> cell rank differs"


@pytest.mark.parametrize("case", small_inputs(), ids=lambda c: c[0])
def test_state_injection_bit_exact(engine, case):
    """Feed the GPU the oracle's iteration-t state; iteration t+1 must be identical bitwise."""
    name, X, h = case
    states = oracle_states(X.astype(np.float64), h, steps=30)
    for t, (keys, cnt, cen) in enumerate(states):
        o = O.iterate_once(keys, cnt, cen, h)
        g = engine.debug_iterate_once(keys, cnt, cen, h)
        assert np.array_equal(_bits(g["swept"]), _bits(o["swept"])), f"{name} t={t}: sweep"
        assert_state_equal((g["keys"], g["counts"], g["centroids"]),
                           (o["keys"], o["counts"], o["centroids"]), f"{name} t={t}")
        assert np.array_equal(g["parent"], o["parent"]), f"{name} t={t}: parent"
        assert g["changed"] == o["changed"] and g["converged"] == o["converged"]
        assert g["maxdisp"] == o["maxdisp"]


@pytest.mark.parametrize("case", small_inputs(), ids=lambda c: c[0])
def test_state_injection_resident_bit_exact(engine, case):
    """K8 state injection: the oracle's iteration-t state fed to ONE iteration of the
    CTA-resident engine (capacity permitting) must give the oracle's iteration t+1 bitwise --
    cells, parent map, max displacement and the do-while exit flag."""
    name, X, h = case
    states = oracle_states(X.astype(np.float64), h, steps=30)
    done = 0
    for t, (keys, cnt, cen) in enumerate(states):
        try:
            g = engine.debug_resident_once(keys, cnt, cen, h)
        except G.InvalidParameterError:  # beyond K8's capacity: the global path's state
            continue
        o = O.iterate_once(keys, cnt, cen, h)
        assert_state_equal((g["keys"], g["counts"], g["centroids"]),
                           (o["keys"], o["counts"], o["centroids"]), f"{name} t={t}")
        assert np.array_equal(g["parent"], o["parent"]), f"{name} t={t}: parent"
        assert g["stop"] == (o["converged"] or not o["changed"]), f"{name} t={t}: exit flag"
        assert g["maxdisp"] == o["maxdisp"], f"{name} t={t}: max displacement"
        done += 1
    assert done > 0


def _check_run(engine, X, h, max_iter, name, flags=0):
    cfg = G.EngineConfig(h, max_iter, record_history=True, debug_flags=flags)
    g = engine.run(X, cfg)
    ofx = O.run(X.astype(np.float64), h, max_iter, O.BUILD_FIXED)
    # bit-exact against the fixed-point-build oracle
    assert g.iterations == ofx["iterations"], name
    assert g.converged == ofx["converged"]
    assert np.array_equal(g.labels, ofx["labels"]), f"{name}: labels"
    assert np.array_equal(_bits(g.centroids), _bits(ofx["centroids"])), f"{name}: centroids"
    assert g.history == ofx["history"], f"{name}: history"
    # tolerance parity against the literal SPEC oracle
    osp = O.run(X.astype(np.float64), h, max_iter, O.BUILD_SPEC)
    agree, match = matched_agreement(g.labels, osp["labels"])
    assert agree >= LABEL_AGREEMENT, f"{name}: label agreement {agree}"
    for a, b in match.items():
        np.testing.assert_allclose(g.centroids[a], osp["centroids"][b], rtol=CENTROID_RTOL,
                                   atol=CENTROID_RTOL * np.abs(X).max())
    return g


@pytest.mark.parametrize("case", small_inputs(), ids=lambda c: c[0])
def test_run_parity(engine, case):
    """Default schedule: CTA-resident engine (K8), global path first when a frame is large."""
    name, X, h = case
    _check_run(engine, X, h, 300, name)


@pytest.mark.parametrize("case", small_inputs(), ids=lambda c: c[0])
def test_run_parity_global_path(engine, case):
    """Every iteration on the multi-CTA global path (K4/K5 kernels)."""
    name, X, h = case
    _check_run(engine, X, h, 300, name, flags=G.GS_DEBUG_GLOBAL_PATH)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_config_full_size(engine, name):
    cfg = CF.CONFIGS[name]
    X = CF.generate(name)[0]
    _check_run(engine, X, cfg.h, cfg.max_iter, name)


def test_batched_frames_heterogeneous(engine):
    """Frames finish at different iterations; each must equal its own independent run."""
    n = 4000
    rng = np.random.default_rng(3)
    frames = [
        np.full((n, 3), 0.5, np.float32),                                   # one cell, 1 iter
        CF.generate("cfg2", scale=n / 154401.0)[0][:n].astype(np.float32),  # image
        rng.normal(0, 0.3, size=(n, 3)).astype(np.float32),                 # one blob
        rng.uniform(0, 1, size=(n, 3)).astype(np.float32),                  # uniform cube
    ]
    frames[1] = np.resize(frames[1], (n, 3))
    X = np.stack(frames)
    h = 0.08
    r = engine.run_batch(X, G.EngineConfig(h, 100, record_history=True))
    for f in range(len(frames)):
        o = O.run(X[f].astype(np.float64), h, 100, O.BUILD_FIXED)
        assert r.k[f] == o["k"] and r.iterations[f] == o["iterations"], f
        assert np.array_equal(r.labels[f], o["labels"]), f
        assert np.array_equal(_bits(r.centroids[f]), _bits(o["centroids"])), f
        assert r.history[f] == o["history"]


def test_cfg4_frames_sampled(engine):
    """cfg4 at full frame size, 16 consecutive frames batched; every frame vs the oracle."""
    cfg = CF.CONFIGS["cfg4"]
    X = CF.generate("cfg4", frames=16, frame0=100)
    r = engine.run_batch(X, G.EngineConfig(cfg.h, cfg.max_iter))
    for f in range(X.shape[0]):
        o = O.run(X[f].astype(np.float64), cfg.h, cfg.max_iter, O.BUILD_FIXED)
        assert r.k[f] == o["k"] and r.iterations[f] == o["iterations"]
        assert np.array_equal(r.labels[f], o["labels"])
        assert np.array_equal(_bits(r.centroids[f]), _bits(o["centroids"]))


def test_determinism(engine):
    X = CF.generate("cfg2")[0]
    a = engine.run(X, G.EngineConfig(0.08, 100))
    b = engine.run(X, G.EngineConfig(0.08, 100))
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(_bits(a.centroids), _bits(b.centroids))


def test_random_property_bit_exact(engine):
    rng = np.random.default_rng(11)
    for trial in range(25):
        d = int(rng.integers(1, 6))
        n = int(rng.integers(1, 3000))
        X = rng.normal(size=(n, d)) * rng.uniform(0.1, 5) + rng.uniform(-20, 20)
        if trial % 3 == 0:
            X = X.astype(np.float32)
        h = float(rng.uniform(0.05, 2.0))
        Xd = np.asarray(X, np.float64)
        ext = np.floor(Xd.max(0) / h) - np.floor(Xd.min(0) / h) + 5   # engine's box + apron
        if np.prod(ext) > 2 ** 28:
            # the dense cell grid covers boxes up to 2^28 cells; wider boxes are refused loudly
            with pytest.raises(G.InvalidParameterError):
                engine.run(X, G.EngineConfig(h, 500))
            continue
        g = engine.run(X, G.EngineConfig(h, 500))
        o = O.run(np.asarray(X, np.float64), h, 500, O.BUILD_FIXED)
        assert np.array_equal(g.labels, o["labels"]), trial
        assert np.array_equal(_bits(g.centroids), _bits(o["centroids"])), trial
        assert g.iterations == o["iterations"]


def test_graph_replay_pinned_buffers():
    """Repeated runs of one shape with pinned host buffers take the optimistic path replayed
    from a CUDA graph; every replay must still equal the oracle bit for bit."""
    import torch
    X = CF.generate("cfg2")[0]
    Xp = torch.from_numpy(X).pin_memory()
    lab = torch.empty(X.shape[0], dtype=torch.int32).pin_memory()
    o = O.run(X.astype(np.float64), 0.08, 100, O.BUILD_FIXED)
    eng = G.Engine(0)
    for rep in range(4):
        k, it, cv = eng.run_raw(Xp.data_ptr(), X.shape[0], 3, G.GS_F32, 1, False,
                                G.EngineConfig(0.08, 100), lab.data_ptr())
        assert int(k[0]) == o["k"] and int(it[0]) == o["iterations"], rep
        assert np.array_equal(lab.numpy(), o["labels"]), rep
        cen = eng.centroids(0, int(k[0]), 3)
        assert np.array_equal(_bits(cen), _bits(o["centroids"])), rep
    # device-resident input and outputs (the bench's `value` configuration)
    Xd = Xp.cuda()
    labd = torch.empty(X.shape[0], dtype=torch.int32, device="cuda")
    for rep in range(3):
        eng.run_raw(Xd.data_ptr(), X.shape[0], 3, G.GS_F32, 1, True, G.EngineConfig(0.08, 100),
                    labd.data_ptr(), device_outputs=True)
        assert np.array_equal(labd.cpu().numpy(), o["labels"]), rep
    eng.close()


@pytest.mark.gpu
def test_graph_replay_new_data_same_shape():
    """The cached graph is keyed on the shape, not on the data: a replay over points with a
    different key box (shifted, wider, narrower) and a different cell count must still equal
    the oracle bit for bit (the box, the frame ranges and the index layout come from the
    device, never from the capture)."""
    import torch
    base = CF.generate("cfg2", scale=0.2)[0].astype(np.float64)
    rng = np.random.default_rng(7)
    variants = [base, base * 0.5 + 0.25, base * 1.7 - 0.3, base + 3.0,
                rng.random(base.shape) * 0.3, base]
    eng = G.Engine(0)
    Xp = torch.empty(base.shape, dtype=torch.float64).pin_memory()
    lab = torch.empty(base.shape[0], dtype=torch.int32).pin_memory()
    for rep, X in enumerate(variants):
        Xp.copy_(torch.from_numpy(np.ascontiguousarray(X)))
        o = O.run(X, 0.08, 100, O.BUILD_FIXED)
        k, it, cv = eng.run_raw(Xp.data_ptr(), X.shape[0], 3, G.GS_F64, 1, False,
                                G.EngineConfig(0.08, 100), lab.data_ptr())
        assert int(k[0]) == o["k"] and int(it[0]) == o["iterations"], rep
        assert np.array_equal(lab.numpy(), o["labels"]), rep
        cen = eng.centroids(0, int(k[0]), 3)
        assert np.array_equal(_bits(cen), _bits(o["centroids"])), rep
    eng.close()


# ---------------------------------------------------------------- segmentation front end (§8(f)1)
def _u8_image(H=96, W=128, seed=3):
    """Voronoi regions of random colours + noise, quantised to 8 bits (a cfg2-like image)."""
    rng = np.random.default_rng(seed)
    sites = rng.uniform(0, 1, size=(10, 2)) * [H, W]
    cols = rng.integers(0, 256, size=(10, 3))
    yy, xx = np.mgrid[0:H, 0:W]
    reg = np.argmin(((yy[..., None] - sites[:, 0]) ** 2 + (xx[..., None] - sites[:, 1]) ** 2), -1)
    img = cols[reg] + rng.normal(0, 6, size=(H, W, 3))
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def _features(img, mode):
    H, W, _ = img.shape
    f = img.reshape(-1, 3).astype(np.float64) / 255.0       # channel / 255
    if mode == "rgbxy":
        yy, xx = np.mgrid[0:H, 0:W]
        f = np.concatenate([f, (xx.reshape(-1, 1) / (W - 1)), (yy.reshape(-1, 1) / (H - 1))], 1)
    return f


@pytest.mark.parametrize("mode,h", [("rgb", 0.08), ("rgbxy", 0.1)])
def test_u8_pixels_bit_exact(engine, mode, h):
    """8-bit pixels turned into features on the device (3 B/pixel read) equal the oracle run
    on the host-made features img / 255 (and x/(W-1), y/(H-1)) bit for bit."""
    img = _u8_image()
    g = engine.run_image(img, G.EngineConfig(h, 100), mode)
    o = O.run(_features(img, mode), h, 100, O.BUILD_FIXED)
    assert np.array_equal(g.labels, o["labels"])
    assert np.array_equal(_bits(g.centroids), _bits(o["centroids"]))
    assert g.iterations == o["iterations"]


def test_u8_spec_feature_examples(engine):
    """black -> (0,0,0), white -> (1,1,1); rgbxy pixel (1,0) of a 2x2 image
    -> x = 1, y = 0.  With h > 1 every pixel shares one cell whose fixed-point mean is exact
    here, so the single centroid is the mean of the features."""
    img = np.array([[[0, 0, 0], [255, 255, 255]], [[0, 0, 0], [255, 255, 255]]], np.uint8)
    g = engine.run_image(img, G.EngineConfig(4.0, 10), "rgbxy")
    assert g.centroids.shape == (1, 5)
    assert np.allclose(g.centroids[0], [0.5, 0.5, 0.5, 0.5, 0.5], rtol=0, atol=1e-15)


def test_render_mean_colours(engine):
    """render: every pixel gets its segment's centroid rgb * 255, rounded
    half-up; a 1-segment image renders uniform."""
    img = _u8_image()
    g = engine.run_image(img, G.EngineConfig(0.08, 100), "rgb")
    out = engine.render(0)
    col = np.clip(np.floor(g.centroids[:, :3] * 255.0 + 0.5), 0, 255).astype(np.uint8)
    assert np.array_equal(out, col[g.labels])
    flat = np.full((8, 8, 3), 77, np.uint8)
    g1 = engine.run_image(flat, G.EngineConfig(0.08, 20), "rgb")
    out1 = engine.render(0)
    assert len(g1.centroids) == 1 and (out1 == out1[0]).all()


def test_graph_replay_after_other_calls(engine):
    """The replayed graph has no memset: K7 leaves the control block clean.  Calls that use
    the block in between (debug build, shard binning, a failing run) must not leak state
    into the next replay."""
    import torch
    X = CF.generate("cfg2", scale=0.2)[0]
    o = O.run(X.astype(np.float64), 0.08, 100, O.BUILD_FIXED)
    Xp = torch.from_numpy(X).pin_memory()
    lab = torch.empty(X.shape[0], dtype=torch.int32).pin_memory()
    eng = G.Engine(0)

    def replay():
        k, it, cv = eng.run_raw(Xp.data_ptr(), X.shape[0], 3, G.GS_F32, 1, False,
                                G.EngineConfig(0.08, 100), lab.data_ptr())
        assert int(k[0]) == o["k"] and int(it[0]) == o["iterations"]
        assert np.array_equal(lab.numpy(), o["labels"])

    for _ in range(2):
        replay()
    eng.debug_build(X.astype(np.float64), 0.08)
    replay()
    lo, hi = eng.shard_keybounds(X, 0.08)
    eng.shard_bin(X, 0.08, X.shape[0], lo, hi)
    replay()
    bad = X.copy()
    bad[5, 1] = np.nan
    with pytest.raises(G.InvalidInputError):
        eng.run(bad, G.EngineConfig(0.08, 100))
    replay()
    eng.close()


def _tolerance_check(labels, centroids, osp, name, xmax):
    """north_star tolerances against the literal SPEC oracle (build mode 0): labels >= 99.9 %
    after an optimal permutation match, matched centroids within 1e-5 relative."""
    agree, match = matched_agreement(labels, osp["labels"])
    assert agree >= LABEL_AGREEMENT, f"{name}: label agreement {agree}"
    for a, b in match.items():
        np.testing.assert_allclose(centroids[a], osp["centroids"][b], rtol=CENTROID_RTOL,
                                   atol=CENTROID_RTOL * xmax, err_msg=name)
    return agree


def test_cfg5_full_size_bit_exact(engine):
    """cfg5 at its full size (64 M points, one cloud): global path (cluster sweeps) then K8,
    bit-exact against the fixed-point-build oracle (labels, centroids, iterations, history),
    and within north_star's tolerances of the literal SPEC oracle (mode 0)."""
    cfg = CF.CONFIGS["cfg5"]
    X = CF.generate("cfg5")[0]
    g = engine.run(X, G.EngineConfig(cfg.h, cfg.max_iter, record_history=True))
    Xd = X.astype(np.float64)
    del X
    o = O.run(Xd, cfg.h, cfg.max_iter, O.BUILD_FIXED)
    assert g.iterations == o["iterations"]
    assert np.array_equal(g.labels, o["labels"])
    assert np.array_equal(_bits(g.centroids), _bits(o["centroids"]))
    assert g.history == o["history"]
    del o
    osp = O.run(Xd, cfg.h, cfg.max_iter, O.BUILD_SPEC)
    _tolerance_check(g.labels, g.centroids, osp, "cfg5", float(np.abs(Xd).max()))


def test_cfg4_all_frames_bit_exact(engine):
    """cfg4 at its full size (256 frames of 640 x 480) in one batched call from host memory
    (the frame-group pipeline); every frame bit-exact vs the fixed-point-build oracle and
    within north_star's tolerances of the literal SPEC oracle (mode 0)."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    cfg = CF.CONFIGS["cfg4"]
    X = CF.generate("cfg4")
    r = engine.run_batch(X, G.EngineConfig(cfg.h, cfg.max_iter))

    def one(f):
        x = X[f].astype(np.float64)
        o = O.run(x, cfg.h, cfg.max_iter, O.BUILD_FIXED)
        assert r.k[f] == o["k"] and r.iterations[f] == o["iterations"], f
        assert np.array_equal(r.labels[f], o["labels"]), f
        assert np.array_equal(_bits(r.centroids[f]), _bits(o["centroids"])), f
        osp = O.run(x, cfg.h, cfg.max_iter, O.BUILD_SPEC)
        return _tolerance_check(r.labels[f], r.centroids[f], osp, f"frame {f}", 1.0)

    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        agree = list(ex.map(one, range(X.shape[0])))
    assert min(agree) >= LABEL_AGREEMENT


def test_frame_group_pipeline(engine):
    """Host batches are pipelined by frame groups (copy of group g+1 overlapping group g):
    forced on a small batch (groups of 2, an odd last group), results equal the whole-batch
    run and the oracle; centroids and history of every frame survive the grouping."""
    import torch
    X = CF.generate("cfg4", scale=0.05, frames=7)
    cfg = G.EngineConfig(0.08, 50, record_history=True)
    whole = engine.run_batch(X, G.EngineConfig(0.08, 50, record_history=True,
                                               debug_flags=G.GS_NO_PIPELINE))
    piped = engine.run_batch(X, G.EngineConfig(0.08, 50, record_history=True,
                                               debug_flags=G.GS_DEBUG_PIPELINE))
    assert np.array_equal(whole.labels, piped.labels)
    assert np.array_equal(whole.k, piped.k) and np.array_equal(whole.iterations, piped.iterations)
    for f in range(X.shape[0]):
        assert np.array_equal(_bits(whole.centroids[f]), _bits(piped.centroids[f])), f
        assert whole.history[f] == piped.history[f], f
        o = O.run(X[f].astype(np.float64), 0.08, 50, O.BUILD_FIXED)
        assert np.array_equal(piped.labels[f], o["labels"]), f
    # pinned host buffers: each group's labels go to a device staging buffer and leave by DMA on
    # a third stream while later groups run (two staging buffers: groups 2, 3 reuse them)
    Xp = torch.from_numpy(X).pin_memory()
    lab = torch.zeros(X.shape[:2], dtype=torch.int32).pin_memory()
    engine.run_raw(Xp.data_ptr(), X.shape[1], 3, G.GS_F32, X.shape[0], False,
                   G.EngineConfig(0.08, 50, debug_flags=G.GS_DEBUG_PIPELINE), lab.data_ptr())
    assert np.array_equal(lab.numpy(), whole.labels)
    # render serves the last group only
    with pytest.raises(G.InvalidParameterError):
        engine.render(0)


@pytest.mark.parametrize("n,batch", [(1003, 5), (4096, 3), (7, 2), (1, 4)])
def test_binning_ragged_frames(engine, n, batch):
    """Batched fp32 frames of ragged sizes (frame starts off the 16-byte grid, a frame smaller
    than a warp, single-point frames) with exact zeros and scattered values; every frame
    bit-exact against the oracle (labels, centroids, history)."""
    rng = np.random.default_rng(n * 31 + batch)
    base = CF.generate("cfg2", scale=0.05)[0].astype(np.float32)
    X = np.stack([np.resize(np.roll(base, 17 * f, 0), (n, 3)) for f in range(batch)])
    X[:, ::7] = rng.uniform(0, 1, size=X[:, ::7].shape).astype(np.float32)
    X[:, 1::11] = 0.0
    X = np.ascontiguousarray(X)
    a = engine.run_batch(X, G.EngineConfig(0.08, 50, record_history=True))
    for f in range(batch):
        o = O.run(X[f].astype(np.float64), 0.08, 50, O.BUILD_FIXED)
        assert np.array_equal(a.labels[f], o["labels"]), f
        assert np.array_equal(_bits(a.centroids[f]), _bits(o["centroids"])), f
        assert a.history[f] == o["history"], f


def test_misaligned_device_input(engine):
    """A device input pointer off the 16-byte grid gives the same labels as the host call."""
    import torch
    X = CF.generate("cfg4", scale=0.1, frames=3)
    B, n, d = X.shape
    buf = torch.zeros(X.size + 1, dtype=torch.float32, device="cuda")
    buf[1:] = torch.from_numpy(X.reshape(-1)).cuda()
    lab = torch.zeros((B, n), dtype=torch.int32, device="cuda")
    cfg = G.EngineConfig(0.08, 50)
    engine.run_raw(buf.data_ptr() + 4, n, d, G.GS_F32, B, True, cfg, lab.data_ptr(),
                   device_outputs=True)
    ref = engine.run_batch(X, cfg)
    assert np.array_equal(lab.cpu().numpy(), ref.labels)


def _xpath_cases():
    rng = np.random.default_rng(77)
    # fp32 image-like frame with values below 2^(23-F) (x*2^F not an integer: the slow branch
    # of the X path), denormals, signed zeros and small negatives (key -1, |x| < h/2)
    X = rng.uniform(-0.3, 1.0, size=(20000, 3)).astype(np.float32)
    X[::5, 0] = rng.uniform(0, 2.0 ** -20, size=X[::5, 0].shape).astype(np.float32)
    X[1::7, 1] = -rng.uniform(0, 2.0 ** -24, size=X[1::7, 1].shape).astype(np.float32)
    X[2::11, 2] = np.float32(1e-40)
    X[3::13] = -0.0
    yield "tiny", X, 0.08
    # a key box whose RN(k h) 2^F has fraction exactly 1/2 (F = 45, h = 0.5 + 2^-46, k = 1): the
    # X path is refused and the dense table takes the generic fp64 path
    Y = rng.uniform(0.0, 3.0, size=(65536, 3)).astype(np.float32)
    yield "tie_box", Y, 0.5 + 2.0 ** -46


@pytest.mark.parametrize("case", list(_xpath_cases()), ids=lambda c: c[0])
def test_binning_x_path_edges(engine, case):
    """K2's fp32 X path (dense tables sum x*2^F and take count * RHE(RN(k h) 2^F) at the
    flush) against the oracle's fixed-point build: its slow branch and its refusal."""
    name, X, h = case
    if name == "tie_box":
        assert G.fixed_shift(len(X), h) == 45
    g = engine.debug_build(X, h)
    o = O.build_grid(X.astype(np.float64), h, O.BUILD_FIXED)
    assert_state_equal(g[:3], o[:3], name)
    assert np.array_equal(g[3], o[3]), "point -> cell rank differs"
    r = engine.run(X, G.EngineConfig(h, 30))
    ro = O.run(X.astype(np.float64), h, 30, O.BUILD_FIXED)
    assert np.array_equal(r.labels, ro["labels"])
    assert np.array_equal(_bits(r.centroids), _bits(ro["centroids"]))


def _component_clouds():
    rng = np.random.default_rng(2206)
    # 600 small separated clumps (3-D, h = 1): far more components of >= 2 cells than SMs, so
    # k_sweep_comp's CTAs take several components each from the device-side ticket
    cen = rng.choice(40 ** 3, size=600, replace=False)
    cen = np.stack([cen // 1600, (cen // 40) % 40, cen % 40], 1) * 6.0
    many = (cen[:, None, :] + rng.normal(0, 0.7, size=(600, 40, 3))).reshape(-1, 3)
    yield "many_components", many, 1.0
    # one connected slab of ~70 K cells next to a few clumps: the plan does not fit a CTA, the
    # component launch is a no-op and the cluster sweep runs instead
    slab = rng.uniform(0, 1, size=(400000, 3)) * [260.0, 260.0, 1.0]
    yield "oversized_component", np.concatenate([slab, many[:4000] + [0, 0, 40.0]]), 1.0


@pytest.mark.parametrize("case", list(_component_clouds()), ids=lambda c: c[0])
def test_component_sweep_tickets_and_fallback(engine, case):
    """The global path's component sweep reads its plan on the device (the host reads it while
    the sweep runs): more components than CTAs, and a component too large for a CTA."""
    name, X, h = case
    cfg = G.EngineConfig(h, 60, record_history=True, debug_flags=G.GS_DEBUG_GLOBAL_PATH)
    g = engine.run(X, cfg)
    o = O.run(X, h, 60, O.BUILD_FIXED)
    assert g.iterations == o["iterations"], name
    assert np.array_equal(g.labels, o["labels"]), name
    assert np.array_equal(_bits(g.centroids), _bits(o["centroids"])), name
    assert g.history == o["history"], name


def test_large_pinned_outputs_by_dma():
    """Pinned label arrays over 16 MB leave through a device buffer and one DMA copy (inside the
    replayed graph), smaller ones are written by K7 directly: a 5.3 M-point cloud and an image
    batch, three runs each (first synchronous, then graph replays), against the oracle."""
    import torch
    eng = G.Engine(0)
    X = CF.generate("cfg5", scale=1 / 12)[0]
    assert X.shape[0] * 4 > (16 << 20)
    Xp = torch.from_numpy(X).pin_memory()
    lab = torch.empty(X.shape[0], dtype=torch.int32).pin_memory()
    o = O.run(X.astype(np.float64), 1.0, 100, O.BUILD_FIXED)
    for rep in range(3):
        lab.fill_(-7)
        k, it, cv = eng.run_raw(Xp.data_ptr(), X.shape[0], 3, G.GS_F32, 1, False,
                                G.EngineConfig(1.0, 100), lab.data_ptr())
        assert int(k[0]) == o["k"] and int(it[0]) == o["iterations"], rep
        assert np.array_equal(lab.numpy(), o["labels"]), rep
    eng.close()
