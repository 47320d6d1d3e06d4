"""Multi-process (gloo) tests of the multi-GPU drivers: the sharded result must equal the
single-process result frame for frame / point for point.  The CPU tests use the oracle (test
infrastructure) as each rank's clusterer; the GPU tests run the engine on every rank."""
import os
import socket

import numpy as np
import pytest

from paper_2206_02200_b200.dist import frame_shard


def test_frame_shard_partitions():
    for nf in (0, 1, 5, 256, 257):
        for world in (1, 2, 3, 4, 8):
            spans = [frame_shard(nf, world, r) for r in range(world)]
            assert sum(c for _, c in spans) == nf
            pos = 0
            for s, c in spans:
                assert s == pos
                pos += c
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        frame_shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames(first, count):
    from paper_2206_02200_b200 import configs as CF
    return CF.generate("cfg4", scale=0.02, frames=count, frame0=first)


def _cluster(X):
    from oracle import oracle as O
    labels, k, it = [], [], []
    for f in range(X.shape[0]):
        r = O.run(X[f].astype(np.float64), 0.08, 50, O.BUILD_FIXED)
        labels.append(r["labels"])
        k.append(r["k"])
        it.append(r["iterations"])
    return np.stack(labels), np.array(k), np.array(it)


def _worker(rank, world, port, nframes, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_02200_b200.dist import max_over_ranks, run_frames
    out = run_frames(_frames, _cluster, nframes)
    t = max_over_ranks(float(rank + 1))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), labels=out["labels"], first=out["first"],
             count=out["count"], k_all=out["k_all"], it_all=out["iterations_all"], tmax=t)
    dist.destroy_process_group()


def _cluster_engine(X):
    from paper_2206_02200_b200 import gridshift as G
    eng = G.Engine(0)
    r = eng.run_batch(X, G.EngineConfig(0.08, 50))
    eng.close()
    return r.labels, np.asarray(r.k), np.asarray(r.iterations)


def _engine_worker(rank, world, port, nframes, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_02200_b200.dist import run_frames
    out = run_frames(_frames, _cluster_engine, nframes)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), labels=out["labels"], first=out["first"],
             count=out["count"], k_all=out["k_all"], it_all=out["iterations_all"])
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_frames_multi_rank_engine_matches_oracle(tmp_path, world):
    """Frame sharding with the ENGINE as each rank's clusterer (all ranks on cuda:0: frames
    are independent, so the ranks' kernels never wait on each other): every frame of every
    shard equals the oracle, and the gathered per-frame k / iterations are complete."""
    import torch.multiprocessing as mp
    nframes = 7
    mp.spawn(_engine_worker, args=(world, _free_port(), nframes, str(tmp_path)), nprocs=world,
             join=True)
    ref_labels, ref_k, ref_it = _cluster(_frames(0, nframes))
    seen = 0
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        f0, c = int(z["first"]), int(z["count"])
        assert np.array_equal(z["labels"], ref_labels[f0:f0 + c])
        assert np.array_equal(z["k_all"], ref_k)
        assert np.array_equal(z["it_all"], ref_it)
        seen += c
    assert seen == nframes


def test_two_rank_gloo_matches_single_process(tmp_path):
    import torch.multiprocessing as mp
    nframes, world = 5, 2
    mp.spawn(_worker, args=(world, _free_port(), nframes, str(tmp_path)), nprocs=world,
             join=True)
    ref_labels, ref_k, ref_it = _cluster(_frames(0, nframes))
    seen = 0
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        f0, c = int(z["first"]), int(z["count"])
        assert np.array_equal(z["labels"], ref_labels[f0:f0 + c])
        assert np.array_equal(z["k_all"], ref_k)
        assert np.array_equal(z["it_all"], ref_it)
        assert float(z["tmax"]) == float(world)   # max over ranks
        seen += c
    assert seen == nframes


# ---------------------------------------------------------------- one cloud over ranks (cfg5)
class CpuShardEngine:
    """CPU replica of the engine's gs_shard_* calls (test infrastructure: numpy fixed-point
    binning exactly as gs_fixq / gs_fix_centroid, then the oracle's iterate_once loop), so the
    rank orchestration in dist.run_cloud runs without a GPU."""
    APRON = 2

    def shard_keybounds(self, X, h):
        k = np.floor(np.asarray(X, np.float64) / h)
        return k.min(0).astype(np.int64), k.max(0).astype(np.int64)

    def _geometry(self, klo, khi):
        ext = (khi - klo + 1 + 2 * self.APRON).astype(np.int64)
        strides = np.ones(len(ext), np.int64)
        for c in range(len(ext) - 2, -1, -1):
            strides[c] = strides[c + 1] * ext[c + 1]
        return klo - self.APRON, ext, strides

    def shard_bin(self, X, h, n_global, klo, khi):
        from oracle import oracle as O
        X = np.asarray(X, np.float64)
        F = O.fixed_shift(n_global, h)
        kmin, ext, strides = self._geometry(np.asarray(klo), np.asarray(khi))
        k = np.floor(X / h).astype(np.int64)
        L = ((k - kmin) * strides).sum(1)
        q = np.rint((X - k.astype(np.float64) * h) * np.ldexp(1.0, F)).astype(np.int64)
        keys, inv = np.unique(L, return_inverse=True)
        counts = np.bincount(inv, minlength=len(keys)).astype(np.uint32)
        sums = np.zeros((len(keys), X.shape[1]), np.int64)
        np.add.at(sums, inv, q)
        self.h, self.F, self.kmin, self.ext, self.strides, self.slot = h, F, kmin, ext, strides, L
        return keys.astype(np.uint32), counts, sums

    def shard_run(self, keys, counts, sums, n_shard, cfg):
        from oracle import oracle as O
        from paper_2206_02200_b200.gridshift import ClusterLabeling
        L, inv = np.unique(keys.astype(np.int64), return_inverse=True)
        cnt = np.bincount(inv, weights=None, minlength=len(L)).astype(np.int64) * 0
        np.add.at(cnt, inv, counts.astype(np.int64))
        qs = np.zeros((len(L), sums.shape[1]), np.int64)
        np.add.at(qs, inv, sums)
        kk = (L[:, None] // self.strides) % self.ext + self.kmin
        cent = kk.astype(np.float64) * self.h + (qs.astype(np.float64) / cnt[:, None]) * np.ldexp(1.0, -self.F)
        root = np.arange(len(L))
        state = dict(keys=kk, counts=cnt, centroids=cent)
        it, conv = 0, False
        while True:  # do-while: converged, unchanged, or max_iter
            r = O.iterate_once(state["keys"], state["counts"], state["centroids"], self.h)
            root = r["parent"][root]
            it += 1
            state = r
            conv = r["converged"] or not r["changed"]
            if conv or it >= cfg.max_iterations:
                break
        labels = root[np.searchsorted(L, self.slot)].astype(np.int32)
        return ClusterLabeling(labels, state["centroids"], it, conv)


def _cloud(n=6000, seed=5, kind="small"):
    if kind == "cfg5":  # a 3% cfg5 cloud: m0 in the tens of thousands (the global path first)
        from paper_2206_02200_b200 import configs as CF
        return CF.generate("cfg5", scale=0.03)[0]
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0, 10, size=(6, 3))
    lab = rng.integers(0, 6, n)
    return (centres[lab] + rng.normal(0, 0.6, size=(n, 3))).astype(np.float32)


def _cloud_worker(rank, world, port, outdir, use_gpu, kind="small"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_02200_b200.dist import point_shard, run_cloud
    X = _cloud(kind=kind)
    p0, c = point_shard(X.shape[0], world, rank)
    if use_gpu:
        from paper_2206_02200_b200 import gridshift as G
        eng = G.Engine(0)
    else:
        eng = CpuShardEngine()
    r = run_cloud(eng, X[p0:p0 + c], 1.0, 100)
    np.savez(os.path.join(outdir, f"c{rank}.npz"), labels=r.labels, cent=r.centroids,
             it=r.iterations, p0=p0, c=c)
    dist.destroy_process_group()


def _check_cloud(outdir, world, ref_labels, ref_cent, ref_it):
    seen = 0
    for r in range(world):
        z = np.load(os.path.join(outdir, f"c{r}.npz"))
        p0, c = int(z["p0"]), int(z["c"])
        assert np.array_equal(z["labels"], ref_labels[p0:p0 + c])
        assert np.array_equal(z["cent"].view(np.int64), ref_cent.view(np.int64))
        assert int(z["it"]) == ref_it
        seen += c
    assert seen == len(ref_labels)


def test_cloud_two_rank_gloo_matches_single_process(tmp_path):
    """One cloud over 2 gloo ranks (CPU replica of the shard calls): every rank's labels and
    the common centroids equal the oracle's single-process run bit for bit."""
    import torch.multiprocessing as mp
    from oracle import oracle as O
    world = 2
    mp.spawn(_cloud_worker, args=(world, _free_port(), str(tmp_path), False), nprocs=world,
             join=True)
    ref = O.run(_cloud().astype(np.float64), 1.0, 100, O.BUILD_FIXED)
    _check_cloud(str(tmp_path), world, ref["labels"], ref["centroids"], ref["iterations"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind,world", [("small", 2), ("small", 3), ("cfg5", 2)])
def test_cloud_multi_rank_engine_matches_single_gpu(tmp_path, kind, world):
    """The engine's gs_shard_* path: R ranks (all on cuda:0, host-side gloo exchange -- the
    ranks' kernels never wait on each other) equal one GPU clustering the whole cloud."""
    import torch.multiprocessing as mp
    from paper_2206_02200_b200 import gridshift as G
    mp.spawn(_cloud_worker, args=(world, _free_port(), str(tmp_path), True, kind), nprocs=world,
             join=True)
    eng = G.Engine(0)
    ref = eng.run(_cloud(kind=kind), G.EngineConfig(1.0, 100))
    _check_cloud(str(tmp_path), world, ref.labels, ref.centroids, ref.iterations)
    eng.close()


# ---------------------------------------------------------------- gs_dist (one process, R ranks)
def _blobs2(n=5000, seed=9):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0, 8, size=(5, 2))
    return c[rng.integers(0, 5, n)] + rng.normal(0, 0.5, size=(n, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,world", [("small", 2), ("small", 3), ("blobs2", 2), ("blobs2", 4),
                                        ("cfg5", 2), ("cfg5", 3)])
def test_dist_slabs_match_single_gpu(kind, world):
    """gs_dist_run_slabs: one cloud, points sharded over R loopback ranks on cuda:0, cells owned
    by dim-0 slabs with the per-iteration halo exchange (swept lower layer, old upper layer),
    migration of rehomed cells and the ordered merge -- labels, centroid bits, iterations and
    history equal to one GPU clustering the whole cloud."""
    from paper_2206_02200_b200 import gridshift as G
    X = _blobs2() if kind == "blobs2" else _cloud(kind=kind)
    h = 0.4 if kind == "blobs2" else 1.0
    cfg = G.EngineConfig(h, 100, record_history=True)
    eng = G.Engine(0)
    ref = eng.run(X, cfg)
    eng.close()
    D = G.Dist([0] * world)
    got = D.run_slabs(X, cfg)
    D.close()
    assert got.iterations == ref.iterations
    assert got.converged == ref.converged
    assert np.array_equal(got.labels, ref.labels)
    assert np.array_equal(got.centroids.view(np.int64), ref.centroids.view(np.int64))
    assert got.history == ref.history


@pytest.mark.gpu
def test_dist_frames_match_single_gpu():
    """gs_dist_run_frames: frame blocks per rank (one host thread each), equal to one batch."""
    from paper_2206_02200_b200 import gridshift as G
    X = _frames(0, 7)
    cfg = G.EngineConfig(0.08, 50)
    eng = G.Engine(0)
    ref = eng.run_batch(X, cfg)
    eng.close()
    D = G.Dist([0, 0, 0])
    got = D.run_frames(X, cfg)
    D.close()
    assert np.array_equal(got.labels, ref.labels)
    assert np.array_equal(got.k, ref.k) and np.array_equal(got.iterations, ref.iterations)
    for f in range(X.shape[0]):
        assert np.array_equal(got.centroids[f].view(np.int64), ref.centroids[f].view(np.int64))
