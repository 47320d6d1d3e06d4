"""Multi-process (world_size 2, gloo, CPU) tests of the frame-sharded driver: the sharded
result must equal the single-process result frame for frame.  The per-rank clustering here
is the CPU oracle (test infrastructure) so the test runs without a GPU; on the GPU box the
same driver calls the engine (bench.py under torchrun)."""
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
