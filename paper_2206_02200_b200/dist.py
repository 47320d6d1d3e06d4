"""Multi-GPU drivers, one process per GPU (torchrun).

* Independent frames (cfg4; independent runs may execute concurrently with
  fully isolated state): frames are partitioned into contiguous blocks, each rank clusters its
  block through its own engine, and nothing crosses the data path -- the only collectives are
  the timing max-reduction and an optional gather of per-frame results for reporting.
* One large cloud (cfg5): points are partitioned into contiguous shards; each rank bins its
  shard into partial cells of the global key box (one all-reduce of key bounds and point
  counts), the partial cells are all-gathered (the one data exchange: integer counts and
  fixed-point sums, so the merge is exact in any order), and every rank runs the identical
  deterministic iteration on the merged cells and labels its own points.  The result is
  bit-identical to one GPU clustering the whole cloud.
"""
from __future__ import annotations

from typing import Callable, List, Tuple

import numpy as np


def frame_shard(nframes: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced block of frames owned by `rank`: (first frame, count)."""
    if world < 1 or not (0 <= rank < world) or nframes < 0:
        raise ValueError("bad shard request")
    base, rem = divmod(nframes, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def max_over_ranks(value: float) -> float:
    """Device-timed durations are reported as the max over ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_frames(X_all_frames_fn: Callable[[int, int], np.ndarray],
               cluster_fn: Callable[[np.ndarray], Tuple[np.ndarray, np.ndarray, np.ndarray]],
               nframes: int, gather: bool = True):
    """Cluster `nframes` frames across the ranks of the default process group.

    X_all_frames_fn(first, count) -> [count, n, d] input of those frames (each rank builds only
    its own frames); cluster_fn(X) -> (labels [count, n], k [count], iterations [count]).
    Returns (first, count, local results) and, when gather, the full per-frame k and
    iteration arrays on every rank (labels stay local: they never cross the data path).
    """
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    first, count = frame_shard(nframes, world, rank)
    X = X_all_frames_fn(first, count)
    labels, k, iters = cluster_fn(X)
    out = {"first": first, "count": count, "labels": labels, "k": k, "iterations": iters}
    if gather and world > 1:
        parts: List = [None] * world
        dist.all_gather_object(parts, (first, np.asarray(k).tolist(),
                                       np.asarray(iters).tolist()))
        k_all = np.zeros(nframes, np.int64)
        it_all = np.zeros(nframes, np.int64)
        for f0, ks, its in parts:
            k_all[f0:f0 + len(ks)] = ks
            it_all[f0:f0 + len(its)] = its
        out["k_all"], out["iterations_all"] = k_all, it_all
    elif gather:
        out["k_all"], out["iterations_all"] = np.asarray(k), np.asarray(iters)
    return out


def point_shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced block of points owned by `rank`: (first point, count)."""
    return frame_shard(n, world, rank)


def _allreduce_np(a: np.ndarray, op: str) -> np.ndarray:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return a
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    dist.all_reduce(t, op={"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX,
                           "sum": dist.ReduceOp.SUM}[op])
    return t.cpu().numpy()


def _allgather_rows(a: np.ndarray) -> np.ndarray:
    """Concatenate every rank's rows (variable counts) in rank order."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return a
    world = dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    cnt = torch.tensor([a.shape[0]], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    sizes = [int(c.item()) for c in cnts]
    mx = max(sizes)
    pad = np.zeros((mx,) + a.shape[1:], a.dtype)
    pad[:a.shape[0]] = a
    # int64 views keep every dtype exact across backends (u32 is not a torch dtype everywhere)
    t = torch.from_numpy(pad.astype(np.int64, copy=False)).to(dev)
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return np.concatenate([p.cpu().numpy()[:sz].astype(a.dtype) for p, sz in zip(parts, sizes)])


def run_cloud(engine, X_local: np.ndarray, h: float, max_iter: int, record_history: bool = False):
    """Cluster ONE point cloud whose rows are split over the ranks (this rank holds X_local,
    a contiguous block).  engine: a gridshift.Engine (or any object with the shard_* methods).
    Returns this rank's ClusterLabeling (labels of its own points; centroids, iterations and
    convergence identical on every rank)."""
    from .gridshift import EngineConfig
    if not (hasattr(X_local, "is_cuda") and X_local.is_cuda):
        X_local = np.ascontiguousarray(X_local)
    n_local = X_local.shape[0]
    klo, khi = engine.shard_keybounds(X_local, h)
    klo = _allreduce_np(np.asarray(klo, np.int64), "min")
    khi = _allreduce_np(np.asarray(khi, np.int64), "max")
    n_global = int(_allreduce_np(np.array([n_local], np.int64), "sum")[0])
    keys, counts, sums = engine.shard_bin(X_local, h, n_global, klo, khi)
    keys = _allgather_rows(np.asarray(keys, np.uint32))
    counts = _allgather_rows(np.asarray(counts, np.uint32))
    sums = _allgather_rows(np.asarray(sums, np.int64))
    return engine.shard_run(keys, counts, sums, n_local,
                            EngineConfig(h, max_iter, record_history))
