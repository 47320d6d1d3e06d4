"""Multi-GPU driver for independent frames (independent runs may execute
concurrently with fully isolated state).

One process per GPU (torchrun); frames are partitioned into contiguous blocks, each rank
clusters its block through its own engine, and nothing crosses the data path: the only
collectives are the timing max-reduction and an optional gather of per-frame results for
reporting.  See DESIGN.md §5 for why the single large cloud (cfg5) uses a different plan.
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
