"""Utterance sharding across GPUs: trials are independent, so the data path
has no collective.  Each rank (one process per GPU) decodes the trials dealt to it; results
travel back host-side.  torch.distributed is plumbing only: a barrier around the timed region
and the max-over-ranks of the device time.
"""

from __future__ import annotations

import numpy as np


def shard_trials(lengths, world: int, rank: int) -> np.ndarray:
    """Length-balanced deal: sort by frame count (longest first, stable), then round-robin.
    Every trial lands on exactly one rank; per-rank frame totals differ by < max(T)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    lengths = np.asarray(lengths)
    order = np.argsort(-lengths, kind="stable")
    return np.sort(order[rank::world])


def gather_results(local_results, local_index, world: int, group=None):
    """Host-side result gather (all_gather_object over the given process group); returns the
    full list in global trial order on every rank."""
    import torch.distributed as dist

    payload = list(zip(local_index.tolist(), local_results))
    parts = [None] * world
    dist.all_gather_object(parts, payload, group=group)
    merged = {}
    for part in parts:
        for i, r in part:
            merged[i] = r
    return [merged[i] for i in sorted(merged)]


def max_over_ranks(value: float, device=None) -> float:
    """Device-time aggregation rule of the benchmark: the slowest rank defines the job time."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
