"""Multi-GPU host logic: one process per GPU, q-rings sharded across ranks.

Every hot quantity of the path (G_q, Y_q, norms, g2) is per ring, and rings
are independent: rings are dealt to ranks by
longest-processing-time on their cost, each rank computes its rings with no
data-path collective, and the per-ring results are gathered to rank 0 (a
few MB of g2).  `torch.distributed` is the plumbing (NCCL on B200s, gloo for
the CPU tests)."""
from __future__ import annotations

from typing import Dict, List, Sequence

import numpy as np


def shard_rings(costs: Sequence[float], world: int) -> List[List[int]]:
    """LPT assignment: rings sorted by decreasing cost, each to the least
    loaded rank (ties -> lowest rank).  Deterministic; every ring exactly once."""
    order = sorted(range(len(costs)), key=lambda r: (-costs[r], r))
    load = [0.0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for r in order:
        j = min(range(world), key=lambda i: (load[i], i))
        out[j].append(r)
        load[j] += float(costs[r])
    return [sorted(o) for o in out]


def ring_costs(ring_pixels: Sequence[int], n_frames: int) -> List[float]:
    """Raw-Gram work of a ring: T(T+1) M_q (the compressed Gram is T(T+1) k,
    identical for every ring, so pixel-proportional cost also balances the
    projection)."""
    return [float(n_frames) * (n_frames + 1) * m for m in ring_pixels]


def gather_rings(local: Dict[int, np.ndarray], n_rings: int, group=None) -> Dict[int, np.ndarray]:
    """Gather per-ring arrays from every rank onto rank 0 (others get {})."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object({int(k): np.asarray(v) for k, v in local.items()}, gathered, dst=0,
                       group=group)
    if rank != 0:
        return {}
    full: Dict[int, np.ndarray] = {}
    for part in gathered:
        for k, v in part.items():
            if k in full:
                raise RuntimeError(f"ring {k} computed by two ranks")
            full[k] = v
    if sorted(full) != list(range(n_rings)):
        raise RuntimeError("gather_rings: missing rings")
    return full


def max_over_ranks(value: float, group=None) -> float:
    """Step time of the job = the slowest rank (timed on each device)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
