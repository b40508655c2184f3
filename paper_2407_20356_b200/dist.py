"""Multi-GPU host logic: one process per GPU, one detector's pixels sharded
across the processes along q-ring boundaries.

Every hot quantity of the path -- the Gram G_q, the norms |x_t|^2, the
coefficients Y_q -- is a sum over the pixels of a ring (gram,
/root/reference/proj/src/linalg.cpp:127-156; project_row,
/root/reference/proj/src/compress.cpp:12-22).  So:

* rings are dealt to processes whole by longest-processing-time on their
  pixel count (the raw Gram costs T(T+1) M_q; the rank-k projection T M_q k);
  each process holds only the frames' pixels of its rings (its pixel slice)
  and computes those rings with no collective on the data path;
* when whole rings cannot balance the processes within `tol` (a ring larger
  than a process's share, or too few rings), the largest pieces are halved
  until they can: a ring whose pixels end up on several processes is a
  *split ring*.  Each holder computes the exact int32 Gram + |x|^2 of its
  share, the shares are summed on the ring's owner (integer sum: exact and
  order-independent, so 1-, 2-, 4- and 8-process Grams are bitwise
  identical), and the owner finishes the ring (norms, zero frames, g2);
* g2 of every ring is gathered to rank 0 (a few MB).

`torch.distributed` is the plumbing: NCCL over NVLink on B200s (device
buffers straight from the library), gloo for the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import numpy as np


def shard_rings(costs: Sequence[float], world: int) -> List[List[int]]:
    """LPT assignment of whole rings: rings sorted by decreasing cost, each
    to the least loaded rank (ties -> lowest rank).  Deterministic; every
    ring exactly once."""
    order = sorted(range(len(costs)), key=lambda r: (-costs[r], r))
    load = [0.0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for r in order:
        j = min(range(world), key=lambda i: (load[i], i))
        out[j].append(r)
        load[j] += float(costs[r])
    return [sorted(o) for o in out]


def ring_costs(ring_pixels: Sequence[int], n_frames: int) -> List[float]:
    """Raw-Gram work of a ring: T(T+1) M_q (the projection is T M_q k:
    pixel-proportional too, so one assignment balances both)."""
    return [float(n_frames) * (n_frames + 1) * m for m in ring_pixels]


@dataclass
class ShardPlan:
    """Which pixels of which ring each process holds.

    ``pieces[rank]`` lists ``(ring, lo, hi)``: positions [lo, hi) of the
    ring's mask (ascending pixel order) held by ``rank``.  A ring held by
    more than one rank is split; its ``owner`` (the holder with the most
    pixels, ties -> lowest rank) finishes it."""

    world: int
    ring_pixels: List[int]
    pieces: List[List[Tuple[int, int, int]]]
    owner: List[int] = field(default_factory=list)
    holders: List[List[int]] = field(default_factory=list)

    def __post_init__(self):
        q = len(self.ring_pixels)
        held = [[0] * self.world for _ in range(q)]
        for rk, ps in enumerate(self.pieces):
            for r, lo, hi in ps:
                held[r][rk] += hi - lo
        self.owner = [max(range(self.world), key=lambda k: (held[r][k], -k)) for r in range(q)]
        self.holders = []
        for r in range(q):
            hs = [k for k in range(self.world) if held[r][k] > 0 and k != self.owner[r]]
            self.holders.append([self.owner[r]] + hs)

    def split_rings(self) -> List[int]:
        return [r for r in range(len(self.ring_pixels)) if len(self.holders[r]) > 1]

    def rank_rings(self, rank: int) -> List[int]:
        """Rings with pixels on ``rank``, ascending (the rank-local ring order)."""
        return sorted({r for r, _, _ in self.pieces[rank]})

    def owned_rings(self, rank: int) -> List[int]:
        return [r for r in range(len(self.ring_pixels)) if self.owner[r] == rank]

    def share(self, rank: int, ring: int) -> np.ndarray:
        """Positions (into the ring's mask) of the pixels ``rank`` holds."""
        parts = [np.arange(lo, hi, dtype=np.int64) for r, lo, hi in self.pieces[rank] if r == ring]
        return np.concatenate(parts) if parts else np.zeros(0, np.int64)

    def loads(self) -> List[int]:
        return [sum(hi - lo for _, lo, hi in ps) for ps in self.pieces]

    def imbalance(self) -> float:
        """max load / ideal load - 1."""
        ld = self.loads()
        ideal = sum(ld) / self.world
        return max(ld) / ideal - 1.0 if ideal > 0 else 0.0


def _merge(pieces: List[Tuple[int, int, int]]) -> List[Tuple[int, int, int]]:
    out: List[Tuple[int, int, int]] = []
    for r, lo, hi in sorted(pieces):
        if out and out[-1][0] == r and out[-1][2] == lo:
            out[-1] = (r, out[-1][1], hi)
        else:
            out.append((r, lo, hi))
    return out


def plan_shards(ring_pixels: Sequence[int], world: int, tol: float = 0.05,
                min_piece: int = 256, max_rounds: int = 256) -> ShardPlan:
    """Ring-aligned pixel sharding: whole rings by LPT on
    their pixel counts; while the most loaded rank exceeds the ideal share by
    more than ``tol``, halve the largest piece (no piece below ``min_piece``
    pixels) and re-deal.  world = 1 gives every ring whole to rank 0."""
    ring_pixels = [int(m) for m in ring_pixels]
    items = [(r, 0, m) for r, m in enumerate(ring_pixels) if m > 0]
    total = float(sum(ring_pixels))
    ideal = total / max(world, 1)

    def deal(its):
        order = sorted(range(len(its)), key=lambda i: (-(its[i][2] - its[i][1]), its[i]))
        load = [0] * world
        out: List[List[Tuple[int, int, int]]] = [[] for _ in range(world)]
        for i in order:
            j = min(range(world), key=lambda k: (load[k], k))
            out[j].append(its[i])
            load[j] += its[i][2] - its[i][1]
        return out, load

    pieces, load = deal(items)
    for _ in range(max_rounds):
        if world == 1 or max(load) <= (1.0 + tol) * ideal:
            break
        big = max(range(len(items)), key=lambda i: (items[i][2] - items[i][1], -i))
        r, lo, hi = items[big]
        if hi - lo < 2 * min_piece:
            break
        mid = lo + (hi - lo) // 2
        items[big:big + 1] = [(r, lo, mid), (r, mid, hi)]
        pieces, load = deal(items)
    return ShardPlan(world, ring_pixels, [_merge(p) for p in pieces])


def rank_slice(plan: ShardPlan, rank: int, masks: Sequence[np.ndarray]):
    """The detector pixels ``rank`` holds and its local ring masks.

    Returns (pixels, local_masks, rings): ``pixels`` = ascending detector
    indices of the rank's pixel slice (the columns of the frames it
    receives); ``local_masks[i]`` = positions in that slice of the pixels of
    global ring ``rings[i]`` (ascending, so every ring keeps its mask order
    and its Gram share is the reference's sum over those pixels)."""
    rings = plan.rank_rings(rank)
    sel = [np.asarray(masks[r], np.int64)[plan.share(rank, r)] for r in rings]
    pixels = np.sort(np.concatenate(sel)) if sel else np.zeros(0, np.int64)
    local = [np.searchsorted(pixels, s) for s in sel]
    return pixels, local, rings


def _backend(group=None) -> str:
    import torch.distributed as dist

    return dist.get_backend(group)


def reduce_split_rings(series, plan: ShardPlan, rank: int, rings: Sequence[int], group=None,
                       strict: bool = False) -> None:
    """Sum every split ring's shares onto its owner and finish it there.

    ``series`` is this rank's FrameSeries after ttc_raw (stored); ``rings``
    its local ring order (rank_slice).  Split rings are visited in global
    order by every holder, so the point-to-point pairs always match.  With
    NCCL the partials stay on the device (the library exports straight into
    CUDA tensors; int32 / int64 adds); with gloo they go through host memory."""
    import torch
    import torch.distributed as dist

    local = {r: i for i, r in enumerate(rings)}
    nccl = _backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else None
    for r in plan.split_rings():
        hs = plan.holders[r]
        if rank not in hs:
            continue
        li = local[r]
        if nccl:
            g = torch.empty(series.partial_elems, dtype=torch.int32, device=dev)
            n2 = torch.empty(series.n_frames, dtype=torch.int64, device=dev)
            torch.cuda.synchronize()  # the library's stream produced the Gram
            series.export_partial(li, g, n2)
            series.ctx.synchronize()
        else:
            gh, nh = series.export_partial(li)
            g, n2 = torch.from_numpy(gh), torch.from_numpy(nh)
        owner = plan.owner[r]
        if rank == owner:
            tg, tn = torch.empty_like(g), torch.empty_like(n2)
            for src in hs[1:]:
                dist.recv(tg, src=src, group=group)
                dist.recv(tn, src=src, group=group)
                g += tg  # int32: modular, exact whenever the total fits (checked on import)
                n2 += tn
            if nccl:
                torch.cuda.synchronize()
                series.import_partial(li, g, n2, strict=strict)
            else:
                series.import_partial(li, g.numpy(), n2.numpy(), strict=strict)
        else:
            dist.send(g, dst=owner, group=group)
            dist.send(n2, dst=owner, group=group)


def gather_g2(series, plan: ShardPlan, rank: int, rings: Sequence[int], group=None,
              compressed: bool = False):
    """g2 values and pair counts of every ring on rank 0 (others: None).

    Each rank contributes the rings it owns; the transfer is one padded
    all-gather (NCCL: device buffers, no host round trip)."""
    import torch
    import torch.distributed as dist

    world = plan.world
    q = len(plan.ring_pixels)
    t = series.n_frames
    owned = [r for r in plan.owned_rings(rank)]
    local = {r: i for i, r in enumerate(rings)}
    per = max(len(plan.owned_rings(k)) for k in range(world))
    nccl = _backend(group) == "nccl"
    if nccl:
        vals, cnts = series.g2_device(compressed=compressed)
        torch.cuda.synchronize()
        series.ctx.synchronize()
        buf = torch.zeros((per, 2, t), dtype=torch.float64, device=vals.device)
        for i, r in enumerate(owned):
            buf[i, 0] = vals[local[r], :t]
            buf[i, 1] = cnts[local[r], :t].to(torch.float64)
        out = torch.empty((world * per, 2, t), dtype=torch.float64, device=vals.device)
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        _, vals, cnts = (series.cg2_all() if compressed else series.g2_all())
        buf = torch.zeros((per, 2, t), dtype=torch.float64)
        for i, r in enumerate(owned):
            buf[i, 0] = torch.from_numpy(vals[local[r]])
            buf[i, 1] = torch.from_numpy(cnts[local[r]].astype(np.float64))
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        out = torch.cat(parts)
    if rank != 0:
        return None
    host = out.cpu().numpy()
    g2 = np.empty((q, t))
    cnt = np.empty((q, t), np.int64)
    for k in range(world):
        for i, r in enumerate(plan.owned_rings(k)):
            g2[r] = host[k * per + i, 0]
            cnt[r] = host[k * per + i, 1].astype(np.int64)
    return g2, cnt


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
