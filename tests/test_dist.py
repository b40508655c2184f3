"""Multi-rank host logic on CPU (gloo, world size 2): the ring-aligned pixel
sharding plan, the split-ring exchange (shares of a ring's exact Gram summed
on its owner) and the g2 gather.  The per-rank compute here is the oracle's
exact integer Gram of each rank's pixel share, standing in for the device
kernels (tests/test_gpu_dist.py runs the same plumbing over the library on a
B200); the sums must reproduce the single-rank Gram bitwise, as the
reference's gram is a sum over pixel stripes (linalg.cpp:127-156)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2407_20356_b200 import dist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("shape,q", [((512, 512), 32), ((1024, 1024), 100), ((1536, 2048), 128),
                                     ((128, 128), 8)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_shards_cover_and_balance(orc, shape, q, world):
    ring, _ = orc.ring_map(shape[0], shape[1], q)
    sizes = np.bincount(ring, minlength=q)
    plan = dist.plan_shards(sizes, world)
    # every pixel of every ring held by exactly one rank
    for r in range(q):
        got = np.sort(np.concatenate([plan.share(k, r) for k in range(world)]))
        assert np.array_equal(got, np.arange(sizes[r])), r
        assert plan.owner[r] in plan.holders[r]
    assert plan.imbalance() <= 0.05 + 1e-12
    if world == 1:
        assert plan.split_rings() == []
    masks = [np.nonzero(ring == r)[0] for r in range(q)]
    seen = np.zeros(ring.size, np.int64)
    for k in range(world):
        pix, local, rings = dist.rank_slice(plan, k, masks)
        assert np.all(np.diff(pix) > 0)
        seen[pix] += 1
        for lm, r in zip(local, rings):
            assert np.all(np.diff(lm) > 0)
            assert np.array_equal(pix[lm], masks[r][plan.share(k, r)])
    assert np.all(seen == 1)


def test_plan_splits_an_oversized_ring():
    plan = dist.plan_shards([10000, 1000, 1000], 2)
    assert plan.split_rings() == [0]
    assert plan.imbalance() <= 0.05


def _pack_tiles(g):
    """numpy statement of the packed exchange format (xpcs_b200.h)."""
    n = g.shape[0]
    nb = (n + 255) // 256
    gp = np.zeros((nb * 256, nb * 256), np.int32)
    gp[:n, :n] = g
    return np.concatenate([gp[i * 256:(i + 1) * 256, j * 256:(j + 1) * 256].ravel()
                           for i in range(nb) for j in range(i, nb)])


class _OracleSeries:
    """CPU stand-in of a FrameSeries' split-ring interface (oracle compute)."""

    def __init__(self, orc, x_rings):
        self.orc = orc
        self.x = x_rings  # per local ring: n x m_share u8
        self.n_frames = x_rings[0].shape[0]
        self.gram = [orc.gram_u8(x).astype(np.int32) for x in x_rings]
        self.norm2 = [(x.astype(np.int64) ** 2).sum(1) for x in x_rings]

    @property
    def partial_elems(self):
        nb = (self.n_frames + 255) // 256
        return nb * (nb + 1) // 2 * 65536

    def export_partial(self, li):
        return _pack_tiles(self.gram[li]), self.norm2[li].copy()

    def import_partial(self, li, g, n2, strict=False):
        assert g.dtype == np.int32 and g.size == self.partial_elems
        self.packed_total = getattr(self, "packed_total", {})
        self.packed_total[li] = g.copy()
        self.norm2[li] = n2.copy()

    def g2_all(self):
        out, cnt = [], []
        for li, x in enumerate(self.x):
            nr = np.sqrt(self.norm2[li].astype(np.float64))
            g = self.orc.gram_u8(x).astype(np.float64)
            c = g / np.outer(nr, nr)
            _, v, k = self.orc.g2_from_ttc(c)
            out.append(v)
            cnt.append(k)
        return None, np.array(out), np.array(cnt)


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as tdist

    import oracle
    from paper_2407_20356_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.c()
    t, h, w, n_rings = 300, 40, 40, 3
    frames = orc.gen_speckle(t, h, w, n_rings, 0.4, 13)
    ring, _ = orc.ring_map(h, w, n_rings)
    masks = [np.nonzero(ring == r)[0] for r in range(n_rings)]
    sizes = [m.size for m in masks]
    plan = D.plan_shards(sizes, world, tol=0.0, min_piece=64)  # force split rings
    pix, local, rings = D.rank_slice(plan, rank, masks)
    xs = [np.ascontiguousarray(frames[:, pix[lm]]) for lm in local]
    s = _OracleSeries(orc, xs)
    D.reduce_split_rings(s, plan, rank, rings)
    ok = len(plan.split_rings()) > 0
    for r in plan.split_rings():
        if plan.owner[r] == rank:
            li = rings.index(r)
            full = orc.gram_u8(frames[:, masks[r]]).astype(np.int32)
            ok = ok and np.array_equal(s.packed_total[li], _pack_tiles(full))
            ok = ok and np.array_equal(s.norm2[li], (frames[:, masks[r]].astype(np.int64) ** 2).sum(1))
    tmax = D.max_over_ranks(float(rank + 1))
    ok = ok and tmax == float(world)
    res = D.gather_g2(s, plan, rank, rings)
    if rank == 0:
        g2, cnt = res
        for r in range(n_rings):
            if r in plan.split_rings():
                continue  # the stand-in's g2 of a split ring is its share's
            c = orc.ttc_raw(frames[:, masks[r]].astype(np.float64))
            _, v, k = orc.g2_from_ttc(c)
            ok = ok and np.abs(g2[r] - v).max() <= 1e-12 and np.array_equal(cnt[r], k)
        q.put(bool(ok))
    tdist.destroy_process_group()


def test_two_rank_split_ring_exchange_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
