"""World-size-2 gloo test of the multi-rank path (CPU): rings are sharded
with dist.shard_rings, every rank computes its rings' raw TTC g2 (here with
the oracle, standing in for the device kernels that need a B200), results
are gathered to rank 0 and must equal the single-rank computation bitwise;
the step time reduction is max-over-ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as tdist

    import oracle
    from paper_2407_20356_b200 import dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.c()
    t, h, w, n_rings = 60, 32, 32, 5
    frames = orc.gen_speckle(t, h, w, n_rings, 0.4, 13)
    ring, _ = orc.ring_map(h, w, n_rings)
    sizes = np.bincount(ring, minlength=n_rings)
    mine = dist.shard_rings(dist.ring_costs(sizes, t), world)[rank]
    local = {}
    for r in mine:
        g = orc.ttc_raw(frames[:, ring == r].astype(np.float64))
        local[r] = orc.g2_from_ttc(g)[1]
    full = dist.gather_rings(local, n_rings)
    tmax = dist.max_over_ranks(float(rank + 1))
    if rank == 0:
        ok = tmax == float(world)
        for r in range(n_rings):
            g = orc.ttc_raw(frames[:, ring == r].astype(np.float64))
            ok = ok and np.array_equal(full[r], orc.g2_from_ttc(g)[1])
        q.put(ok)
    tdist.destroy_process_group()


def test_two_rank_ring_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
