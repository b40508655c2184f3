"""The multi-GPU path through the library (two processes on cuda:0, gloo for
the plumbing -- this box has one GPU and NCCL refuses two ranks on one
device; the kernels of the two processes never wait on each other).

Each process receives only its pixel slice of the detector (dist.rank_slice),
runs ingest + the exact Gram on it, split rings' shares are exported, summed
on their owner and imported (xg_series_export_partial / import_partial), and
g2 is gathered to rank 0.  Every ring's int32 Gram must be bitwise the
single-process Gram (the reference's gram is a sum over pixels,
linalg.cpp:127-156), and g2 within 1e-13 of it."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

T, H, W, Q, MU, SEED = 600, 96, 96, 5, 0.15, 41


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tol, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as tdist

    import oracle
    import paper_2407_20356_b200 as xg
    from paper_2407_20356_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.c()
    frames = orc.gen_speckle(T, H, W, Q, MU, SEED)
    ring, _ = orc.ring_map(H, W, Q)
    masks = [np.nonzero(ring == r)[0] for r in range(Q)]
    plan = D.plan_shards([m.size for m in masks], world, tol=tol, min_piece=128)
    pix, local, rings = D.rank_slice(plan, rank, masks)
    ctx = xg.Context(0)
    lay = xg.RingLayout(ctx, pix.size, local)
    s = xg.FrameSeries(lay, T).load(np.ascontiguousarray(frames[:, pix])).ttc_raw()
    D.reduce_split_rings(s, plan, rank, rings)
    res = D.gather_g2(s, plan, rank, rings)
    grams = {r: s.ttc(rings.index(r), "gram") for r in plan.owned_rings(rank)}
    norms = {r: s.norms(rings.index(r))[0] for r in plan.owned_rings(rank)}
    allg = D.gather_rings(grams, Q) if world > 1 else grams
    alln = D.gather_rings(norms, Q) if world > 1 else norms
    if rank == 0:
        out_q.put((plan.split_rings(), allg, alln, res[0], res[1]))
    tdist.destroy_process_group()


def _run(world, tol):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tol, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    return res


def test_two_process_sharded_equals_single(orc):
    _, g1, n1, g2_1, c1 = _run(1, 0.05)
    split, g2r, n2r, g2_2, c2 = _run(2, 0.0)  # tol 0 forces split rings
    assert split, "the plan must exercise the split-ring exchange"
    frames = orc.gen_speckle(T, H, W, Q, MU, SEED)
    ring, _ = orc.ring_map(H, W, Q)
    for r in range(Q):
        assert np.array_equal(g2r[r], g1[r]), f"ring {r}: int Gram differs from 1 process"
        assert np.array_equal(g1[r].astype(np.int64), orc.gram_u8(frames[:, ring == r]))
        assert np.array_equal(n2r[r], n1[r])
        assert np.array_equal(c2[r], c1[r])
        assert np.abs(g2_2[r] - g2_1[r]).max() <= 1e-13, r
        c_ref = orc.ttc_raw(frames[:, ring == r].astype(np.float64))
        assert np.abs(g2_2[r] - orc.g2_from_ttc(c_ref)[1]).max() <= 1e-12, r


def _nccl_worker(port, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as tdist

    import oracle
    import paper_2407_20356_b200 as xg
    from paper_2407_20356_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    orc = oracle.c()
    frames = orc.gen_speckle(T, H, W, Q, MU, SEED)
    ring, _ = orc.ring_map(H, W, Q)
    masks = [np.nonzero(ring == r)[0] for r in range(Q)]
    plan = D.plan_shards([m.size for m in masks], 1)
    pix, local, rings = D.rank_slice(plan, 0, masks)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = xg.Context(0, stream=st.cuda_stream)
    s = xg.FrameSeries(xg.RingLayout(ctx, pix.size, local), T)
    s.load(torch.from_numpy(np.ascontiguousarray(frames[:, pix])).cuda()).ttc_raw()
    g2, cnt = D.gather_g2(s, plan, 0, rings)  # NCCL path: device buffers of the library
    _, v, c = s.g2_all()
    out_q.put(bool(np.array_equal(g2, v) and np.array_equal(cnt, c)))
    tdist.destroy_process_group()


def test_nccl_gather_of_device_g2_buffers():
    """The NCCL branch of dist.gather_g2 (every step of the multi-GPU bench):
    the library's device g2 buffers wrapped as CUDA tensors
    (__cuda_array_interface__) and all-gathered; one rank, so it runs here."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0 and res is True


def test_partial_export_import_device_buffers(ctx, orc):
    """export_partial / import_partial with CUDA buffers (the NCCL split-ring
    path): exporting a ring's share and importing twice its Gram and norm^2
    (the sum over an identical twin share) must give the Gram doubled
    (exactly) and unchanged C and g2; importing
    the original restores every bit."""
    import torch

    import paper_2407_20356_b200 as xg

    frames = orc.gen_speckle(T, H, W, Q, MU, SEED)
    ring, _ = orc.ring_map(H, W, Q)
    s = xg.FrameSeries(xg.RingLayout.from_ring_map(ctx, ring, Q), T).load(frames).ttc_raw()
    r = 2
    g0, c0 = s.ttc(r, "gram"), s.ttc(r, "f64")
    _, v0, k0 = s.g2(r)
    gd = torch.empty(s.partial_elems, dtype=torch.int32, device="cuda")
    nd = torch.empty(T, dtype=torch.int64, device="cuda")
    s.export_partial(r, gd, nd)
    ctx.synchronize()
    s.import_partial(r, gd * 2, nd * 2)  # the sum of two identical shares
    assert np.array_equal(s.ttc(r, "gram"), 2 * g0)
    assert np.abs(s.ttc(r, "f64") - c0).max() <= 1e-15
    _, v1, k1 = s.g2(r)
    assert np.array_equal(k1, k0) and np.abs(v1 - v0).max() <= 1e-13
    s.import_partial(r, gd, nd)
    assert np.array_equal(s.ttc(r, "gram"), g0)
    gh, nh = s.export_partial(r)  # host buffers
    assert np.array_equal(gh, gd.cpu().numpy()) and np.array_equal(nh, nd.cpu().numpy())
