"""Streaming (kHz) mode on the GPU: frames pushed one by one (K1 for one
frame, K5 raw column, K6 sparse projection + compressed column).

Invariants, after the reference's streaming tests (test_correlate.cpp:138-157,
test_compress.cpp:101-113, acceptance criterion 9):
  * the streamed exact Gram equals the oracle's gram(counts) bitwise;
  * streamed coefficients equal the batch GPU coefficients bitwise;
  * streamed C~ (f64 dots of the coefficient history) matches the oracle's
    ttc_compressed on the same V within the F32 tolerance, and the batch GPU
    C~ within 1e-5;
  * g2 accumulated per lag matches g2_from_ttc (raw: 1e-12)."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [16, 5, 37])
def test_stream_raw_and_compressed(ctx, orc, k):
    t, h, w, q = 150, 48, 48, 3
    frames = orc.gen_speckle(t, h, w, q, 0.4, 77)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    basis = xg.Basis(lay, k)
    vs = []
    for r in range(q):
        xq = frames[:, ring == r].astype(np.float64)
        v = xg.build_online_from_frames(xq[:64], k)
        vs.append(v)
        basis.set_ring(r, v)
    st = xg.FrameStream(lay, t, basis=basis, store_ttc=True)
    for i in range(t):
        st.push(frames[i])
    assert st.n_frames == t
    batch = xg.FrameSeries(lay, t).load(frames).compress(basis).ttc_compressed()
    for r in range(q):
        xq = frames[:, ring == r]
        assert np.array_equal(st.ttc(r, dtype="gram").astype(np.int64), orc.gram_u8(xq))
        c_ref = orc.ttc_raw(xq.astype(np.float64))
        assert np.abs(st.ttc(r) - c_ref).max() <= 1e-12
        _, g2, cnt = st.g2(r)
        _, g2_ref, cnt_ref = orc.g2_from_ttc(c_ref)
        assert np.array_equal(cnt, cnt_ref)
        assert np.abs(g2 - g2_ref).max() <= 1e-12
        y_s, n_s = st.coeffs(r)
        y_b, n_b = batch.coeffs(r)
        assert np.array_equal(y_s, y_b), "streamed coefficients must equal batch bitwise"
        assert np.array_equal(n_s, n_b)
        y_ref, _ = orc.compress_series(xq.astype(np.float64), vs[r])
        cc_ref, _ = orc.ttc_compressed(y_ref)
        cc = st.ttc(r, compressed=True)
        assert np.abs(cc - cc_ref).max() <= 1e-5 * np.abs(cc_ref).max()
        assert np.abs(cc - batch.cttc(r)).max() <= 1e-5 * np.abs(cc_ref).max()
        _, cg2, _ = st.g2(r, compressed=True)
        assert np.abs(cg2 - orc.g2_from_ttc(cc_ref)[1]).max() <= 1e-5


def test_stream_capacity_and_zero_frame(ctx, orc):
    t, h, w, q = 20, 16, 16, 2
    frames = orc.gen_speckle(t, h, w, q, 0.5, 5)
    ring, _ = orc.ring_map(h, w, q)
    frames[4, ring == 1] = 0
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    st = xg.FrameStream(lay, t)
    for i in range(t):
        st.push(frames[i])
    with pytest.raises(xg.ShapeError):
        st.push(frames[0])
    _, g2, cnt = st.g2(1)
    assert cnt[0] == t - 1 and cnt[1] == t - 3


@pytest.mark.parametrize("mu", [0.05, 0.8])
def test_sparse_stream_equals_dense(ctx, orc, mu):
    """Sparse raw streaming (pixel-major history, nonzeros only) gives the
    dense stream's exact Gram columns and g2 bitwise, at low and high
    occupancy (incl. an all-zero frame)."""
    t, h, w, q = 90, 40, 44, 3
    frames = orc.gen_speckle(t, h, w, q, mu, 81)
    frames[17] = 0
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    dense = xg.FrameStream(lay, t, store_ttc=True)
    sparse = xg.FrameStream(lay, t, store_ttc=True, sparse=True)
    for i in range(t):
        dense.push(frames[i])
        sparse.push(frames[i])
    for r in range(q):
        gd, gs = dense.ttc(r, dtype="gram"), sparse.ttc(r, dtype="gram")
        assert np.array_equal(gs, gd)
        assert np.array_equal(gs.astype(np.int64), orc.gram_u8(frames[:, ring == r]))
        _, g2d, cd = dense.g2(r)
        _, g2s, cs = sparse.g2(r)
        assert np.array_equal(g2s, g2d) and np.array_equal(cs, cd)


@pytest.mark.parametrize("basis_k,raw,evf", [(0, True, None), (6, True, None), (6, False, None),
                                              (37, True, None), (130, True, None), (0, True, "128"),
                                              (6, True, "128")])
def test_push_many_equals_single_pushes(ctx, orc, monkeypatch, basis_k, raw, evf):
    """push_many (one library call for n frames) == n push() calls:
    photon-event push_many ingests 16 frames per launch (batch slots for the
    nonzero lists, a zero frame inside a batch, a partial last batch) and
    forms the batch's columns together (K5s over all its frames, K6 on
    tensor cores reading each coefficient row once for the batch, lag sums
    folded in frame order); single pushes chain push t + 1's ingest beside
    push t's column kernel (K6b, SIMT).  The Gram, the raw lag sums and the
    coefficients must not change a bit; the compressed columns (3xTF32
    tensor cores vs SIMT fp32) agree to fp32 rounding (2e-6 of max |C~|, the
    contract is 1e-5) and their lag counts exactly.  Raw or compressed-only;
    k = 130 takes the two-chunk (k > 128) compressed kernels.  evf = 128: the batches walk
    sealed 128-frame event blocks (single pushes keep the dense history)."""
    import torch

    if evf:
        monkeypatch.setenv("XG_STREAM_EVENT_FRAMES", evf)

    t, h, w, q = 300, 96, 96, 4
    frames = orc.gen_speckle(t, h, w, q, 0.08, 93)
    frames[40] = 0
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    basis = None
    if basis_k:
        basis = xg.Basis(lay, basis_k)
        xg.FrameSeries(lay, 200).load(frames[64:264]).build_basis(basis_k, basis=basis)
    dev = torch.from_numpy(frames).cuda()
    a = xg.FrameStream(lay, t, basis=basis, store_ttc=True, sparse=True, raw=raw)
    b = xg.FrameStream(lay, t, basis=basis, store_ttc=True, sparse=True, raw=raw)
    for i in range(t):
        a.push(dev[i])
    b.push_many(dev[:100])
    b.push(dev[100])  # single pushes between batches
    b.push_many(dev[101:])
    for r in range(q):
        if raw:
            ga, gb = a.ttc(r, dtype="gram"), b.ttc(r, dtype="gram")
            assert np.array_equal(ga, gb)
            assert np.array_equal(gb.astype(np.int64), orc.gram_u8(frames[:, ring == r]))
            _, va, ca = a.g2(r)
            _, vb, cb = b.g2(r)
            assert np.array_equal(va, vb) and np.array_equal(ca, cb)
        if basis_k:
            assert np.array_equal(a.coeffs(r)[0], b.coeffs(r)[0])
            ta = a.ttc(r, compressed=True, dtype="f32").astype(np.float64)
            tb = b.ttc(r, compressed=True, dtype="f32").astype(np.float64)
            assert np.abs(ta - tb).max() <= 2e-6 * np.abs(ta).max()
            _, va, ca = a.g2(r, compressed=True)
            _, vb, cb = b.g2(r, compressed=True)
            assert np.abs(va - vb).max() <= 2e-6 * np.abs(va).max() and np.array_equal(ca, cb)


@pytest.mark.parametrize("mus", [(0.08,), (0.5,), (0.6, 0.03)])
def test_event_history_equals_dense(ctx, orc, monkeypatch, mus):
    """Sealed photon-event blocks (XG_STREAM_EVENT_FRAMES frames each, the
    per-pixel event lists the batched raw columns read instead of the dense
    history; every 8 blocks merged into one level-1 segment) give the dense
    columns' results bitwise: Gram == oracle gram, g2 == single pushes.
    T = 1300 at 128-frame blocks: one merged segment (frames 0-1023) plus
    level-0 blocks 8-9 plus the dense tail.  mu = 0.5 overflows the
    1/8-occupancy event pool, so its blocks (and the segment) stay dense
    (the fallback read of the dense history); the mixed run has bright dense
    blocks first, then sparse ones."""
    import torch

    monkeypatch.setenv("XG_STREAM_EVENT_FRAMES", "128")
    t, h, w, q = 1300, 96, 96, 4
    parts = np.array_split(np.arange(t), len(mus))
    frames = np.concatenate([orc.gen_speckle(len(ix), h, w, q, mu, 31 + i)
                             for i, (ix, mu) in enumerate(zip(parts, mus))])
    frames[200] = 0
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    dev = torch.from_numpy(frames).cuda()
    a = xg.FrameStream(lay, t, store_ttc=True, sparse=True)  # single pushes: dense history
    b = xg.FrameStream(lay, t, store_ttc=True, sparse=True)
    for i in range(t):
        a.push(dev[i])
    b.push_many(dev[:333])  # seals block 0 at the batch starting at frame 128, block 1 at 256
    b.push(dev[333])
    b.push_many(dev[334:])
    for r in range(q):
        ga, gb = a.ttc(r, dtype="gram"), b.ttc(r, dtype="gram")
        assert np.array_equal(ga, gb), r
        assert np.array_equal(gb.astype(np.int64), orc.gram_u8(frames[:, ring == r])), r
        _, va, ca = a.g2(r)
        _, vb, cb = b.g2(r)
        assert np.array_equal(va, vb) and np.array_equal(ca, cb), r
