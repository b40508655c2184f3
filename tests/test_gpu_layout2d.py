"""2D ingest bands (xg_layout_create_2d): on a detector wider than 512 pixels
the ingest reads 32-row x 512-column blocks instead of 16384-pixel raster
strips.  Only the ring-major column order differs, so every result -- the
exact Gram, norms, g2, the projection coefficients -- must equal the 1D
layout's bitwise and the oracle's (gram, linalg.cpp:127-156; compress_series,
compress.cpp:48-81).  Shapes cover full blocks, partial edge blocks in both
directions, a width that is not a multiple of 16 (falls back to strips), and
scattered masks."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("t,h,w,q,mu,kind", [
    (260, 64, 1024, 8, 0.1, "rings"),      # two full block columns
    (200, 80, 1040, 5, 0.2, "rings"),      # partial rows (80 = 2 x 32 + 16), 16-column edge block
    (150, 40, 600, 4, 0.3, "rings"),       # width % 16 != 0: raster strips
    (180, 70, 1536, 6, 0.2, "scattered"),  # irregular masks, 3 block columns
])
def test_2d_layout_equals_1d(ctx, orc, t, h, w, q, mu, kind):
    frames = orc.gen_speckle(t, h, w, q, mu, 91)
    if kind == "rings":
        ring, _ = orc.ring_map(h, w, q)
    else:
        ring = np.random.default_rng(4).integers(-1, q, size=h * w).astype(np.int32)
    l1 = xg.RingLayout.from_ring_map(ctx, ring, q)
    l2 = xg.RingLayout.from_ring_map(ctx, ring.reshape(h, w), q)
    assert l2.shape == (h, w)
    s1 = xg.FrameSeries(l1, t).load(frames).ttc_raw()
    s2 = xg.FrameSeries(l2, t).load(frames).ttc_raw()
    k = 6
    b1, b2 = xg.Basis(l1, k), xg.Basis(l2, k)
    rng = np.random.default_rng(2)
    for r in range(q):
        xq = frames[:, ring == r]
        g2d = s2.ttc(r, "gram")
        assert np.array_equal(g2d, s1.ttc(r, "gram"))
        assert np.array_equal(g2d.astype(np.int64), orc.gram_u8(xq))
        assert np.array_equal(s2.norms(r)[0], s1.norms(r)[0])
        _, v1, c1 = s1.g2(r)
        _, v2, c2 = s2.g2(r)
        assert np.array_equal(c1, c2) and np.abs(v1 - v2).max() <= 1e-13
        v, _ = np.linalg.qr(rng.standard_normal((xq.shape[1], k)))
        b1.set_ring(r, v)
        b2.set_ring(r, v)
    s1.compress(b1)
    s2.compress(b2)
    for r in range(q):
        assert np.array_equal(s1.coeffs(r)[0], s2.coeffs(r)[0])


def test_2d_layout_chunked_host_and_stream(ctx, orc):
    """Chunked compress, the host-overlapped raw path and the streaming
    ingest on a 2D layout."""
    t, h, w, q = 96, 64, 1024, 5
    frames = orc.gen_speckle(t, h, w, q, 0.3, 92)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring.reshape(h, w), q)
    basis = xg.Basis(lay, 4)
    xg.FrameSeries(lay, 48).load(frames[:48]).build_basis(4, basis=basis)
    one = xg.FrameSeries(lay, t).load(frames).compress(basis)
    ch = xg.FrameSeries(lay, t, x_frames=32)
    for i in range(0, t, 32):
        ch.compress_chunk(basis, frames[i:i + 32], first=(i == 0))
    host = xg.FrameSeries(lay, t).ttc_raw_host(frames)
    st = xg.FrameStream(lay, t, basis=basis, store_ttc=True)
    for i in range(t):
        st.push(frames[i])
    for r in range(q):
        g_ref = orc.gram_u8(frames[:, ring == r])
        assert np.array_equal(one.coeffs(r)[0], ch.coeffs(r)[0])
        assert np.array_equal(one.coeffs(r)[0], st.coeffs(r)[0])
        assert np.array_equal(host.ttc(r, "gram").astype(np.int64), g_ref)
        assert np.array_equal(st.ttc(r, dtype="gram").astype(np.int64), g_ref)


def test_ring_blocked_frames_on_a_large_detector(ctx, orc, ref):
    """> 400 kB ring-major rows: the frames (and basis digits) are stored
    ring-blocked with per-ring TMA maps.  Exact Gram bitwise, projection
    against the reference's compress_series, the chunked path, and the device
    basis (whose W = Xn^T U GEMM reads the ring blocks) against the
    reference's build_online_from_frames."""
    import torch

    t, h, w, q, k = 300, 640, 704, 6, 8
    frames = orc.gen_speckle(t, h, w, q, 0.05, 94)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring.reshape(h, w), q)
    s = xg.FrameSeries(lay, t).load(torch.from_numpy(frames).cuda()).ttc_raw()
    basis = xg.Basis(lay, k)
    vs, _, _ = xg.FrameSeries(lay, 64).load(frames[:64]).build_basis(k, basis=basis)
    s.compress(basis)
    ch = xg.FrameSeries(lay, t, x_frames=128)
    for i in range(0, t, 128):
        ch.compress_chunk(basis, frames[i:i + 128], first=(i == 0))
    for r in range(q):
        xq = frames[:, ring == r]
        assert np.array_equal(s.ttc(r, "gram").astype(np.int64), orc.gram_u8(xq)), r
        v_ref, _ = ref.build_online_from_frames(xq[:64].astype(np.float64), k)
        assert np.abs(vs[r] - v_ref).max() <= 1e-10, r
        y_ref, _ = ref.compress_series(xq.astype(np.float64), vs[r])
        y, _ = s.coeffs(r)
        assert np.abs(y - y_ref).max() <= 1e-6 * np.abs(y_ref).max(), r
        assert np.array_equal(ch.coeffs(r)[0], y)
