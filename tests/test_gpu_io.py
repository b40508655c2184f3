"""Formats from/to device buffers: a series' and a
stream's compressed rows written as XCMP stores and read back by the
reference's own io::read_compressed; XFSR frames files (reference-written
u16/f32/f64 and the new u8) loaded straight into a series."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


def _setup(ctx, orc, t, h, w, q, mu, seed):
    frames = orc.gen_speckle(t, h, w, q, mu, seed)
    ring, _ = orc.ring_map(h, w, q)
    return frames, ring, xg.RingLayout.from_ring_map(ctx, ring, q)


def test_series_xcmp_read_by_reference(ctx, orc, ref, tmp_path):
    frames, ring, lay = _setup(ctx, orc, 150, 40, 40, 2, 0.6, 81)
    basis = xg.Basis(lay, 8)
    xg.FrameSeries(lay, 40).load(frames[:40]).build_basis(8, basis=basis)
    s = xg.FrameSeries(lay, 150).load(frames).compress(basis)
    for r in range(2):
        p = tmp_path / f"r{r}.xcmp"
        s.write_xcmp(r, p, 1234 + r)
        k, h, y, nr = ref.read_compressed(p)
        yy, nn = s.coeffs(r)
        assert (k, h) == (8, 1234 + r)
        assert np.array_equal(y, yy) and np.array_equal(nr, nn)


def test_stream_appends_xcmp(ctx, orc, ref, tmp_path):
    frames, ring, lay = _setup(ctx, orc, 60, 32, 32, 2, 0.8, 82)
    basis = xg.Basis(lay, 6)
    xg.FrameSeries(lay, 30).load(frames[:30]).build_basis(6, basis=basis)
    st = xg.FrameStream(lay, 60, basis=basis, sparse=True)
    p = tmp_path / "stream.xcmp"
    for t in range(25):
        st.push(frames[t])
    st.append_xcmp(1, p, 99)              # rows 0..24 (creates the store)
    for t in range(25, 60):
        st.push(frames[t])
    st.append_xcmp(1, p, 99, from_frame=25)
    k, h, y, nr = ref.read_compressed(p)
    yy, nn = st.coeffs(1)
    assert y.shape == (60, 6) and np.array_equal(y, yy) and np.array_equal(nr, nn)
    with pytest.raises(xg.BindingError):
        st.append_xcmp(1, p, 100, from_frame=60)


@pytest.mark.parametrize("dtype", [0, 2, 3])
def test_load_xfsr_equals_direct_load(ctx, orc, ref, tmp_path, dtype):
    frames, ring, lay = _setup(ctx, orc, 90, 36, 36, 3, 0.5, 83)
    p = tmp_path / "f.xfsr"
    if dtype == 3:
        xg.write_xfsr(p, frames, 0.01)
    else:
        ref.write_frames(p, frames.astype(np.float64), 0.01, dtype)
    a = xg.FrameSeries(lay, 90).load_xfsr(p).ttc_raw()
    b = xg.FrameSeries(lay, 90).load(frames).ttc_raw()
    assert a.frame_period == 0.01
    for r in range(3):
        assert np.array_equal(a.ttc(r, "gram"), b.ttc(r, "gram"))
    with pytest.raises(xg.ShapeError):
        xg.FrameSeries(xg.RingLayout(ctx, 100, [np.arange(10)]), 90).load_xfsr(p)


def test_ttc_tile_sink_round_trip(ctx, orc, tmp_path):
    """XTTC tile files stream the stored TTC (upper triangle, 256-row blocks)
    and read back to exactly the readback matrices."""
    frames, ring, lay = _setup(ctx, orc, 300, 40, 40, 2, 0.5, 84)
    basis = xg.Basis(lay, 8)
    xg.FrameSeries(lay, 40).load(frames[:40]).build_basis(8, basis=basis)
    s = xg.FrameSeries(lay, 300).load(frames).ttc_raw()
    s.compress(basis).ttc_compressed()
    for r in range(2):
        s.write_ttc(r, tmp_path / "g.xttc", "gram")
        assert np.array_equal(xg.read_xttc(tmp_path / "g.xttc"), s.ttc(r, "gram"))
        s.write_ttc(r, tmp_path / "c.xttc", "f64")
        assert np.array_equal(xg.read_xttc(tmp_path / "c.xttc"), s.ttc(r, "f64"))
        s.write_ttc(r, tmp_path / "k.xttc", "f32", compressed=True)
        assert np.array_equal(xg.read_xttc(tmp_path / "k.xttc"), s.cttc(r, "f32"))
    assert (tmp_path / "g.xttc").stat().st_size == 20 + 300 * 301 // 2 * 4
    with pytest.raises(xg.ContractError):
        s.write_ttc(0, tmp_path / "x.xttc", "f32")  # raw TTC has no f32 sink


def test_device_basis_saved_as_xenc_for_the_reference(ctx, orc, ref, tmp_path):
    """A basis built on the device, written as XENC, loads in the reference
    (its EncodingMatrix checks orthonormality to 1e-10) and binds stores by
    the same content hash."""
    frames, ring, lay = _setup(ctx, orc, 80, 32, 32, 2, 0.6, 85)
    vs, sig, rank = xg.FrameSeries(lay, 80).load(frames).build_basis(12)
    for r in range(2):
        p = tmp_path / f"r{r}.xenc"
        xg.write_xenc(p, vs[r], sig[r], mode=1)
        v, spec, mode = ref.read_encoder(p)
        assert mode == 1 and np.array_equal(v, vs[r]) and np.array_equal(spec, sig[r])
        assert xg.content_hash(vs[r], 1) == ref.content_hash(vs[r], 1)
