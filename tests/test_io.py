"""On-disk formats on the host side: the XCMP writer /
appender and the XFSR reader against the reference's own io.cpp (oracle/_ref:
read_compressed, write_frames, read_frames) -- no GPU needed."""
import numpy as np
import pytest

import oracle
import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _rows(n, k, seed):
    rng = np.random.default_rng(seed)
    y = rng.standard_normal((n, k))
    y /= np.linalg.norm(y, axis=1, keepdims=True) * 1.5  # |row| <= 1
    return y, rng.uniform(1.0, 50.0, n)


def test_xcmp_write_read_by_reference(tmp_path, ref):
    y, nr = _rows(37, 9, 1)
    p = tmp_path / "a.xcmp"
    xg.write_xcmp(p, y, nr, 0xDEADBEEFCAFE)
    k, h, y2, n2 = ref.read_compressed(p)
    assert (k, h) == (9, 0xDEADBEEFCAFE)
    assert np.array_equal(y2, y) and np.array_equal(n2, nr)
    assert p.stat().st_size == 32 + 37 * 8 * 10


def test_xcmp_appender_semantics(tmp_path, ref):
    y1, n1 = _rows(5, 4, 2)
    y2, n2 = _rows(7, 4, 3)
    p = tmp_path / "s.xcmp"
    xg.write_xcmp(p, y1, n1, 7, append=True)   # creates
    xg.write_xcmp(p, y2, n2, 7, append=True)   # extends, rewrites N
    k, h, y, nr = ref.read_compressed(p)
    assert np.array_equal(y, np.vstack([y1, y2])) and np.array_equal(nr, np.r_[n1, n2])
    with pytest.raises(xg.ShapeError):
        xg.write_xcmp(p, np.zeros((1, 5)) + 0.1, [1.0], 7, append=True)
    with pytest.raises(xg.BindingError):
        xg.write_xcmp(p, y1, n1, 8, append=True)
    raw = p.read_bytes()
    (tmp_path / "t.xcmp").write_bytes(raw[:-3])  # truncated store
    with pytest.raises(xg.FormatError) as e:
        xg.write_xcmp(tmp_path / "t.xcmp", y1, n1, 7, append=True)
    assert e.value.offset == len(raw) - 3
    with pytest.raises(xg.NormalizationError) as e:
        xg.write_xcmp(tmp_path / "z.xcmp", y1, np.r_[n1[:2], 0.0, n1[3:]], 7)
    assert e.value.frame_index == 2


def test_xcmp_writer_enforces_append_contract(tmp_path, ref):
    """Rows the reference reader's append() would reject (model.cpp:184-193:
    non-finite, or above unit norm) are refused at write time."""
    y, nr = _rows(4, 3, 5)
    bad = y.copy()
    bad[2] *= 1.0 / np.linalg.norm(bad[2]) * 1.001
    with pytest.raises(xg.ContractError):
        xg.write_xcmp(tmp_path / "n.xcmp", bad, nr, 1)
    bad = y.copy()
    bad[1, 0] = np.nan
    with pytest.raises(xg.ContractError):
        xg.write_xcmp(tmp_path / "f.xcmp", bad, nr, 1)
    edge = y.copy()
    edge[0] /= np.linalg.norm(edge[0])  # exactly unit norm is accepted
    xg.write_xcmp(tmp_path / "u.xcmp", edge, nr, 1)
    assert np.array_equal(ref.read_compressed(tmp_path / "u.xcmp")[2], edge)


@pytest.mark.parametrize("dtype", [0, 1, 2])
def test_xfsr_reference_files_read_as_counts(tmp_path, ref, dtype):
    rng = np.random.default_rng(dtype)
    x = rng.integers(0, 256, size=(6, 50)).astype(np.float64)
    p = tmp_path / f"f{dtype}.xfsr"
    ref.write_frames(p, x, 0.25, dtype)
    fr, per = xg.read_xfsr(p)
    assert per == 0.25 and fr.dtype == np.uint8 and np.array_equal(fr, x.astype(np.uint8))


def test_xfsr_u8_round_trip_and_checks(tmp_path, ref):
    rng = np.random.default_rng(9)
    x = rng.integers(0, 256, size=(4, 33), dtype=np.uint8)
    p = tmp_path / "u8.xfsr"
    xg.write_xfsr(p, x, 0.5)
    fr, per = xg.read_xfsr(p)
    assert per == 0.5 and np.array_equal(fr, x)
    assert p.stat().st_size == 36 + x.size
    rc, off = ref.read_frames_status(p)  # dtype 3 is new: the reference refuses it at the dtype
    assert rc == 7 and off == 8
    raw = p.read_bytes()
    (tmp_path / "cut.xfsr").write_bytes(raw[:-1])
    with pytest.raises(xg.FormatError) as e:
        xg.read_xfsr(tmp_path / "cut.xfsr")
    assert e.value.offset == len(raw) - 1
    (tmp_path / "magic.xfsr").write_bytes(b"XFSQ" + raw[4:])
    with pytest.raises(xg.FormatError) as e:
        xg.read_xfsr(tmp_path / "magic.xfsr")
    assert e.value.offset == 0
    f = tmp_path / "frac.xfsr"
    ref.write_frames(f, np.full((2, 3), 1.5), 1.0, 2)
    with pytest.raises(xg.ContractError):
        xg.read_xfsr(f)


def test_xenc_round_trips_with_reference(tmp_path, ref, orc):
    """XENC (io.cpp:273-321): our writer is read by the reference (which
    checks orthonormality and spectrum order on load), the reference's
    writer is read by ours, bitwise; layout errors are FormatError with the
    byte offset."""
    x = orc.random_positive_matrix(20, 300, 4)
    v, spec = ref.build_online_from_frames(x, 6)
    p = tmp_path / "a.xenc"
    xg.write_xenc(p, v, spec, mode=1)
    v2, s2, md = ref.read_encoder(p)
    assert md == 1 and np.array_equal(v2, v) and np.array_equal(s2, spec)
    assert p.stat().st_size == 33 + 8 * spec.size + 8 * v.size
    q = tmp_path / "b.xenc"
    ref.write_encoder(q, v, spec, 0)
    v3, s3, md3 = xg.read_xenc(q)
    assert md3 == 0 and np.array_equal(v3, v) and np.array_equal(s3, spec)
    assert q.read_bytes() == p.read_bytes()[:8] + bytes([0]) + p.read_bytes()[9:]
    raw = p.read_bytes()
    (tmp_path / "cut.xenc").write_bytes(raw[:-8])
    with pytest.raises(xg.FormatError) as e:
        xg.read_xenc(tmp_path / "cut.xenc")
    assert e.value.offset == len(raw) - 8
