"""K9: the encoding basis built on the device (xg_series_build_basis) against
the reference's own encoder (oracle/_ref build_online_from_frames /
build_offline, encoder.cpp:13-60 -> gram_svd, linalg.cpp:279-439), per ring.

Bar: V within 1e-10 after the shared sign convention and the spectrum within
1e-12 relative (the same bar as the host builder in test_host.py; the device
path is not bit-identical -- parallel Jacobi order, int Gram normalised after
the dot products, Cholesky-QR instead of MGS -- but each step is backward
stable in f64).  Plus: orthonormal columns, typed errors, and the device
basis driving the compressed path like a host-set one."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


def _series(ctx, orc, t, h, w, q, mu, seed):
    frames = orc.gen_speckle(t, h, w, q, mu, seed)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    return frames, ring, lay, xg.FrameSeries(lay, t).load(frames)


@pytest.mark.parametrize("t,h,w,q,mu,k,seed", [
    (64, 48, 48, 3, 0.5, 16, 61),
    (129, 64, 64, 4, 0.4, 32, 62),     # odd T: padded Jacobi order
    (256, 64, 64, 2, 0.3, 64, 63),
    (40, 32, 40, 2, 1.0, 7, 64),
])
def test_device_basis_matches_reference(ctx, orc, ref, t, h, w, q, mu, k, seed):
    frames, ring, lay, s = _series(ctx, orc, t, h, w, q, mu, seed)
    vs, sig, rank = s.build_basis(k)
    for r in range(q):
        xq = frames[:, ring == r].astype(np.float64)
        v_ref, spec_ref = ref.build_online_from_frames(xq, k)
        assert rank[r] == spec_ref.size
        assert vs[r].shape == v_ref.shape
        assert np.abs(vs[r] - v_ref).max() <= 1e-10, f"ring {r}"
        assert np.abs(sig[r] - spec_ref).max() <= 1e-12 * spec_ref[0]
        assert np.abs(vs[r].T @ vs[r] - np.eye(k)).max() <= 1e-12


def test_device_basis_full_rank(ctx, orc, ref):
    """k = 0: build_offline (the full numerical rank of every ring)."""
    frames, ring, lay, s = _series(ctx, orc, 48, 40, 40, 2, 0.8, 65)
    vs, sig, rank = s.build_basis(0)
    for r in range(2):
        xq = frames[:, ring == r].astype(np.float64)
        v_ref = ref.build_offline(xq)
        assert vs[r].shape == v_ref.shape and rank[r] == v_ref.shape[1]
        assert np.abs(vs[r] - v_ref).max() <= 1e-10


def test_device_basis_rank_deficient_and_errors(ctx, orc):
    """Repeated training frames: rank < T, RankError carries the achievable
    rank; a zero training frame raises NormalizationError (frame, ring)."""
    h = w = 32
    ring, _ = orc.ring_map(h, w, 2)
    lay = xg.RingLayout.from_ring_map(ctx, ring, 2)
    base = orc.gen_speckle(6, h, w, 2, 1.0, 66)
    frames = np.vstack([base, base, base])  # 18 frames, rank <= 6
    s = xg.FrameSeries(lay, 18).load(frames)
    _, _, rank = s.build_basis(0)
    assert all(rank <= 6)
    with pytest.raises(xg.RankError) as e:
        s.build_basis(10)
    assert e.value.achievable_rank <= 6
    z = base.copy()
    z[2, ring == 1] = 0
    s2 = xg.FrameSeries(lay, 6).load(z)
    with pytest.raises(xg.NormalizationError) as e:
        s2.build_basis(2)
    assert e.value.frame_index == 2 and e.value.ring == 1


def test_device_basis_drives_compression(ctx, orc):
    """The Basis filled on the device compresses exactly like the same V set
    from the host, bitwise (same digits)."""
    t, h, w, q, k = 200, 48, 48, 3, 16
    frames, ring, lay, s = _series(ctx, orc, t, h, w, q, 0.4, 67)
    train = xg.FrameSeries(lay, 64).load(frames[:64])
    b_dev = xg.Basis(lay, k)
    vs, _, _ = train.build_basis(k, basis=b_dev)
    b_host = xg.Basis(lay, k)
    for r in range(q):
        b_host.set_ring(r, vs[r])
    s.compress(b_dev)
    y_dev = [s.coeffs(r)[0].copy() for r in range(q)]
    s.compress(b_host)
    for r in range(q):
        assert np.array_equal(y_dev[r], s.coeffs(r)[0])


# ---- f64 training rows of any values (xg_build_basis / _batch): row_normalize
# and S in the reference's own f64 order on the device, then the same K9
# pipeline.  Same bar as the count builder.
@pytest.mark.parametrize("n,m,k,seed", [(16, 64, 8, 1), (40, 500, 20, 2), (64, 3000, 32, 3)])
def test_f64_rows_basis_builder_matches_reference(orc, ref, n, m, k, seed):
    x = orc.random_positive_matrix(n, m, seed)
    v = xg.build_online_from_frames(x, k)
    vr, _ = ref.build_online_from_frames(x, k)
    assert np.abs(v - vr).max() <= 1e-10
    assert np.abs(v.T @ v - np.eye(k)).max() <= 1e-10


def test_f64_rows_basis_builder_full_rank_and_errors(orc, ref):
    x = orc.random_positive_matrix(12, 48, 5)
    v = xg.build_online_from_frames(x, 0)
    assert np.abs(v - ref.build_offline(x)).max() <= 1e-10
    with pytest.raises(xg.RankError) as ei:
        xg.build_online_from_frames(np.ones((4, 8)), 2)      # rank-1 corpus
    assert ei.value.achievable_rank == 1
    z = orc.random_positive_matrix(5, 10, 1)
    z[3] = 0.0
    with pytest.raises(xg.NormalizationError) as ei:
        xg.build_online_from_frames(z, 2)
    assert ei.value.frame_index == 3


def test_f64_rows_ring_bases_batch_equals_single(orc):
    xs = [orc.random_positive_matrix(24, m, 10 + m) for m in (50, 77, 120)]
    par = xg.build_ring_bases(xs, 6, threads=3)
    for x, v in zip(xs, par):
        assert np.array_equal(v, xg.build_online_from_frames(x, 6))
