"""Compressed-path parity on the GPU (K3 tcgen05 int8-digit projection, K4
tcgen05 bf16x3 compressed Gram, fused g2) against the CPU oracle with the
SAME basis V (the reference's own build_online_from_frames when oracle/_ref
is built, else an orthonormal basis from the oracle fixture).

Tolerances (BASELINE north_star): F32-accurate mode within 1e-5 relative
(max|dC| / max|C_ref|); BF16 mode within 1e-2.  Coefficients are checked at
1e-6 of max|Y| (3 int8 digits represent V to ~3e-8 of max|V_j|)."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


def _basis(orc, xq, k, seed):
    """Orthonormal M_q x k basis from a training prefix (QR of the
    row-normalised frames' transpose; parity needs only a fixed V)."""
    try:
        import oracle

        if oracle.ref_available():
            v, _ = oracle.ref().build_online_from_frames(xq[: max(2 * k, 64)].astype(np.float64), k)
            return v
    except Exception:
        pass
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((xq.shape[1], k)))
    return q


@pytest.mark.parametrize("t,h,w,q,mu,k,seed", [
    (300, 64, 64, 4, 0.3, 16, 41),
    (200, 48, 48, 3, 0.5, 32, 42),
    (260, 64, 64, 2, 0.4, 64, 43),
    (150, 40, 40, 2, 0.4, 10, 44),    # rank not a multiple of 16
    (130, 48, 48, 2, 0.5, 5, 45),     # odd rank
    (300, 64, 64, 1, 0.4, 100, 46),   # two N-tiles of coefficients
])
def test_compress_and_ttc_compressed(ctx, orc, t, h, w, q, mu, k, seed):
    frames = orc.gen_speckle(t, h, w, q, mu, seed)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames)
    basis = xg.Basis(lay, k)
    vs = []
    for r in range(q):
        xq = frames[:, ring == r]
        v = _basis(orc, xq, k, seed + r)
        vs.append(v)
        basis.set_ring(r, v)
    s.compress(basis).ttc_compressed()
    for r in range(q):
        xq = frames[:, ring == r].astype(np.float64)
        y_ref, n_ref = orc.compress_series(xq, vs[r])
        y, nrm = s.coeffs(r)
        assert np.array_equal(nrm, n_ref)
        assert np.abs(y - y_ref).max() <= 1e-6 * np.abs(y_ref).max()
        c_ref, _ = orc.ttc_compressed(y_ref)
        c = s.cttc(r)
        rel = np.abs(c - c_ref).max() / np.abs(c_ref).max()
        assert rel <= 1e-5, rel
        _, g2_ref, cnt_ref = orc.g2_from_ttc(c_ref)
        _, g2, cnt = s.cg2(r)
        assert np.array_equal(cnt, cnt_ref)
        assert np.abs(g2 - g2_ref).max() <= 1e-5 * np.abs(g2_ref).max()


def test_bf16_mode_within_1e2(ctx, orc):
    t, h, w, q, k = 256, 64, 64, 2, 32
    frames = orc.gen_speckle(t, h, w, q, 0.3, 51)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames)
    basis = xg.Basis(lay, k, digits=2)
    vs = [_basis(orc, frames[:, ring == r], k, 60 + r) for r in range(q)]
    for r in range(q):
        basis.set_ring(r, vs[r])
    s.compress(basis).ttc_compressed(mode="bf16")
    for r in range(q):
        y_ref, _ = orc.compress_series(frames[:, ring == r].astype(np.float64), vs[r])
        c_ref, _ = orc.ttc_compressed(y_ref)
        assert np.abs(s.cttc(r) - c_ref).max() <= 1e-2 * np.abs(c_ref).max()


def test_full_rank_homomorphic_identity(ctx, orc):
    """Full-rank offline basis: C~ reproduces the raw TTC (Eq. 11 of the
    paper; reference test_correlate.cpp:58-65 at 1e-10 in f64) -- here to the
    F32-mode tolerance."""
    t, h, w, q = 96, 32, 32, 1
    frames = orc.gen_speckle(t, h, w, q, 1.0, 71)
    ring = np.zeros(h * w, np.int32)
    xn, _ = orc.row_normalize(frames.astype(np.float64))
    # orthonormal basis of the row space (full rank k = t)
    qm, _ = np.linalg.qr(xn.T)
    k = qm.shape[1]
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    basis = xg.Basis(lay, k).set_ring(0, qm)
    s.compress(basis).ttc_compressed()
    c_raw = s.ttc(0)
    assert np.abs(s.cttc(0) - c_raw).max() <= 1e-5


def test_compressed_g2_only_mode(ctx, orc):
    t, h, w, q, k = 300, 48, 48, 2, 16
    frames = orc.gen_speckle(t, h, w, q, 0.4, 52)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    basis = xg.Basis(lay, k)
    for r in range(q):
        basis.set_ring(r, _basis(orc, frames[:, ring == r], k, 70 + r))
    a = xg.FrameSeries(lay, t).load(frames).compress(basis).ttc_compressed()
    b = xg.FrameSeries(lay, t).load(frames).compress(basis).ttc_compressed(store=False)
    for r in range(q):
        assert np.array_equal(a.cg2(r)[1], b.cg2(r)[1])
    with pytest.raises(xg.ContractError):
        b.cttc(0)


def test_chunked_compress_equals_one_shot(ctx, orc):
    """A series fed in chunks through a frame buffer smaller than the series
    (xg_series_compress_chunk) gives bitwise the batch coefficients, C~ and
    g2; the raw path is refused on it."""
    t, h, w, q, k = 700, 48, 48, 2, 32
    frames = orc.gen_speckle(t, h, w, q, 0.4, 61)
    frames[300] = 0  # a zero frame inside a chunk
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    basis = xg.Basis(lay, k)
    for r in range(q):
        basis.set_ring(r, _basis(orc, frames[:, ring == r], k, 80 + r))
    one = xg.FrameSeries(lay, t).load(frames).compress(basis).ttc_compressed()
    ch = xg.FrameSeries(lay, t, x_frames=256)
    for i, t0 in enumerate(range(0, t, 250)):
        ch.compress_chunk(basis, frames[t0:t0 + 250], first=(i == 0))
    ch.ttc_compressed()
    for r in range(q):
        y1, n1 = one.coeffs(r)
        y2, n2 = ch.coeffs(r)
        assert np.array_equal(y1, y2) and np.array_equal(n1, n2)
        assert np.array_equal(one.cttc(r), ch.cttc(r))
        assert np.array_equal(one.cg2(r)[1], ch.cg2(r)[1])
        assert np.array_equal(one.cg2(r)[2], ch.cg2(r)[2])
    with pytest.raises(xg.ContractError):
        ch.ttc_raw()
    # the chunked series' g2 by FFT of its coefficients (no C~), zero frame
    # included: same counts, same values to the fused path's fp32 accuracy
    fused = [ch.cg2(r) for r in range(q)]
    ch.ttc_compressed(store=False, spectral=True)
    for r in range(q):
        _, g_sp, c_sp = ch.cg2(r)
        assert np.array_equal(c_sp, fused[r][2])
        assert np.abs(g_sp - fused[r][1]).max() <= 1e-5 * np.abs(fused[r][1]).max()


def test_rel_error_report_matches_oracle(ctx, orc):
    """Device ttc_rel_error(raw C, compressed C~) per ring equals the oracle's
    ttc_rel_error on the same two matrices (sum order differs: 1e-12 rel)."""
    t, h, w, q, k = 300, 48, 48, 3, 8
    frames = orc.gen_speckle(t, h, w, q, 0.4, 91)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    basis = xg.Basis(lay, k)
    for r in range(q):
        basis.set_ring(r, _basis(orc, frames[:, ring == r], k, 90 + r))
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw().compress(basis).ttc_compressed()
    rel = s.rel_error()
    for r in range(q):
        ref = orc.ttc_rel_error(s.ttc(r, "f64"), s.cttc(r).astype(np.float64))
        assert abs(rel[r] - ref) <= 1e-12 * ref + 1e-15, (r, rel[r], ref)
        assert 0.0 < rel[r] < 1.0


def _g2_exact(y, nr):
    """f64 g2 of C~ = Y Y^T over the nonzero frames (per-lag dot products)."""
    n = y.shape[0]
    ok = nr > 0
    sums = np.zeros(n)
    cnt = np.zeros(n, np.int64)
    for d in range(n):
        sums[d] = float(np.einsum("ij,ij->", y[: n - d], y[d:]))
        cnt[d] = int(np.sum(ok[: n - d] & ok[d:]))
    return np.where(cnt > 0, sums / np.maximum(cnt, 1), 0.0), cnt


@pytest.mark.parametrize("t,k,zero", [(1500, 16, False), (4100, 8, False), (9000, 5, True)])
def test_spectral_g2_matches_exact_and_fused(ctx, orc, t, k, zero):
    """XG_G2_SPECTRAL: g2 from the FFT of the coefficient series (one and
    several 4096-frame blocks, odd k, a flagged frame) equals the f64 g2 of
    Y Y^T to 1e-11 and the fused-epilogue g2 to its fp32 accuracy."""
    h = w = 32
    q = 2
    frames = orc.gen_speckle(t, h, w, q, 0.5, 90 + k)
    ring, _ = orc.ring_map(h, w, q)
    if zero:
        frames = frames.copy()
        frames[4500, ring == 1] = 0
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    basis = xg.Basis(lay, k)
    xg.FrameSeries(lay, 64).load(frames[:64]).build_basis(k, basis=basis)
    s = xg.FrameSeries(lay, t).load(frames).compress(basis)
    s.ttc_compressed(store=False, spectral=True)
    spec = [s.cg2(r) for r in range(q)]
    s.ttc_compressed(store=False)
    for r in range(q):
        y, nr = s.coeffs(r)
        g_ex, c_ex = _g2_exact(y, nr)
        _, g_sp, c_sp = spec[r]
        _, g_fu, c_fu = s.cg2(r)
        assert np.array_equal(c_sp, c_ex) and np.array_equal(c_sp, c_fu)
        assert np.abs(g_sp - g_ex).max() <= 1e-11 * np.abs(g_ex).max()
        assert np.abs(g_sp - g_fu).max() <= 1e-5 * np.abs(g_ex).max()
    with pytest.raises(xg.ContractError):
        s.ttc_compressed(store=True, spectral=True)


def test_lossy_error_non_increasing_in_k(ctx, orc):
    """Reference test_correlate.cpp:80-93 on the device path: with the
    device-built offline basis truncated to k = 1 .. rank, ttc_rel_error(raw,
    compressed) (device) does not increase with k (to the F32 mode's noise)
    and full rank reaches the homomorphic identity."""
    t, h, w, q = 24, 32, 32, 1
    frames = orc.gen_speckle(t, h, w, q, 1.0, 95)
    ring = np.zeros(h * w, np.int32)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    vs, _, rank = xg.FrameSeries(lay, t).load(frames).build_basis(0)
    prev = 1e300
    for k in range(1, int(rank[0]) + 1):
        basis = xg.Basis(lay, k).set_ring(0, np.ascontiguousarray(vs[0][:, :k]))
        s.compress(basis).ttc_compressed()
        err = float(s.rel_error()[0])
        assert err <= prev + 2e-6, (k, err, prev)
        prev = err
    assert prev <= 1e-5  # full rank: C~ == C to the F32 mode's accuracy


def test_compressed_ttc_psd_and_unit_bounded(ctx, orc):
    """Reference test_correlate.cpp:95-106: C~ of a truncated basis is
    positive semidefinite and its diagonal <= 1 (here within the F32 mode's
    1e-5 contract; C~ = Y Y^T with |y_t| <= 1)."""
    t, h, w, q, k = 64, 32, 32, 2, 3
    frames = orc.gen_speckle(t, h, w, q, 0.8, 96)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames)
    basis = xg.Basis(lay, k)
    xg.FrameSeries(lay, t).load(frames).build_basis(k, basis=basis)
    s.compress(basis).ttc_compressed()
    for r in range(q):
        c = s.cttc(r)
        lam = np.linalg.eigvalsh(c)
        assert lam.min() >= -1e-5 * lam.max()
        assert np.diag(c).max() <= 1.0 + 1e-5
        y, _ = s.coeffs(r)
        assert np.linalg.norm(y, axis=1).max() <= 1.0 + 1e-12
