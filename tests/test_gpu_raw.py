"""Raw TTC parity on the GPU (K1 ingest + K2 tcgen05 int8 Gram + K7 g2)
against the CPU oracle, through the C ABI.

Bar: (i) the int32 Gram equals xpcs::gram(counts) bitwise;
(ii) the normalised C is within 1e-12 abs of ttc_raw (reference tolerance,
test_correlate.cpp:43); g2 within 1e-12 of g2_from_ttc(ttc_raw)."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


def _data(orc, t, h, w, q, mu, seed):
    frames = orc.gen_speckle(t, h, w, q, mu, seed)
    ring, _ = orc.ring_map(h, w, q)
    return frames, ring


@pytest.mark.parametrize("t,h,w,q,mu,seed", [
    (300, 64, 64, 8, 0.1, 11),     # partial 128/256 tiles
    (64, 32, 48, 3, 0.5, 12),      # single tile, non-square detector
    (520, 96, 96, 5, 0.08, 13),    # several tile rows/cols
])
def test_raw_gram_bitwise_and_ttc(ctx, orc, t, h, w, q, mu, seed):
    frames, ring = _data(orc, t, h, w, q, mu, seed)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    for r in range(q):
        idx = np.nonzero(ring == r)[0]
        xq = frames[:, idx]
        g_ref = orc.gram_u8(xq)
        g_gpu = s.ttc(r, "gram")
        assert np.array_equal(g_gpu.astype(np.int64), g_ref), f"ring {r}: int Gram mismatch"
        c_gpu = s.ttc(r, "f64")
        c_ref = orc.ttc_raw(xq.astype(np.float64))
        assert np.abs(c_gpu - c_ref).max() <= 1e-12
        assert np.array_equal(c_gpu, c_gpu.T)
        _, g2_ref, cnt_ref = orc.g2_from_ttc(c_ref)
        _, g2_gpu, cnt_gpu = s.g2(r)
        assert np.array_equal(cnt_gpu, cnt_ref)
        assert np.abs(g2_gpu - g2_ref).max() <= 1e-12
        norms, nz = s.norms(r)
        assert nz == 0
        assert np.array_equal(norms, np.sqrt((xq.astype(np.float64) ** 2).sum(1)))


@pytest.mark.parametrize("kind", ["scattered", "thin"])
def test_raw_gram_irregular_masks(ctx, orc, kind):
    """Masks whose runs are shorter than 4 pixels (scattered pixels, 1-2 px
    rings) exercise the ingest's multi-run groups and byte-gather path."""
    t, h, w, q = 200, 100, 110, 7
    frames = orc.gen_speckle(t, h, w, 4, 0.2, 21)
    rng = np.random.default_rng(5)
    if kind == "scattered":
        ring = rng.integers(-1, q, size=h * w).astype(np.int32)
    else:
        yy, xx = np.mgrid[0:h, 0:w]
        rad = np.hypot(yy - h / 2, xx - w / 2).ravel()
        ring = np.where(rad < 2 * q * 1.5, (rad / 1.5).astype(np.int32) % q, -1).astype(np.int32)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    for r in range(q):
        xq = frames[:, np.nonzero(ring == r)[0]]
        assert np.array_equal(s.ttc(r, "gram").astype(np.int64), orc.gram_u8(xq)), f"ring {r}"
        norms, _ = s.norms(r)
        assert np.array_equal(norms, np.sqrt((xq.astype(np.float64) ** 2).sum(1)))


def test_raw_against_reference_library(ctx, orc, ref):
    """Same check against the UNMODIFIED reference (oracle/_ref)."""
    t, h, w, q = 200, 48, 48, 4
    frames, ring = _data(orc, t, h, w, q, 0.1, 21)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    for r in range(q):
        xq = frames[:, ring == r].astype(np.float64)
        assert np.array_equal(s.ttc(r, "gram").astype(np.float64), ref.gram(xq))
        c_ref = ref.ttc_raw(xq)
        assert np.abs(s.ttc(r, "f64") - c_ref).max() <= 1e-12


def test_zero_frame_strict_and_flagged(ctx, orc):
    t, h, w, q = 40, 16, 16, 2
    frames, ring = _data(orc, t, h, w, q, 0.3, 5)
    frames[7, ring == 0] = 0
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames)
    with pytest.raises(xg.NormalizationError) as ei:
        s.ttc_raw(strict=True)
    assert ei.value.frame_index == 7 and ei.value.ring == 0
    s.ttc_raw()
    _, nz = s.norms(0)
    assert nz == 1
    _, _, cnt = s.g2(0)
    assert cnt[0] == t - 1


def test_fused_g2_matches_standalone_pass(ctx, orc):
    """g2 from the K2 epilogue (per-tile diagonal sums + fold) equals the
    independent standalone pass over the stored Gram to rounding, and both
    hit the oracle."""
    t, h, w, q = 700, 64, 64, 3
    frames, ring = _data(orc, t, h, w, q, 0.1, 31)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    fused = [s.g2(r) for r in range(q)]
    s.compute_g2()
    for r in range(q):
        _, v2, c2 = s.g2(r)
        _, v1, c1 = fused[r]
        assert np.array_equal(c1, c2)
        assert np.abs(v1 - v2).max() <= 1e-13
        c_ref = orc.ttc_raw(frames[:, ring == r].astype(np.float64))
        assert np.abs(v1 - orc.g2_from_ttc(c_ref)[1]).max() <= 1e-12


@pytest.mark.parametrize("t,h,w", [(2, 3, 5), (3, 1, 7), (129, 17, 31), (257, 130, 130)])
def test_raw_tiny_and_odd_shapes(ctx, orc, t, h, w):
    """Smallest series (T=2), detectors smaller than one 16-byte vector or not
    a multiple of 16 pixels (the ingest's non-bulk band copy), single-pixel
    rings, tile-edge frame counts (T = 128k+1, 256k+1) and band edges."""
    rng = np.random.default_rng(t + h + w)
    frames = rng.integers(0, 4, size=(t, h * w), dtype=np.uint8)
    frames[:, 0] = 1  # ring 0 below has one pixel, keep it nonzero
    m = h * w
    masks = [np.array([0]), np.arange(1, m, 2), np.arange(2, m, 2)]
    masks = [mk for mk in masks if mk.size]
    lay = xg.RingLayout(ctx, m, masks)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    for r, mk in enumerate(masks):
        xq = frames[:, mk]
        assert np.array_equal(s.ttc(r, "gram").astype(np.int64), orc.gram_u8(xq)), f"ring {r}"
        c = s.ttc(r, "f64")
        assert np.abs(c - orc.ttc_raw(xq.astype(np.float64))).max() <= 1e-12
        _, g2, cnt = s.g2(r)
        _, g2_ref, cnt_ref = orc.g2_from_ttc(orc.ttc_raw(xq.astype(np.float64)))
        assert np.array_equal(cnt, cnt_ref) and np.abs(g2 - g2_ref).max() <= 1e-12


def test_raw_rejects_single_frame_and_bad_masks(ctx):
    lay = xg.RingLayout(ctx, 16, [np.arange(4)])
    with pytest.raises(xg.ContractError):
        xg.FrameSeries(lay, 1).load(np.ones((1, 16), np.uint8)).ttc_raw()
    with pytest.raises(xg.MaskError):
        xg.RingLayout(ctx, 16, [np.array([3, 3])])
    with pytest.raises(xg.MaskError):
        xg.RingLayout(ctx, 16, [np.array([16])])
    with pytest.raises(xg.MaskError):
        xg.RingLayout(ctx, 16, [np.array([], dtype=np.int64)])
    with pytest.raises(xg.ShapeError):
        xg.FrameSeries(lay, 4).load(np.ones((5, 16), np.uint8))


def test_int32_gram_overflow_is_a_contract_error(ctx):
    """The exact int32 Gram holds |x|^2 < 2^31 (255^2 * 33025 pixels); a
    brighter ring is refused with ContractError (SURVEY 8 K2 int32 overflow),
    never wrapped.  Just below the limit stays exact."""
    m = 34000
    lay = xg.RingLayout(ctx, m, [np.arange(m)])
    hot = np.full((2, m), 255, np.uint8)
    s = xg.FrameSeries(lay, 2).load(hot)
    with pytest.raises(xg.ContractError):  # device-detected: raised by the next sync
        s.ttc_raw()
        s.ttc(0, "gram")
    ok = hot.copy()
    ok[:, 33000:] = 0  # 255^2 * 33000 < 2^31
    s = xg.FrameSeries(lay, 2).load(ok).ttc_raw()
    assert s.ttc(0, "gram")[0, 1] == 255 * 255 * 33000


def test_host_overlapped_path_equals_two_calls(ctx, orc):
    """ttc_raw_host (chunked H2D overlapped with ingest and per-column-block
    Gram launches) gives bitwise the same Gram, C and g2 as load + ttc_raw."""
    t, h, w, q = 1300, 40, 40, 3
    frames, ring = _data(orc, t, h, w, q, 0.3, 41)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    a = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    b = xg.FrameSeries(lay, t).ttc_raw_host(frames)
    for r in range(q):
        assert np.array_equal(a.ttc(r, "gram"), b.ttc(r, "gram"))
        assert np.array_equal(a.ttc(r, "f64"), b.ttc(r, "f64"))
        _, ga, ca = a.g2(r)
        _, gb, cb = b.g2(r)
        assert np.array_equal(ga, gb) and np.array_equal(ca, cb)
    _, gall, call = b.g2_all()
    for r in range(q):
        _, gr, cr = b.g2(r)
        assert np.array_equal(gall[r], gr) and np.array_equal(call[r], cr)


def test_g2_only_mode_equals_stored_mode(ctx, orc):
    """store=False (XG_NO_STORE): the fused g2 without writing any TTC tile
    equals the stored run's g2 bitwise; TTC readback is refused."""
    t, h, w, q = 400, 40, 40, 3
    frames, ring = _data(orc, t, h, w, q, 0.2, 51)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    a = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    b = xg.FrameSeries(lay, t).load(frames).ttc_raw(store=False)
    for r in range(q):
        _, ga, ca = a.g2(r)
        _, gb, cb = b.g2(r)
        assert np.array_equal(ga, gb) and np.array_equal(ca, cb)
    with pytest.raises(xg.ContractError):
        b.ttc(0)


def test_bright_frames_take_the_fp64_g2_path(ctx, orc):
    """|x|^2 >= 2^23 (bright rings): the Gram entries are no longer exact in
    fp32, so the fused g2 runs its FP64 branch (weights from the staged
    (hi, lo) split of 1/|x|).  g2 still within 1e-12 of the oracle."""
    t, m = 300, 4000
    rng = np.random.default_rng(77)
    frames = rng.integers(100, 256, size=(t, m), dtype=np.uint8)  # |x|^2 ~ 1e8 > 2^23
    lay = xg.RingLayout(ctx, m, [np.arange(0, m, 2), np.arange(1, m, 2)])
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    for r, idx in enumerate([np.arange(0, m, 2), np.arange(1, m, 2)]):
        xq = frames[:, idx].astype(np.float64)
        assert (xq ** 2).sum(1).max() >= 2 ** 23
        c_ref = orc.ttc_raw(xq)
        _, g2_ref, cnt_ref = orc.g2_from_ttc(c_ref)
        _, g2, cnt = s.g2(r)
        assert np.array_equal(cnt, cnt_ref)
        assert np.abs(g2 - g2_ref).max() <= 1e-12


def test_megapixel_detector_many_bands(ctx, orc):
    """C3/C4 geometry (1024 x 1024, 50 rings: 64 ingest bands of 16384
    pixels, rings crossing band edges, many pieces per band): exact Gram and
    norms of sampled rings against the oracle."""
    t, h, w, q = 160, 1024, 1024, 50
    rng = np.random.default_rng(88)
    frames = rng.poisson(0.05, size=(t, h * w)).clip(0, 255).astype(np.uint8)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    s = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    for r in (0, 7, 24, 49):
        xq = frames[:, ring == r]
        assert np.array_equal(s.ttc(r, "gram").astype(np.int64), orc.gram_u8(xq)), f"ring {r}"
        norms, _ = s.norms(r)
        assert np.array_equal(norms, np.sqrt((xq.astype(np.float64) ** 2).sum(1)))
