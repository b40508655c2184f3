"""The reference's Python surface (``xpcsvd``, proj/python/bindings.cpp) on the
B200 library: the hot-path properties the reference's own Python smoke tests
check (proj/python/tests/test_smoke.py: homomorphic identity, stream == batch,
ttc_extend == recompute, typed errors, mask selection), plus bitwise equality
with the reference library (oracle/_ref) on the same inputs."""
import numpy as np
import pytest

import paper_2407_20356_b200.xpcsvd as xv

pytestmark = pytest.mark.gpu


def _frames(n, m, seed):
    rng = np.random.default_rng(seed)
    return xv.FrameSeries(rng.exponential(1.0, size=(n, m)), 1.0)


def test_homomorphic_identity_end_to_end(ref):
    frames = _frames(24, 96, 3)
    enc = xv.build_offline(frames)
    store = xv.compress_series(frames, enc)
    g_raw = xv.ttc_raw(frames)
    g_cmp = xv.ttc_compressed(store)
    assert g_cmp.lossless
    assert np.abs(g_raw.values - g_cmp.values).max() <= 1e-10
    g2_raw, g2_cmp = xv.g2_from_ttc(g_raw, 1.0), xv.g2_from_ttc(g_cmp, 1.0)
    assert np.abs(g2_raw.values - g2_cmp.values).max() <= 1e-10
    assert g2_raw.counts == list(range(24, 0, -1))
    # the reference's bits on the same inputs
    assert np.array_equal(g_raw.values, ref.ttc_raw(frames.intensities))
    y_ref, n_ref = ref.compress_series(frames.intensities, enc.v)
    assert np.array_equal(store.coefficients, y_ref) and np.array_equal(store.norms, n_ref)
    c_ref, ll = ref.ttc_compressed(y_ref)
    assert ll and np.array_equal(g_cmp.values, c_ref)
    _, v_ref, _ = ref.g2_from_ttc(c_ref, 1.0)
    assert np.array_equal(g2_cmp.values, v_ref)


def test_streaming_matches_batch():
    frames = _frames(16, 64, 5)
    enc = xv.truncate(xv.build_offline(frames), 4)
    batch = xv.compress_series(frames, enc)
    stream = xv.CompressedSeries(4, batch.encoder_id)
    x = frames.intensities
    for t in range(16):
        coeffs, norm = xv.compress_frame(x[t], enc)
        stream.append(coeffs, norm)
    assert np.array_equal(stream.coefficients, batch.coefficients)
    assert np.array_equal(stream.norms, batch.norms)
    assert np.array_equal(xv.ttc_compressed(stream).values, xv.ttc_compressed(batch).values)


def test_ttc_extend_matches_recompute():
    frames = _frames(10, 48, 11)
    enc = xv.truncate(xv.build_offline(frames), 3)
    x = frames.intensities
    store = xv.CompressedSeries(3, xv.compress_series(frames, enc).encoder_id)
    for t in range(2):
        store.append(*xv.compress_frame(x[t], enc))
    g = xv.ttc_compressed(store)
    for t in range(2, 10):
        coeffs, norm = xv.compress_frame(x[t], enc)
        g = xv.ttc_extend(g, store, coeffs)
        store.append(coeffs, norm)
    g_batch = xv.ttc_compressed(xv.compress_series(frames, enc))
    assert np.array_equal(g.values, g_batch.values)
    with pytest.raises(xv.ShapeError):
        xv.ttc_extend(g, store, np.zeros(2))  # k mismatch


def test_errors_are_typed():
    frames = _frames(6, 24, 17)
    with pytest.raises(xv.RankError) as e:
        xv.build_online_from_frames(frames, 100)
    assert e.value.achievable_rank == 6
    with pytest.raises(xv.ContractError):
        xv.ttc_raw(_frames(1, 8, 1))
    zero = xv.FrameSeries(np.vstack([np.ones(8), np.zeros(8), np.ones(8)]), 1.0)
    with pytest.raises(xv.NormalizationError) as e:
        xv.ttc_raw(zero)
    assert e.value.frame_index == 1


def test_mask_selection_then_correlate(ref):
    frames = _frames(4, 16, 19)
    masked = xv.apply_mask(frames, xv.PixelMask(16, [1, 5, 7]))
    assert masked.n_pixels == 3
    assert np.array_equal(masked.intensities, frames.intensities[:, [1, 5, 7]])
    assert np.array_equal(xv.ttc_raw(masked).values, ref.ttc_raw(masked.intensities))


def test_count_data_takes_the_tensor_core_path(ref, monkeypatch):
    """Integer photon counts go through the exact u8 Gram (C within 1e-12 of
    the reference) and the device Gram-trick SVD (V within 1e-10); with
    XPCS_B200_EXACT=1 the f64 replicas return the reference's bits."""
    rng = np.random.default_rng(23)
    frames = xv.FrameSeries(rng.poisson(1.5, size=(60, 300)).astype(np.float64), 1.0)
    g = xv.ttc_raw(frames)
    g_ref = ref.ttc_raw(frames.intensities)
    assert np.abs(g.values - g_ref).max() <= 1e-12
    enc = xv.build_online_from_frames(frames, 12)
    v_ref, spec_ref = ref.build_online_from_frames(frames.intensities, 12)
    assert np.abs(enc.v - v_ref).max() <= 1e-10
    assert np.abs(np.asarray(enc.spectrum)[:spec_ref.size] - spec_ref).max() <= 1e-12 * spec_ref[0]
    zero = xv.FrameSeries(np.vstack([np.ones(8), np.zeros(8), 2 * np.ones(8)]), 1.0)
    with pytest.raises(xv.NormalizationError) as e:
        xv.ttc_raw(zero)
    assert e.value.frame_index == 1
    monkeypatch.setenv("XPCS_B200_EXACT", "1")
    assert np.array_equal(xv.ttc_raw(frames).values, g_ref)
