"""Reference-facing f64 entries (K9): the reference's operation order on the
GPU, so results must equal the oracle (itself pinned bitwise to the
reference) BIT FOR BIT -- including the reference's own acceptance
invariants: streaming extends == batch, stripes > 16384 pixels, zero-skip
projection, sequential g2."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,seed", [(8, 32, 1), (37, 1000, 2), (9, 20000, 3), (2, 5, 4)])
def test_ttc_raw_bitwise(ctx, orc, n, m, seed):
    x = orc.random_positive_matrix(n, m, seed)
    assert np.array_equal(xg.ttc_raw(x), orc.ttc_raw(x))


def test_ttc_raw_counts_and_errors(ctx, orc):
    f = orc.gen_speckle(120, 32, 32, 2, 0.3, 9).astype(np.float64)
    assert np.array_equal(xg.ttc_raw(f), orc.ttc_raw(f))
    with pytest.raises(xg.ContractError):
        xg.ttc_raw(f[:1])
    z = f[:10].copy()
    z[6] = 0.0
    with pytest.raises(xg.NormalizationError) as ei:
        xg.ttc_raw(z)
    assert ei.value.frame_index == 6


def test_compress_series_frame_bitwise(ctx, orc):
    f = orc.gen_speckle(64, 24, 24, 1, 0.5, 3).astype(np.float64)   # sparse counts
    v = np.linalg.qr(np.random.default_rng(0).standard_normal((576, 12)))[0]
    y, n = xg.compress_series(f, v)
    y0, n0 = orc.compress_series(f, v)
    assert np.array_equal(y, y0) and np.array_equal(n, n0)
    for i in (0, 5, 63):
        c, nr = xg.compress_frame(f[i], v)
        c0, nr0 = orc.compress_frame(f[i], v)
        assert np.array_equal(c, c0) and nr == nr0
        assert np.array_equal(c, y[i])            # stream == batch (compress.cpp:64)


def test_compress_series_u8_counts_bitwise(ctx, orc):
    """xg_f64_compress_series_u8 (the drop-in's route for integer counts: u8
    over PCIe, widened on the device) == the f64 entry == the oracle, bit for
    bit, at sizes where the widening kernel's 16-byte body and ragged tail
    both run; a zero frame keeps its index."""
    import ctypes as C

    from paper_2407_20356_b200 import _abi

    def run(fn, x, v):
        n, m = x.shape
        k = v.shape[1]
        y = np.empty((n, k))
        nr = np.empty(n)
        rc = fn(x.ctypes.data_as(C.c_void_p if x.dtype == np.uint8 else _abi.PD), n, m,
                v.ctypes.data_as(_abi.PD), k, y.ctypes.data_as(_abi.PD), nr.ctypes.data_as(_abi.PD))
        return rc, y, nr

    for (t, h, w, mu, k, seed) in [(64, 24, 24, 0.5, 12, 3), (33, 17, 13, 3.0, 7, 4)]:
        f8 = orc.gen_speckle(t, h, w, 1, mu, seed)
        f = f8.astype(np.float64)
        v = np.linalg.qr(np.random.default_rng(seed).standard_normal((h * w, k)))[0]
        rc8, y8, n8 = run(_abi.lib.xg_f64_compress_series_u8, np.ascontiguousarray(f8), v)
        rc, y, n = run(_abi.lib.xg_f64_compress_series, f, v)
        assert rc8 == 0 and rc == 0
        y0, n0 = orc.compress_series(f, v)
        assert np.array_equal(y8, y) and np.array_equal(n8, n)
        assert np.array_equal(y8, y0) and np.array_equal(n8, n0)
    f8 = np.ascontiguousarray(f8)
    f8[5] = 0
    rc8, _, _ = run(_abi.lib.xg_f64_compress_series_u8, f8, v)
    assert rc8 == _abi.ERR_NORMALIZATION and _abi.lib.xg_f64_last_payload() == 5


def test_ttc_compressed_extend_g2_bitwise(ctx, orc):
    x = orc.random_positive_matrix(50, 128, 8)
    v = np.linalg.qr(np.random.default_rng(1).standard_normal((128, 5)))[0]
    y, _ = orc.compress_series(x, v)
    g, ll = xg.ttc_compressed(y)
    g0, ll0 = orc.ttc_compressed(y)
    assert np.array_equal(g, g0) and ll == ll0
    # sequential extends == batch bitwise (test_correlate.cpp:138-157)
    st, _ = xg.ttc_compressed(y[:2])
    for t in range(2, 50):
        st, _ = xg.ttc_extend(st, y[:t], y[t])
    assert np.array_equal(st, g)
    for period in (1.0, 0.25):
        for a, b in zip(xg.g2_from_ttc(g, period), orc.g2_from_ttc(g, period)):
            assert np.array_equal(a, b)
    graw = orc.ttc_raw(x)
    assert xg.ttc_rel_error(graw, g) == orc.ttc_rel_error(graw, g)


def test_full_rank_homomorphic_identity_f64(ctx, orc, ref):
    """acceptance criterion 1 / test_correlate.cpp:58-65 through the GPU entries."""
    x = orc.random_positive_matrix(16, 64, 4)
    v = ref.build_offline(x)
    y, _ = xg.compress_series(x, v)
    g, ll = xg.ttc_compressed(y)
    assert ll
    assert np.abs(g - xg.ttc_raw(x)).max() <= 1e-10
