"""The CPU oracle (oracle/xpcs_oracle.c) pinned to the reference.

Bitwise against the committed golden vectors produced by the UNMODIFIED
reference (tests/golden/make_golden.py), and -- when oracle/_ref is built
(this container) -- against the live reference on more cases.  These are
the pins required before the oracle may judge the GPU path."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_rng_bitwise(orc, gold):
    idx = gold["rng_idx"]
    for seed, tag in [(1, 0), (7, 1), (7, 98), (2024, 3)]:
        base = orc.L.xo_rng_substream(seed, tag)
        bits = np.array([orc.L.xo_rng_bits(base, int(i)) for i in idx], np.uint64)
        assert np.array_equal(bits, gold[f"rng_bits_{seed}_{tag}"])
        nrm = np.array([orc.L.xo_rng_normal(base, int(i)) for i in idx])
        assert np.array_equal(nrm, gold[f"rng_normal_{seed}_{tag}"])
        ex = np.array([orc.L.xo_rng_exponential(base, int(i)) for i in idx])
        assert np.array_equal(ex, gold[f"rng_exp_{seed}_{tag}"])


def test_unit_fixtures_bitwise(orc, gold):
    x = orc.random_positive_matrix(8, 32, 1)
    assert np.array_equal(x, gold["ut_x_8x32"])
    assert np.array_equal(orc.ttc_raw(x), gold["ut_ttc_raw_8x32"])
    x2 = orc.random_positive_matrix(20, 20000, 5)
    assert np.array_equal(orc.gram(x2), gold["ut_gram_20x20000"])


def test_speckle_pipeline_bitwise(orc, gold):
    t, h, w, q, mu, seed = gold["sp_params"]
    t, h, w, q, seed = int(t), int(h), int(w), int(q), int(seed)
    frames = orc.gen_speckle(t, h, w, q, mu, seed)
    assert np.array_equal(frames, gold["sp_frames"])
    ring, _ = orc.ring_map(h, w, q)
    assert np.array_equal(ring, gold["sp_ring"])
    for r in range(q):
        xq = frames[:, ring == r]
        assert np.array_equal(orc.gram_u8(xq).astype(np.float64), gold[f"sp_gram_{r}"])
        assert np.array_equal(orc.gram(xq.astype(np.float64)), gold[f"sp_gram_{r}"])
        g = orc.ttc_raw(xq.astype(np.float64))
        assert np.array_equal(g, gold[f"sp_ttc_{r}"])
        lags, vals, cnt = orc.g2_from_ttc(g, 0.5)
        assert np.array_equal(vals, gold[f"sp_g2_{r}"])
        assert np.array_equal(cnt, gold[f"sp_g2cnt_{r}"])
        assert np.array_equal(lags, gold[f"sp_g2lags_{r}"])
        v = gold[f"sp_v_{r}"]
        y, nrm = orc.compress_series(xq.astype(np.float64), v)
        assert np.array_equal(y, gold[f"sp_y_{r}"])
        assert np.array_equal(nrm, gold[f"sp_norms_{r}"])
        gc, _ = orc.ttc_compressed(y)
        assert np.array_equal(gc, gold[f"sp_cttc_{r}"])
        # streaming extends == batch (correlate.cpp:37-65; SPEC "bitwise")
        assert np.array_equal(gold[f"sp_cttc_stream_{r}"], gc)
        st = gc[:2, :2].copy()
        for i in range(2, t):
            st, _ = orc.ttc_extend(st, y[:i], y[i])
        assert np.array_equal(st, gc)
        assert orc.ttc_rel_error(g, gc) == gold[f"sp_relerr_{r}"][0]


def test_int_gram_equals_f64_gram_and_normalisation_gap(orc, gold):
    """SURVEY finding 3: gram(counts) is exact integers; normalising the
    exact integer Gram afterwards is within 1e-12 of ttc_raw."""
    frames, ring = gold["sp_frames"], gold["sp_ring"]
    for r in range(int(gold["sp_params"][3])):
        gi = orc.gram_u8(frames[:, ring == r])
        n = np.sqrt(np.diag(gi).astype(np.float64))
        c = gi / np.outer(n, n)
        assert np.abs(c - gold[f"sp_ttc_{r}"]).max() <= 1e-12


def test_reference_tests_cases(orc):
    """Cases of the reference's own unit tests (test_correlate.cpp)."""
    g = orc.ttc_raw(np.array([[1.0, 2, 3, 4], [1, 2, 3, 4]]))
    assert np.allclose(g, 1.0, atol=1e-12)                        # :13-21
    g = orc.ttc_raw(np.array([[1.0, 1, 0, 0], [0, 0, 1, 1]]))
    assert abs(g[0, 1]) <= 1e-12 and abs(g[0, 0] - 1) <= 1e-12    # :23-29
    x = orc.random_positive_matrix(8, 32, 1)                      # :31-46 naive oracle
    g = orc.ttc_raw(x)
    n = np.sqrt((x * x).sum(1))
    assert np.abs(g - (x @ x.T) / np.outer(n, n)).max() <= 1e-12
    with pytest.raises(oracle.OracleError):                       # :54 (N < 2)
        orc.ttc_raw(orc.random_positive_matrix(1, 8, 3))
    lags, vals, cnt = orc.g2_from_ttc(np.ones((4, 4)), 2.0)       # :159-167
    assert list(vals) == [1.0] * 4 and list(lags) == [0, 2, 4, 6] and list(cnt) == [4, 3, 2, 1]
    _, vals, _ = orc.g2_from_ttc(np.eye(4))                       # :169-175
    assert list(vals) == [1.0, 0.0, 0.0, 0.0]
    z = np.zeros((3, 16))                                         # test_compress.cpp:49-64
    z[0, 0] = 1.0
    z[2, 3] = 1.0
    with pytest.raises(oracle.OracleError) as ei:
        orc.compress_series(z, np.eye(16)[:, :4])
    assert ei.value.payload == 1


def test_generator_subset_and_determinism(orc):
    f = orc.gen_speckle(30, 20, 28, 4, 0.4, 11)
    assert np.array_equal(f, orc.gen_speckle(30, 20, 28, 4, 0.4, 11))
    pix = np.array([0, 3, 55, 200, 559])
    assert np.array_equal(orc.gen_speckle_pixels(30, 20, 28, 4, 0.4, 11, pix), f[:, pix])
    m = orc.gen_speckle(400, 32, 32, 2, 0.1, 3)
    assert abs(m.mean() - 0.1) < 0.01                             # mean photons / pixel


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_live_reference_random_cases(orc, ref):
    rng = np.random.default_rng(5)
    for n, m in [(5, 7), (33, 1000), (12, 16385), (3, 40000)]:
        x = rng.exponential(size=(n, m))
        assert np.array_equal(orc.gram(x), ref.gram(x))
        assert np.array_equal(orc.ttc_raw(x), ref.ttc_raw(x))
        v = np.linalg.qr(rng.standard_normal((m, min(n, 6))))[0]
        assert all(np.array_equal(a, b) for a, b in zip(orc.compress_series(x, v),
                                                        ref.compress_series(x, v)))
        for i in range(n):
            a, b = orc.compress_frame(x[i], v), ref.compress_frame(x[i], v)
            assert np.array_equal(a[0], b[0]) and a[1] == b[1]
