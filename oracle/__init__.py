"""CPU checkers for the XPCS correlation hot path -- TEST INFRASTRUCTURE ONLY.

Two independent CPU implementations live here:

* ``C``   -- ctypes over ``liboracle.so``, the C restatement in
  ``xpcs_oracle.c`` (bit-for-bit the reference's operation order).
* ``Ref`` -- ctypes over ``_ref/libxpcsvd_ref.so``, the UNMODIFIED reference
  library compiled from ``/root/reference`` by ``oracle/Makefile``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` / ``--impl reference`` legs) may import this package, and
only as the checker or the timed CPU baseline -- never as the product.  The
product (``paper_2407_20356_b200``) must not import it.
"""
from __future__ import annotations

import ctypes as C_
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libxpcsvd_ref.so")

_d = C_.POINTER(C_.c_double)
_i64 = C_.POINTER(C_.c_int64)
_u8 = C_.POINTER(C_.c_uint8)
_i32 = C_.POINTER(C_.c_int32)
I64 = C_.c_int64
U64 = C_.c_uint64


def _p(a: np.ndarray, ty):
    return a.ctypes.data_as(ty)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code: int, payload: int = -1):
        super().__init__(f"oracle error code {code} payload {payload}")
        self.code = code
        self.payload = payload


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class _COracle:
    """The C restatement (xpcs_oracle.c)."""

    def __init__(self, path: str = LIB_ORACLE):
        L = C_.CDLL(path)
        self.L = L
        L.xo_rng_substream.restype = U64
        L.xo_rng_substream.argtypes = [U64, U64]
        L.xo_rng_bits.restype = U64
        L.xo_rng_bits.argtypes = [U64, U64]
        for f in ("xo_rng_uniform", "xo_rng_normal", "xo_rng_exponential"):
            getattr(L, f).restype = C_.c_double
            getattr(L, f).argtypes = [U64, U64]
        L.xo_random_positive_matrix.argtypes = [I64, I64, U64, _d]
        L.xo_random_matrix.argtypes = [I64, I64, U64, _d]
        L.xo_dot.restype = C_.c_double
        L.xo_dot.argtypes = [_d, _d, I64]
        L.xo_gram.argtypes = [_d, I64, I64, _d]
        L.xo_gram_u8.argtypes = [_u8, I64, I64, _i64]
        L.xo_row_normalize.restype = I64
        L.xo_row_normalize.argtypes = [_d, I64, I64, _d, _d]
        L.xo_ttc_raw.restype = I64
        L.xo_ttc_raw.argtypes = [_d, I64, I64, _d]
        L.xo_ttc_compressed.restype = C_.c_int
        L.xo_ttc_compressed.argtypes = [_d, I64, I64, _d]
        L.xo_ttc_extend.restype = C_.c_int
        L.xo_ttc_extend.argtypes = [_d, I64, _d, I64, _d, _d]
        L.xo_g2_from_ttc.argtypes = [_d, I64, C_.c_double, _d, _d, _i64]
        L.xo_ttc_rel_error.restype = C_.c_double
        L.xo_ttc_rel_error.argtypes = [_d, _d, I64]
        L.xo_compress_frame.restype = C_.c_int
        L.xo_compress_frame.argtypes = [_d, I64, _d, I64, _d, _d]
        L.xo_compress_series.restype = I64
        L.xo_compress_series.argtypes = [_d, I64, I64, _d, I64, _d, _d]
        L.xo_apply_mask.argtypes = [_d, I64, I64, _i64, I64, _d]
        L.xo_ring_map.argtypes = [I64, I64, I64, _i32, _d]
        L.xo_gen_speckle.argtypes = [I64, I64, I64, I64, C_.c_double, C_.c_int,
                                     C_.c_double, U64, _u8]
        L.xo_gen_speckle_pixels.argtypes = [I64, I64, I64, I64, C_.c_double, C_.c_int,
                                            C_.c_double, U64, _i64, I64, _u8]

    # -- rng / fixtures
    def random_positive_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols), np.float64)
        self.L.xo_random_positive_matrix(rows, cols, seed, _p(out, _d))
        return out

    def random_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols), np.float64)
        self.L.xo_random_matrix(rows, cols, seed, _p(out, _d))
        return out

    # -- linalg / correlate
    def gram(self, x):
        x = _f64(x)
        n, m = x.shape
        g = np.empty((n, n), np.float64)
        self.L.xo_gram(_p(x, _d), n, m, _p(g, _d))
        return g

    def gram_u8(self, x):
        x = np.ascontiguousarray(x, dtype=np.uint8)
        n, m = x.shape
        g = np.empty((n, n), np.int64)
        self.L.xo_gram_u8(_p(x, _u8), n, m, _p(g, _i64))
        return g

    def row_normalize(self, x):
        x = _f64(x)
        n, m = x.shape
        out = np.empty_like(x)
        norms = np.empty(n, np.float64)
        bad = self.L.xo_row_normalize(_p(x, _d), n, m, _p(out, _d), _p(norms, _d))
        if bad >= 0:
            raise OracleError(4, bad)
        return out, norms

    def ttc_raw(self, x):
        x = _f64(x)
        n, m = x.shape
        g = np.empty((n, n), np.float64)
        bad = self.L.xo_ttc_raw(_p(x, _d), n, m, _p(g, _d))
        if bad == -2:
            raise OracleError(2)
        if bad >= 0:
            raise OracleError(4, bad)
        return g

    def ttc_compressed(self, y):
        y = _f64(y)
        n, k = y.shape
        g = np.empty((n, n), np.float64)
        lossless = self.L.xo_ttc_compressed(_p(y, _d), n, k, _p(g, _d))
        return g, bool(lossless)

    def ttc_extend(self, g, y, row):
        g, y, row = _f64(g), _f64(y), _f64(row)
        n, k = y.shape
        out = np.empty((n + 1, n + 1), np.float64)
        lossless = self.L.xo_ttc_extend(_p(g, _d), n, _p(y, _d), k, _p(row, _d), _p(out, _d))
        return out, bool(lossless)

    def g2_from_ttc(self, g, period=1.0):
        g = _f64(g)
        n = g.shape[0]
        lags = np.empty(n)
        vals = np.empty(n)
        counts = np.empty(n, np.int64)
        self.L.xo_g2_from_ttc(_p(g, _d), n, period, _p(lags, _d), _p(vals, _d),
                              _p(counts, _i64))
        return lags, vals, counts

    def ttc_rel_error(self, a, b):
        a, b = _f64(a), _f64(b)
        return self.L.xo_ttc_rel_error(_p(a, _d), _p(b, _d), a.size)

    # -- compress
    def compress_series(self, x, v):
        x, v = _f64(x), _f64(v)
        n, m = x.shape
        k = v.shape[1]
        coeffs = np.empty((n, k))
        norms = np.empty(n)
        bad = self.L.xo_compress_series(_p(x, _d), n, m, _p(v, _d), k, _p(coeffs, _d),
                                        _p(norms, _d))
        if bad >= 0:
            raise OracleError(4, bad)
        return coeffs, norms

    def compress_frame(self, frame, v):
        frame, v = _f64(frame), _f64(v)
        k = v.shape[1]
        coeffs = np.empty(k)
        norm = C_.c_double(0.0)
        if self.L.xo_compress_frame(_p(frame, _d), frame.size, _p(v, _d), k,
                                    _p(coeffs, _d), C_.byref(norm)):
            raise OracleError(4, 0)
        return coeffs, norm.value

    def apply_mask(self, x, idx):
        x = _f64(x)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        n, m = x.shape
        out = np.empty((n, idx.size))
        self.L.xo_apply_mask(_p(x, _d), n, m, _p(idx, _i64), idx.size, _p(out, _d))
        return out

    # -- synthetic data
    def ring_map(self, h, w, q):
        ring = np.empty(h * w, np.int32)
        rad = np.empty(h * w, np.float64)
        self.L.xo_ring_map(h, w, q, _p(ring, _i32), _p(rad, _d))
        return ring, rad

    def gen_speckle_pixels(self, t, h, w, q, mu, seed, pix, gamma_mode=0, gamma_a=0.002):
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        out = np.empty((t, pix.size), np.uint8)
        self.L.xo_gen_speckle_pixels(t, h, w, q, mu, gamma_mode, gamma_a, seed, _p(pix, _i64),
                                     pix.size, _p(out, _u8))
        return out

    def gen_speckle(self, t, h, w, q, mu, seed, gamma_mode=0, gamma_a=0.002):
        out = np.empty((t, h * w), np.uint8)
        self.L.xo_gen_speckle(t, h, w, q, mu, gamma_mode, gamma_a, seed, _p(out, _u8))
        return out


class _RefOracle:
    """The unmodified reference library (oracle/_ref/libxpcsvd_ref.so)."""

    def __init__(self, path: str = LIB_REF):
        L = C_.CDLL(path)
        self.L = L
        L.ref_last_payload.restype = I64
        L.ref_gram.argtypes = [_d, I64, I64, _d]
        L.ref_row_normalize.argtypes = [_d, I64, I64, _d, _d]
        L.ref_ttc_raw.argtypes = [_d, I64, I64, _d]
        L.ref_ttc_compressed.argtypes = [_d, _d, I64, I64, _d, C_.POINTER(C_.c_int)]
        L.ref_ttc_extend_stream.argtypes = [_d, _d, I64, I64, _d]
        L.ref_ttc_extend.argtypes = [_d, I64, _d, _d, I64, _d, _d]
        L.ref_g2_from_ttc.argtypes = [_d, I64, C_.c_double, _d, _d, _i64]
        L.ref_ttc_background.argtypes = [_d, I64, I64, _d]
        L.ref_read_compressed.argtypes = [C_.c_char_p, _i64, C_.POINTER(U64), _i64, _d, _d]
        L.ref_write_frames.argtypes = [C_.c_char_p, _d, I64, I64, C_.c_double, C_.c_int]
        L.ref_read_frames_status.argtypes = [C_.c_char_p, _i64, _i64]
        L.ref_write_encoder.argtypes = [C_.c_char_p, _d, I64, I64, _d, I64, C_.c_int]
        L.ref_read_encoder.argtypes = [C_.c_char_p, _i64, _i64, _i64, C_.POINTER(C_.c_int), _d, _d]
        L.ref_fit_kww.argtypes = [_d, _d, I64, C_.c_double, C_.c_double, _d]
        L.ref_ttc_rel_error.argtypes = [_d, _d, I64, _d]
        L.ref_compress_series.argtypes = [_d, I64, I64, _d, I64, _d, _d]
        L.ref_compress_frame.argtypes = [_d, I64, _d, I64, _d, _d]
        L.ref_build_online_from_frames.argtypes = [_d, I64, I64, I64, _d, _d, _i64]
        L.ref_build_offline.argtypes = [_d, I64, I64, _d, _i64]
        L.ref_apply_mask.argtypes = [_d, I64, I64, _i64, I64, _d]
        L.ref_content_hash.argtypes = [_d, I64, I64, C_.c_int, C_.POINTER(U64)]
        L.ref_rng_bits.restype = U64
        L.ref_rng_bits.argtypes = [U64, U64, U64]
        L.ref_rng_normal.restype = C_.c_double
        L.ref_rng_normal.argtypes = [U64, U64, U64]
        L.ref_rng_exponential.restype = C_.c_double
        L.ref_rng_exponential.argtypes = [U64, U64, U64]

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.L.ref_last_payload())

    def gram(self, x):
        x = _f64(x)
        n, m = x.shape
        g = np.empty((n, n))
        self._chk(self.L.ref_gram(_p(x, _d), n, m, _p(g, _d)))
        return g

    def ttc_raw(self, x):
        x = _f64(x)
        n, m = x.shape
        g = np.empty((n, n))
        self._chk(self.L.ref_ttc_raw(_p(x, _d), n, m, _p(g, _d)))
        return g

    def ttc_compressed(self, y, norms=None):
        y = _f64(y)
        n, k = y.shape
        norms = _f64(np.ones(n) if norms is None else norms)
        g = np.empty((n, n))
        ll = C_.c_int(0)
        self._chk(self.L.ref_ttc_compressed(_p(y, _d), _p(norms, _d), n, k, _p(g, _d),
                                            C_.byref(ll)))
        return g, bool(ll.value)

    def ttc_extend_stream(self, y, norms=None):
        y = _f64(y)
        n, k = y.shape
        norms = _f64(np.ones(n) if norms is None else norms)
        g = np.empty((n, n))
        self._chk(self.L.ref_ttc_extend_stream(_p(y, _d), _p(norms, _d), n, k, _p(g, _d)))
        return g

    def g2_from_ttc(self, g, period=1.0):
        g = _f64(g)
        n = g.shape[0]
        lags, vals = np.empty(n), np.empty(n)
        counts = np.empty(n, np.int64)
        self._chk(self.L.ref_g2_from_ttc(_p(g, _d), n, period, _p(lags, _d), _p(vals, _d),
                                         _p(counts, _i64)))
        return lags, vals, counts

    def read_compressed(self, path):
        """io::read_compressed -> (k, encoder hash, coefficients n x k, norms)."""
        k, n, h = I64(0), I64(0), U64(0)
        p = str(path).encode()
        self._chk(self.L.ref_read_compressed(p, C_.byref(k), C_.byref(h), C_.byref(n), None, None))
        y = np.empty((n.value, k.value))
        nr = np.empty(n.value)
        self._chk(self.L.ref_read_compressed(p, C_.byref(k), C_.byref(h), C_.byref(n), _p(y, _d),
                                             _p(nr, _d)))
        return k.value, h.value, y, nr

    def write_frames(self, path, x, period, dtype):
        x = _f64(x)
        self._chk(self.L.ref_write_frames(str(path).encode(), _p(x, _d), x.shape[0], x.shape[1],
                                          period, dtype))

    def write_encoder(self, path, v, spectrum, mode):
        v, sp = _f64(v), _f64(spectrum)
        self._chk(self.L.ref_write_encoder(str(path).encode(), _p(v, _d), v.shape[0], v.shape[1],
                                           _p(sp, _d), sp.size, mode))

    def read_encoder(self, path):
        """io::read_encoder -> (V, spectrum, mode); raises OracleError(7) on FormatError."""
        m, k, sl, md = I64(0), I64(0), I64(0), C_.c_int(0)
        p = str(path).encode()
        self._chk(self.L.ref_read_encoder(p, C_.byref(m), C_.byref(k), C_.byref(sl), C_.byref(md),
                                          None, None))
        v = np.empty((m.value, k.value))
        sp = np.empty(sl.value)
        self._chk(self.L.ref_read_encoder(p, C_.byref(m), C_.byref(k), C_.byref(sl), C_.byref(md),
                                          _p(v, _d), _p(sp, _d)))
        return v, sp, md.value

    def read_frames_status(self, path):
        """(status, payload): 0 ok, 7 FormatError (payload = byte offset)."""
        n, m = I64(0), I64(0)
        rc = self.L.ref_read_frames_status(str(path).encode(), C_.byref(n), C_.byref(m))
        return rc, self.L.ref_last_payload()

    def ttc_background(self, g, exclusion=0):
        g = _f64(g)
        out = C_.c_double(0.0)
        self._chk(self.L.ref_ttc_background(_p(g, _d), g.shape[0], exclusion, C_.byref(out)))
        return out.value

    def fit_kww(self, lags, values, min_lag, max_lag):
        """(status, [B, C, t0, rms]): status 0 ok, 10 FitDegenerateError,
        11 FitError (params = its best()), 2 ContractError."""
        lags, values = _f64(lags), _f64(values)
        out = np.zeros(4)
        rc = self.L.ref_fit_kww(_p(lags, _d), _p(values, _d), lags.size, min_lag, max_lag,
                                _p(out, _d))
        return rc, out

    def content_hash(self, v, mode):
        v = _f64(v)
        out = U64(0)
        self._chk(self.L.ref_content_hash(_p(v, _d), v.shape[0], v.shape[1], mode, C_.byref(out)))
        return int(out.value)

    def ttc_rel_error(self, a, b):
        a, b = _f64(a), _f64(b)
        out = C_.c_double(0)
        self._chk(self.L.ref_ttc_rel_error(_p(a, _d), _p(b, _d), a.shape[0], C_.byref(out)))
        return out.value

    def compress_series(self, x, v):
        x, v = _f64(x), _f64(v)
        n, m = x.shape
        k = v.shape[1]
        coeffs, norms = np.empty((n, k)), np.empty(n)
        self._chk(self.L.ref_compress_series(_p(x, _d), n, m, _p(v, _d), k, _p(coeffs, _d),
                                             _p(norms, _d)))
        return coeffs, norms

    def compress_frame(self, frame, v):
        frame, v = _f64(frame), _f64(v)
        k = v.shape[1]
        coeffs = np.empty(k)
        norm = C_.c_double(0)
        self._chk(self.L.ref_compress_frame(_p(frame, _d), frame.size, _p(v, _d), k,
                                            _p(coeffs, _d), C_.byref(norm)))
        return coeffs, norm.value

    def build_online_from_frames(self, x, k):
        x = _f64(x)
        n, m = x.shape
        v = np.empty((m, k))
        spec = np.empty(n)
        slen = C_.c_int64(0)
        self._chk(self.L.ref_build_online_from_frames(_p(x, _d), n, m, k, _p(v, _d),
                                                      _p(spec, _d), C_.byref(slen)))
        return v, spec[: slen.value]

    def build_offline(self, x):
        x = _f64(x)
        n, m = x.shape
        v = np.empty((m, n))
        kk = C_.c_int64(0)
        self._chk(self.L.ref_build_offline(_p(x, _d), n, m, _p(v, _d), C_.byref(kk)))
        r = kk.value
        return np.ascontiguousarray(v.ravel()[: m * r].reshape(m, r))

    def apply_mask(self, x, idx):
        x = _f64(x)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        n, m = x.shape
        out = np.empty((n, idx.size))
        self._chk(self.L.ref_apply_mask(_p(x, _d), n, m, _p(idx, _i64), idx.size, _p(out, _d)))
        return out


_c = None
_ref = None


def c() -> _COracle:
    global _c
    if _c is None:
        if not os.path.exists(LIB_ORACLE):
            build()
        _c = _COracle()
    return _c


def ref_available() -> bool:
    return os.path.exists(LIB_REF)


def ref() -> _RefOracle:
    global _ref
    if _ref is None:
        _ref = _RefOracle()
    return _ref
