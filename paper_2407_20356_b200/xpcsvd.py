"""Drop-in for the reference's Python module ``xpcsvd`` on the correlation
hot path (proj/python/bindings.cpp:62-262), backed by the B200 library.

``import paper_2407_20356_b200.xpcsvd as xpcsvd`` gives the reference's
names, argument meanings, result types and exception classes for:

    PixelMask, FrameSeries, apply_mask, EncoderMode, EncodingMatrix,
    build_offline, build_online_from_frames, truncate, content_hash,
    CompressedSeries, compress_series, compress_frame,
    TTCMatrix, ttc_raw, ttc_compressed, ttc_extend, G2Curve, g2_from_ttc,
    ttc_rel_error

Routing, as the C++ drop-in (integration/b200_engine.hpp):
  * intensities that are integer photon counts in [0, 255] (detector data)
    take the tensor-core path: ``ttc_raw`` via the exact u8 int32 Gram (C
    within 1e-12 of the reference), the basis (``build_offline`` /
    ``build_online_from_frames``) via the device Gram-trick SVD (K9, V within
    1e-10 of the reference);
  * anything else, every other function, and every call under
    ``XPCS_B200_EXACT=1`` use the ``xg_f64_*`` entry points (k_exact.cu),
    which replay the reference's f64 operation order (the reference's bits),
    and, for the basis of non-count data, the library's host f64 restatement
    of gram_svd (setup only, untimed).
For u8 count data at scale use the batched ring API (``FrameSeries`` /
``RingLayout`` in the package root) directly.

The validation rules and messages follow model.cpp:10-40 (masks, series),
model.cpp:70-94 (encoders), model.cpp:139-212 (stores) and model.cpp:214-240
(TTC matrices).  Not mirrored (outside SURVEY.md section 8): file formats,
synthetic generators, analysis fits, decompress.
"""
from __future__ import annotations

import enum

import numpy as np

from . import (BindingError, ContractError, Context, DeviceError, Error, FormatError,  # noqa: F401
               MaskError, NormalizationError, RankError, ShapeError)
from . import _abi
from . import compress_frame as _compress_frame
from . import compress_series as _compress_series
from . import g2_from_ttc as _g2_from_ttc
from . import ttc_compressed as _ttc_compressed
from . import ttc_extend as _ttc_extend
from . import ttc_raw as _ttc_raw
from . import ttc_rel_error as _ttc_rel_error
from ._abi import lib

_CTX = None


def _ctx():
    """The xg_f64_* entry points run on the current device; keep one context
    alive so the device is initialised (and fail loudly without a B200)."""
    global _CTX
    if _CTX is None:
        _CTX = Context(0)
    return _CTX


def _exact_only() -> bool:
    import os

    return os.environ.get("XPCS_B200_EXACT") == "1"


def _as_counts(x: np.ndarray):
    """u8 copy when every intensity is an integer count in [0, 255], else None."""
    if _exact_only() or x.size == 0 or x.min() < 0 or x.max() > 255:
        return None
    if not np.array_equal(x, np.floor(x)):
        return None
    return x.astype(np.uint8)


def _one_ring_series(u8: np.ndarray):
    """A device series over one ring holding every pixel of ``u8``."""
    from . import FrameSeries as _Series, RingLayout as _Layout

    ctx = _ctx()
    n, m = u8.shape
    lay = _Layout(ctx, m, [np.arange(m, dtype=np.int64)])
    return _Series(lay, n).load(u8)


# ------------------------------------------------------------------ model
class PixelMask:
    """xpcs::PixelMask (model.hpp:16-24, model.cpp:10-26)."""

    def __init__(self, full_pixels: int, indices):
        idx = [int(i) for i in indices]
        if not idx:
            raise MaskError("pixel mask selects no pixels")
        for i, v in enumerate(idx):
            if v < 0 or v >= full_pixels:
                raise MaskError(f"mask index {v} out of range for {full_pixels} pixels")
            if i > 0 and v <= idx[i - 1]:
                raise MaskError(f"mask indices not strictly ascending at position {i}")
        self.full_pixels = int(full_pixels)
        self.indices = idx

    @property
    def count(self) -> int:
        return len(self.indices)


class FrameSeries:
    """xpcs::FrameSeries (model.hpp:26-36, model.cpp:28-40): non-negative
    f64 intensities (n x m), frame period, optional mask."""

    def __init__(self, intensities, frame_period: float = 1.0, mask: PixelMask | None = None):
        x = np.array(intensities, dtype=np.float64, copy=True)
        if x.ndim != 2:
            raise ShapeError("frame series must be a 2-D array (frames x pixels)")
        if not (frame_period > 0.0) or not np.isfinite(frame_period):
            raise ContractError("frame_period must be positive and finite")
        if np.any(x < 0.0):
            raise ContractError("negative intensity in frame series")
        if mask is not None and mask.count != x.shape[1]:
            raise MaskError(f"mask selects {mask.count} pixels but series has {x.shape[1]}")
        self._x = x
        self.frame_period = float(frame_period)
        self.mask = mask

    @property
    def n_frames(self) -> int:
        return self._x.shape[0]

    @property
    def n_pixels(self) -> int:
        return self._x.shape[1]

    @property
    def intensities(self) -> np.ndarray:
        return self._x.copy()


def apply_mask(frames: FrameSeries, mask: PixelMask) -> FrameSeries:
    """xpcs::apply_mask (model.cpp:42-59): the mask's columns, in mask order."""
    if frames.mask is not None:
        raise MaskError("series is already masked")
    if mask.full_pixels != frames.n_pixels:
        raise MaskError(f"mask covers {mask.full_pixels} pixels but frames have "
                        f"{frames.n_pixels}")
    return FrameSeries(frames._x[:, mask.indices], frames.frame_period, mask)


# ---------------------------------------------------------------- encoder
class EncoderMode(enum.IntEnum):
    OFFLINE = 0
    ONLINE_RELATED = 1
    ONLINE_UNRELATED = 2


class EncodingMatrix:
    """xpcs::EncodingMatrix (model.hpp:53-67): M x K orthonormal V, the
    descending spectrum it came from, and the mode."""

    def __init__(self, v, spectrum, mode: EncoderMode):
        v = np.ascontiguousarray(v, dtype=np.float64)
        spectrum = np.asarray(spectrum, dtype=np.float64)
        if spectrum.size < v.shape[1]:
            raise ContractError("encoder spectrum shorter than column count")
        bad = np.nonzero(spectrum[:-1] < spectrum[1:])[0]
        if bad.size:
            raise ContractError(f"encoder spectrum not descending at index {bad[0]}")
        self._v = v
        self._spectrum = spectrum.copy()
        self.mode = EncoderMode(mode)

    @property
    def k(self) -> int:
        return self._v.shape[1]

    @property
    def n_pixels(self) -> int:
        return self._v.shape[0]

    @property
    def v(self) -> np.ndarray:
        return self._v.copy()

    @property
    def spectrum(self) -> np.ndarray:
        return self._spectrum.copy()


def _content_hash_u64(enc: EncodingMatrix) -> int:
    return int(lib.xg_content_hash(enc._v.ctypes.data_as(_abi.PD), enc.n_pixels, enc.k,
                                   int(enc.mode)))


def content_hash(enc: EncodingMatrix) -> str:
    """xpcs::content_hash (model.cpp:116-125): 16 lowercase hex digits."""
    return f"{_content_hash_u64(enc):016x}"


def _encoder_from_rows(x: np.ndarray, mode: EncoderMode, k: int) -> EncodingMatrix:
    import ctypes as C
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, m = x.shape
    u8 = _as_counts(x) if n <= 2048 else None
    # both branches run K9 on the device: counts from their exact int32 Gram,
    # other rows from the reference-order f64 S (xg_build_basis)
    if u8 is not None:
        vs, sig, rank = _one_ring_series(u8).build_basis(k)
        return EncodingMatrix(vs[0], sig[0], mode)
    kk = k if k > 0 else n
    v = np.empty((m, kk), np.float64)
    sig = np.empty(n, np.float64)
    rank = C.c_int64(0)
    rc = lib.xg_build_basis(x.ctypes.data_as(_abi.PD), n, m, k, v.ctypes.data_as(_abi.PD),
                            sig.ctypes.data_as(_abi.PD), C.byref(rank))
    r = int(rank.value)
    if rc == _abi.ERR_RANK:
        raise RankError(f"requested k = {k} exceeds the numerical rank {r} of the training rows",
                        r)
    if rc == _abi.ERR_NORMALIZATION:
        raise NormalizationError(f"frame {r} has zero norm", r)
    if rc in (_abi.ERR_CUDA, _abi.ERR_DEVICE):
        raise DeviceError(f"basis construction needs a CUDA device (status {rc})")
    if rc != _abi.OK:
        raise ContractError(f"basis construction failed with status {rc}")
    if k == 0:
        v = np.ascontiguousarray(v.ravel()[: m * r].reshape(m, r))
    return EncodingMatrix(v, sig[:r], mode)


def build_offline(frames: FrameSeries) -> EncodingMatrix:
    """xpcs::build_offline (encoder.cpp:32-37): full numerical rank."""
    if frames.n_frames < 2:
        raise ContractError("build_offline: need at least 2 frames")
    return _encoder_from_rows(frames._x, EncoderMode.OFFLINE, 0)


def build_online_from_frames(prior: FrameSeries, k: int) -> EncodingMatrix:
    """xpcs::build_online_from_frames (encoder.cpp:53-60)."""
    if k < 1:
        raise ContractError("build_online_from_frames: k must be >= 1")
    if prior.n_frames < 2:
        raise ContractError("build_online_from_frames: need at least 2 frames")
    return _encoder_from_rows(prior._x, EncoderMode.ONLINE_RELATED, k)


def truncate(enc: EncodingMatrix, k: int) -> EncodingMatrix:
    """xpcs::truncate (encoder.cpp:62-72)."""
    if k < 1 or k > enc.k:
        raise ContractError(f"truncate: k = {k} outside [1, {enc.k}]")
    if k == enc.k:
        return enc
    return EncodingMatrix(enc._v[:, :k], enc._spectrum, enc.mode)


# --------------------------------------------------------------- compress
class CompressedSeries:
    """xpcs::CompressedSeries (model.hpp:88-122, model.cpp:139-212):
    append-only coefficient rows bound to an encoder id."""

    def __init__(self, k: int, encoder_id: int):
        if k == 0:
            raise ContractError("compressed series needs k >= 1")
        self._k = int(k)
        self._id = int(encoder_id)
        self._rows: list[np.ndarray] = []
        self._norms: list[float] = []

    def append(self, coefficients, norm: float) -> None:
        c = np.asarray(coefficients, dtype=np.float64).ravel()
        if c.size != self._k:
            raise ShapeError(f"append: row has {c.size} coefficients, store holds k = {self._k}")
        if not (norm > 0.0) or not np.isfinite(norm):
            raise ContractError("append: frame norm must be positive and finite")
        if not np.all(np.isfinite(c)):
            raise ContractError("append: non-finite coefficient")
        sq = 0.0
        for v in c:  # the reference's sequential sum (model.cpp:184-193)
            sq += v * v
        if sq > (1.0 + 1e-10) * (1.0 + 1e-10):
            raise ContractError(f"append: coefficient row norm {np.sqrt(sq):f} exceeds 1 "
                                "(not a projection of a unit row)")
        self._rows.append(c.copy())
        self._norms.append(float(norm))

    @property
    def k(self) -> int:
        return self._k

    @property
    def encoder_id(self) -> int:
        return self._id

    @property
    def n_frames(self) -> int:
        return len(self._norms)

    @property
    def coefficients(self) -> np.ndarray:
        if not self._rows:
            return np.zeros((0, self._k))
        return np.vstack(self._rows)

    @property
    def norms(self) -> np.ndarray:
        return np.asarray(self._norms, dtype=np.float64)


def compress_series(frames: FrameSeries, encoder: EncodingMatrix) -> CompressedSeries:
    """xpcs::compress_series (compress.cpp:48-81) on the GPU."""
    _ctx()
    y, nr = _compress_series(frames._x, encoder._v)
    store = CompressedSeries(encoder.k, _content_hash_u64(encoder))
    store._rows = [row.copy() for row in y]
    store._norms = [float(v) for v in nr]
    return store


def compress_frame(frame, encoder: EncodingMatrix):
    """xpcs::compress_frame (compress.cpp:34-46) -> (coefficients, norm)."""
    _ctx()
    return _compress_frame(frame, encoder._v)


# -------------------------------------------------------------- correlate
class TTCMatrix:
    """xpcs::TTCMatrix (model.hpp:127-138), validated as model.cpp:214-240."""

    def __init__(self, values, lossless: bool):
        g = np.ascontiguousarray(values, dtype=np.float64)
        n = g.shape[0]
        if g.ndim != 2 or g.shape[1] != n:
            raise ShapeError("TTC matrix must be square")
        asym = np.argwhere(np.triu(g != g.T))
        if asym.size:
            i, j = asym[0]
            raise ContractError(f"TTC matrix not symmetric at ({i},{j})")
        oob = np.argwhere(np.triu((g < -1.0 - 1e-10) | (g > 1.0 + 1e-10)))
        if oob.size:
            i, j = oob[0]
            raise ContractError(f"TTC entry out of [-1, 1] bounds at ({i},{j})")
        d = np.diag(g)
        neg = np.nonzero(d < 0.0)[0]
        if neg.size:
            raise ContractError(f"TTC diagonal negative at {neg[0]}")
        if lossless:
            dev = np.nonzero(np.abs(d - 1.0) > 1e-10)[0]
            if dev.size:
                raise ContractError(f"lossless TTC diagonal deviates from 1 at {dev[0]}")
        self._g = g
        self.lossless = bool(lossless)

    @property
    def n(self) -> int:
        return self._g.shape[0]

    @property
    def values(self) -> np.ndarray:
        return self._g.copy()


class G2Curve:
    """xpcs::G2Curve: lags (d * frame_period), values, counts (N - d)."""

    def __init__(self, lags, values, counts):
        self.lags = np.asarray(lags)
        self.values = np.asarray(values)
        self.counts = [int(c) for c in counts]


def ttc_raw(frames: FrameSeries) -> TTCMatrix:
    """xpcs::ttc_raw (correlate.cpp:19-25) on the GPU: counts through the
    exact u8 Gram (within 1e-12), other data bit-exact on the f64 replica."""
    if frames.n_frames < 2:
        raise ContractError("ttc_raw: need at least 2 frames")
    _ctx()
    u8 = _as_counts(frames._x)
    if u8 is not None:
        s = _one_ring_series(u8)
        try:
            s.ttc_raw(strict=True)
        except NormalizationError as e:  # the reference's message (linalg.cpp:446-449)
            raise NormalizationError(f"row_normalize: frame {e.frame_index} has zero norm",
                                     e.frame_index) from None
        return TTCMatrix(s.ttc(0, "f64"), True)
    return TTCMatrix(_ttc_raw(frames._x), True)


def ttc_compressed(store: CompressedSeries) -> TTCMatrix:
    """xpcs::ttc_compressed (correlate.cpp:27-35) on the GPU, bit-exact."""
    if store.n_frames < 2:
        raise ContractError("ttc_compressed: need at least 2 frames")
    _ctx()
    g, lossless = _ttc_compressed(store.coefficients)
    return TTCMatrix(g, lossless)


def ttc_extend(ttc: TTCMatrix, store: CompressedSeries, new_row) -> TTCMatrix:
    """xpcs::ttc_extend (correlate.cpp:37-65): one new row/column on the GPU."""
    _ctx()
    y = store.coefficients if store.n_frames else np.zeros((0, store.k))
    g, lossless = _ttc_extend(ttc._g, y, new_row)
    return TTCMatrix(g, lossless)


def g2_from_ttc(ttc: TTCMatrix, frame_period: float = 1.0) -> G2Curve:
    """xpcs::g2_from_ttc (correlate.cpp:67-85)."""
    _ctx()
    lags, vals, cnt = _g2_from_ttc(ttc._g, frame_period)
    return G2Curve(lags, vals, cnt)


def ttc_rel_error(ttc: TTCMatrix, ttc_approx: TTCMatrix) -> float:
    """xpcs::ttc_rel_error (correlate.cpp:87-108)."""
    _ctx()
    return _ttc_rel_error(ttc._g, ttc_approx._g)
