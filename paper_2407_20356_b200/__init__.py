"""B200-native XPCS two-time correlation (arXiv 2407.20356 hot path).

Python host mirror of the reference's operator API (namespace ``xpcs``,
/root/reference/proj/include/xpcsvd/*.hpp) over the C ABI of
``libxpcs_b200.so``.  Every numeric result is computed by the sm_100a
kernels of that library; this module only marshals buffers and maps status
codes onto the reference's exception hierarchy (errors.hpp:11-74).
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _abi
from ._abi import lib


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """xpcs::Error"""


class ShapeError(Error):
    """xpcs::ShapeError"""


class ContractError(Error):
    """xpcs::ContractError"""


class MaskError(Error):
    """xpcs::MaskError"""


class NormalizationError(Error):
    """xpcs::NormalizationError; ``frame_index`` (+ ``ring`` for batched rings)."""

    def __init__(self, msg: str, frame_index: int, ring: int = -1):
        super().__init__(msg)
        self.frame_index = frame_index
        self.ring = ring


class RankError(Error):
    def __init__(self, msg: str, achievable_rank: int):
        super().__init__(msg)
        self.achievable_rank = achievable_rank


class BindingError(Error):
    pass


class FormatError(Error):
    """xpcs::FormatError; ``offset`` = byte offset of the first inconsistency."""

    def __init__(self, msg: str, offset: int = -1):
        super().__init__(msg)
        self.offset = offset


class DeviceError(Error):
    """CUDA failure, missing sm_100 device, or a kernel self-check failure."""


_ERRS = {
    _abi.ERR_SHAPE: ShapeError,
    _abi.ERR_CONTRACT: ContractError,
    _abi.ERR_MASK: MaskError,
    _abi.ERR_BINDING: BindingError,
    _abi.ERR_FORMAT: FormatError,
}


def _check(ctx_handle, rc: int) -> None:
    if rc == _abi.OK:
        return
    msg = lib.xg_last_error(ctx_handle).decode() if ctx_handle else f"status {rc}"
    if rc == _abi.ERR_NORMALIZATION:
        ring = C.c_int32(-1)
        frame = lib.xg_last_error_payload(ctx_handle, C.byref(ring))
        raise NormalizationError(msg, int(frame), int(ring.value))
    if rc == _abi.ERR_RANK:
        raise RankError(msg, int(lib.xg_last_error_payload(ctx_handle, None)))
    if rc == _abi.ERR_FORMAT:
        raise FormatError(msg, int(lib.xg_last_error_payload(ctx_handle, None)))
    raise _ERRS.get(rc, DeviceError)(msg or f"status {rc}")


def _as_counts_u8(frames) -> np.ndarray:
    """Photon counts as contiguous u8.  Wider integer or float input is
    accepted when every value is an integer in [0, 255]; anything else raises
    ContractError instead of wrapping (the u8 path has no counts > 255)."""
    a = np.asarray(frames)
    if a.dtype == np.uint8:
        return np.ascontiguousarray(a)
    if a.size:
        if a.dtype.kind == "f" and not np.all(np.isfinite(a)):
            raise ContractError("frames contain non-finite values")
        lo, hi = a.min(), a.max()
        if lo < 0 or hi > 255:
            raise ContractError(f"frame counts must lie in [0, 255] (got [{lo}, {hi}])")
        if a.dtype.kind == "f" and not np.array_equal(a, np.rint(a)):
            raise ContractError("frames must hold integer photon counts")
    return np.ascontiguousarray(a, dtype=np.uint8)


def _tensor_frames(frames, ctx: "Context", pixels: int, n: int | None, what: str,
                   host_ok: bool = True, device_ok: bool = True):
    """Validate a torch tensor of u8 frames handed to the library by pointer:
    uint8, contiguous (a strided view would feed the wrong pixels), exactly
    n x pixels elements, on the context's device (or in host memory).
    Returns (n, on_device)."""
    if str(getattr(frames, "dtype", "")) != "torch.uint8":
        raise ContractError(f"{what}: frames tensor must be uint8 photon counts")
    if not frames.is_contiguous():
        raise ContractError(f"{what}: frames tensor must be contiguous")
    on_dev = bool(getattr(frames, "is_cuda", False))
    if on_dev and not device_ok:
        raise ContractError(f"{what} takes host frames; use load() for device ones")
    if not on_dev and not host_ok:
        raise ContractError(f"{what} takes device frames")
    if on_dev and frames.device.index != ctx.device:
        raise ContractError(f"{what}: frames are on cuda:{frames.device.index}, the context "
                            f"on cuda:{ctx.device}")
    if n is None:
        n = int(frames.shape[0]) if frames.dim() > 1 else 1
    if n < 1 or frames.numel() != n * pixels:
        raise ShapeError(f"{what}: frames tensor has {frames.numel()} elements, expected "
                         f"{n} x {pixels}")
    return n, on_dev


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- formats
def _io_check(rc: int) -> None:
    """Errors of the host format helpers (xg_io_*)."""
    if rc == _abi.OK:
        return
    msg = lib.xg_io_last_error().decode()
    payload = int(lib.xg_io_last_payload())
    if rc == _abi.ERR_FORMAT:
        raise FormatError(msg, payload)
    if rc == _abi.ERR_NORMALIZATION:
        raise NormalizationError(msg, payload)
    raise _ERRS.get(rc, DeviceError)(msg or f"status {rc}")


def write_xfsr(path, frames, frame_period: float = 1.0) -> None:
    """XFSR frames file with dtype 3 = u8 photon counts (new; the reference's
    io.cpp:150-184 writes u16/f32/f64)."""
    a = _as_counts_u8(frames)
    if a.ndim != 2:
        raise ShapeError("frames must be N x M")
    _io_check(lib.xg_io_write_xfsr_u8(str(path).encode(), _ptr(a), a.shape[0], a.shape[1],
                                      float(frame_period)))


def read_xfsr(path):
    """Any XFSR frames file (dtype u16/f32/f64 as the reference, or u8) as
    u8 photon counts + frame period; read_frames' checks (io.cpp:187-225)."""
    n, m, per = C.c_int64(0), C.c_int64(0), C.c_double(0.0)
    p = str(path).encode()
    _io_check(lib.xg_io_read_xfsr_u8(p, None, 0, C.byref(n), C.byref(m), C.byref(per)))
    out = np.empty((n.value, m.value), np.uint8)
    _io_check(lib.xg_io_read_xfsr_u8(p, _ptr(out), out.size, C.byref(n), C.byref(m),
                                     C.byref(per)))
    return out, per.value


def content_hash(v, mode: int = 1) -> int:
    """content_hash_u64 (model.cpp:99-114) of a basis V (m x k) and mode: the
    encoder id an XCMP store is bound to."""
    vv = np.ascontiguousarray(v, dtype=np.float64)
    return int(lib.xg_content_hash(vv.ctypes.data_as(_abi.PD), vv.shape[0], vv.shape[1], int(mode)))


def write_xenc(path, v, spectrum, mode: int = 1) -> None:
    """XENC encoder file of one ring's basis (io.cpp:273-285): V (m x k, mask
    order), its spectrum, mode 0 offline / 1 online-related / 2 unrelated."""
    vv = np.ascontiguousarray(v, dtype=np.float64)
    sp = np.ascontiguousarray(spectrum, dtype=np.float64)
    if vv.ndim != 2 or sp.ndim != 1 or sp.size < vv.shape[1]:
        raise ShapeError("V must be m x k with at least k spectrum values")
    _io_check(lib.xg_io_write_xenc(str(path).encode(), int(mode), vv.shape[0], vv.shape[1],
                                   sp.ctypes.data_as(_abi.PD), sp.size, vv.ctypes.data_as(_abi.PD)))


def read_xenc(path):
    """An XENC encoder file -> (V m x k, spectrum, mode) (io.cpp:287-321)."""
    mode, m, k, sl = C.c_int32(0), C.c_int64(0), C.c_int64(0), C.c_int64(0)
    p = str(path).encode()
    _io_check(lib.xg_io_read_xenc(p, C.byref(mode), C.byref(m), C.byref(k), C.byref(sl), None, None))
    v = np.empty((m.value, k.value))
    sp = np.empty(sl.value)
    _io_check(lib.xg_io_read_xenc(p, C.byref(mode), C.byref(m), C.byref(k), C.byref(sl),
                                  sp.ctypes.data_as(_abi.PD), v.ctypes.data_as(_abi.PD)))
    return v, sp, int(mode.value)


def read_xttc(path) -> np.ndarray:
    """An XTTC tile file (FrameSeries.write_ttc) as the full symmetric matrix."""
    raw = open(path, "rb").read()
    if len(raw) < 20 or raw[:4] != b"XTTC":
        raise FormatError("bad magic, expected \"XTTC\"", 0)
    ver, code = np.frombuffer(raw[4:12], "<u4")
    n = int(np.frombuffer(raw[12:20], "<u8")[0])
    if ver != 1 or code > 2:
        raise FormatError(f"unsupported XTTC version {ver} / dtype {code}", 4)
    dt = {0: "<f8", 1: "<f4", 2: "<i4"}[int(code)]
    tri = np.frombuffer(raw[20:], dt)
    if tri.size != n * (n + 1) // 2:
        raise FormatError("XTTC payload length does not match n", 20)
    out = np.zeros((n, n), tri.dtype)
    iu = np.triu_indices(n)
    out[iu] = tri
    out.T[iu] = tri
    return out


def write_xcmp(path, coefficients, norms, encoder_hash: int, append: bool = False) -> None:
    """XCMP compressed store from host rows (io.cpp:319-441; append like
    CompressedFileAppender)."""
    y = np.ascontiguousarray(coefficients, dtype=np.float64)
    nr = np.ascontiguousarray(norms, dtype=np.float64)
    if y.ndim != 2 or nr.shape != (y.shape[0],):
        raise ShapeError("coefficients must be N x k with N norms")
    _io_check(lib.xg_io_write_xcmp(str(path).encode(), y.shape[1], int(encoder_hash), y.shape[0],
                                   nr.ctypes.data_as(_abi.PD), y.ctypes.data_as(_abi.PD),
                                   1 if append else 0))


# ---------------------------------------------------------------- context
class Context:
    """One device + one CUDA stream (xg_ctx).  ``stream`` may be a raw
    cudaStream_t handle (int) such as ``torch.cuda.current_stream().cuda_stream``."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        rc = lib.xg_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h))
        if rc != _abi.OK:
            raise DeviceError(f"xg_ctx_create(device={device}) failed with status {rc} "
                              "(an sm_100 B200 GPU is required; there is no CPU path)")
        self.h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            lib.xg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def synchronize(self) -> None:
        _check(self.h, lib.xg_synchronize(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(lib.xg_kernel_launches(self.h))


# ----------------------------------------------------------------- layout
class RingLayout:
    """A set of q-ring ``PixelMask``s (model.hpp:16-24) over a detector of
    ``full_pixels`` pixels.  ``masks[r]`` are strictly ascending indices."""

    def __init__(self, ctx: Context, full_pixels: int, masks: Sequence[np.ndarray],
                 shape: tuple | None = None):
        """``shape`` = (height, width) of a row-major detector (full_pixels =
        height * width): on a detector wider than 512 pixels the ingest then
        reads 2D blocks (xg_layout_create_2d); results are identical."""
        self.ctx = ctx
        self.full_pixels = int(full_pixels)
        if shape is not None and int(shape[0]) * int(shape[1]) != self.full_pixels:
            raise ShapeError(f"shape {tuple(shape)} does not hold {self.full_pixels} pixels")
        self.shape = tuple(int(v) for v in shape) if shape is not None else None
        self.masks = [np.ascontiguousarray(m, dtype=np.int64) for m in masks]
        offs = np.zeros(len(self.masks) + 1, np.int64)
        offs[1:] = np.cumsum([m.size for m in self.masks])
        idx = np.concatenate(self.masks) if self.masks else np.zeros(0, np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        h = C.c_void_p()
        if self.shape is not None:
            _check(ctx.h, lib.xg_layout_create_2d(ctx.h, self.shape[0], self.shape[1],
                                                  len(self.masks), offs.ctypes.data_as(_abi.PI64),
                                                  idx.ctypes.data_as(_abi.PI64), C.byref(h)))
        else:
            _check(ctx.h, lib.xg_layout_create(ctx.h, self.full_pixels, len(self.masks),
                                               offs.ctypes.data_as(_abi.PI64),
                                               idx.ctypes.data_as(_abi.PI64), C.byref(h)))
        self.h = h

    @classmethod
    def from_ring_map(cls, ctx: Context, ring_of_pixel: np.ndarray, n_rings: int,
                      shape: tuple | None = None):
        """Masks from a per-pixel ring index (-1 = no ring); a 2D map (or
        ``shape``) gives the detector geometry to the ingest."""
        rp = np.asarray(ring_of_pixel)
        if shape is None and rp.ndim == 2:
            shape = rp.shape
        rp = rp.ravel()
        masks = [np.nonzero(rp == r)[0] for r in range(n_rings)]
        return cls(ctx, rp.size, masks, shape=shape)

    @property
    def n_rings(self) -> int:
        return len(self.masks)

    def ring_pixels(self, r: int) -> int:
        return int(lib.xg_layout_ring_pixels(self.h, r))

    def __del__(self):
        if getattr(self, "h", None):
            lib.xg_layout_destroy(self.h)
            self.h = None


# ------------------------------------------------------------------ basis
def build_online_from_frames(prior: np.ndarray, k: int) -> np.ndarray:
    """V (m x k) from a prior series (encoder.cpp:53-60); k = 0 -> full
    numerical rank (build_offline, encoder.cpp:32-37).  Runs on the current
    CUDA device (K9 over f64 rows, xg_build_basis); at most 2048 rows."""
    x = np.ascontiguousarray(prior, dtype=np.float64)
    n, m = x.shape
    if n < 2:
        raise ContractError("build_online_from_frames: need at least 2 frames")
    if k < 0:
        raise ContractError("build_online_from_frames: k must be >= 1")
    rank = C.c_int64(0)
    kk = k if k > 0 else n
    v = np.empty((m, kk), np.float64)
    sig = np.empty(n, np.float64)
    rc = lib.xg_build_basis(x.ctypes.data_as(_abi.PD), n, m, k, v.ctypes.data_as(_abi.PD),
                            sig.ctypes.data_as(_abi.PD), C.byref(rank))
    if rc == _abi.ERR_RANK:
        raise RankError(f"requested k = {k} exceeds the numerical rank {rank.value}",
                        int(rank.value))
    if rc == _abi.ERR_NORMALIZATION:
        raise NormalizationError(f"frame {rank.value} has zero norm", int(rank.value))
    if rc in (_abi.ERR_CUDA, _abi.ERR_DEVICE):
        raise DeviceError(f"build_basis needs a CUDA device (status {rc})")
    if rc != _abi.OK:
        raise ContractError(f"build_basis failed with status {rc} (n <= 2048 rows, m >= 1)")
    if k == 0:
        v = np.ascontiguousarray(v.ravel()[: m * rank.value].reshape(m, rank.value))
    return v


def build_ring_bases(prior_per_ring: Sequence[np.ndarray], k: int, threads: int = 0):
    """build_online_from_frames for every ring in one device pass (K9)."""
    xs = [np.ascontiguousarray(x, dtype=np.float64) for x in prior_per_ring]
    n = xs[0].shape[0]
    vs = [np.empty((x.shape[1], k), np.float64) for x in xs]
    q = len(xs)
    xp = (_abi.PD * q)(*[x.ctypes.data_as(_abi.PD) for x in xs])
    vp = (_abi.PD * q)(*[v.ctypes.data_as(_abi.PD) for v in vs])
    ms = np.array([x.shape[1] for x in xs], np.int64)
    ranks = np.zeros(q, np.int64)
    rc = lib.xg_build_basis_batch(q, xp, n, ms.ctypes.data_as(_abi.PI64), k, vp, threads,
                                  ranks.ctypes.data_as(_abi.PI64))
    if rc == _abi.ERR_RANK:
        raise RankError(f"k = {k} exceeds a ring's numerical rank", int(ranks.min()))
    if rc in (_abi.ERR_CUDA, _abi.ERR_DEVICE):
        raise DeviceError(f"build_ring_bases needs a CUDA device (status {rc})")
    if rc != _abi.OK:
        raise ContractError(f"build_ring_bases failed with status {rc}")
    return vs


class Basis:
    """Per-ring rank-k encoding matrices (EncodingMatrix, model.hpp:53-67) on
    the device, as `digits` signed-int8 planes per column (3: ~3e-8 of
    max|V|; 2: ~8e-6)."""

    def __init__(self, layout: RingLayout, k: int, digits: int = 3):
        self.layout = layout
        self.ctx = layout.ctx
        self.k = int(k)
        h = C.c_void_p()
        _check(self.ctx.h, lib.xg_basis_create(self.ctx.h, layout.h, self.k, digits, C.byref(h)))
        self.h = h

    def set_ring(self, ring: int, v: np.ndarray) -> "Basis":
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.shape != (self.layout.ring_pixels(ring), self.k):
            raise ShapeError(f"basis of ring {ring} must be "
                             f"{self.layout.ring_pixels(ring)} x {self.k}, got {v.shape}")
        _check(self.ctx.h, lib.xg_basis_set_ring(self.h, ring, v.ctypes.data_as(_abi.PD)))
        return self

    def __del__(self):
        if getattr(self, "h", None):
            lib.xg_basis_destroy(self.h)
            self.h = None


class _DeviceArray:
    """__cuda_array_interface__ view of a library-owned device buffer (keeps
    its owner alive)."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}
        self._owner = owner


# ----------------------------------------------------------------- series
class FrameSeries:
    """Device-resident photon-count frames of one detector, correlated per
    q-ring (the reference's ``FrameSeries`` + ``apply_mask`` per ring,
    model.hpp:26-40).  Frames are u8 counts in raster order."""

    def __init__(self, layout: RingLayout, max_frames: int, frame_period: float = 1.0,
                 x_frames: int | None = None):
        """``x_frames`` < max_frames: the frame buffer holds only that many
        frames; feed the series with compress_chunk() (compressed path only)
        -- for series larger than HBM."""
        if not (frame_period > 0.0):
            raise ContractError("frame_period must be positive and finite")
        self.layout = layout
        self.ctx = layout.ctx
        self.max_frames = int(max_frames)
        self.frame_period = float(frame_period)
        h = C.c_void_p()
        _check(self.ctx.h, lib.xg_series_create2(self.ctx.h, layout.h, self.max_frames,
                                                 int(x_frames or max_frames), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib.xg_series_destroy(self.h)
            self.h = None

    @property
    def n_frames(self) -> int:
        return int(lib.xg_series_frames(self.h))

    def load(self, frames, n_frames: int | None = None) -> "FrameSeries":
        """Ingest ``frames`` (n x full_pixels u8): a numpy array (host, copied
        H2D) or any object exposing ``data_ptr()`` (a CUDA torch tensor)."""
        if hasattr(frames, "data_ptr"):  # torch tensor: CUDA (device) or pinned host
            n, on_dev = _tensor_frames(frames, self.ctx, self.layout.full_pixels, n_frames, "load")
            _check(self.ctx.h, lib.xg_series_load_frames(self.h, C.c_void_p(frames.data_ptr()),
                                                         n, 1 if on_dev else 0))
            # a host tensor's copy is asynchronous: keep it alive until replaced
            self._keep = None if on_dev else frames
            return self
        a = _as_counts_u8(frames)
        if a.ndim != 2 or a.shape[1] != self.layout.full_pixels:
            raise ShapeError(f"frames must be n x {self.layout.full_pixels}, got {a.shape}")
        _check(self.ctx.h, lib.xg_series_load_frames(self.h, _ptr(a), a.shape[0], 0))
        self._keep = a
        return self

    def load_events(self, frame_off, pix, val) -> "FrameSeries":
        """Ingest photon-event frames: frame f's events are pix[frame_off[f]:
        frame_off[f+1]] (raster pixel indices, unique within a frame) with
        counts val[...]; every other pixel is 0.  The same series as
        ``load`` of the dense frames (xg_series_load_events).  numpy arrays
        (host: int64 / int32 / uint8, copied H2D) or torch tensors of those
        dtypes, all on the context's device or all in (pinned) host memory."""
        if hasattr(frame_off, "data_ptr"):
            ts = (frame_off, pix, val)
            for t_, dt in zip(ts, ("torch.int64", "torch.int32", "torch.uint8")):
                if str(t_.dtype) != dt or not t_.is_contiguous() or t_.dim() != 1:
                    raise ShapeError(f"load_events: expected contiguous 1-D {dt} tensors")
            on_dev = frame_off.is_cuda
            if any(t_.is_cuda != on_dev for t_ in ts):
                raise ShapeError("load_events: frame_off, pix and val must share a device")
            if on_dev and frame_off.device.index != self.ctx.device:
                raise ShapeError("load_events: tensors on another device than the context")
            n = frame_off.numel() - 1
            if pix.numel() != val.numel():
                raise ShapeError("load_events: pix and val differ in length")
            _check(self.ctx.h, lib.xg_series_load_events(
                self.h, C.c_void_p(frame_off.data_ptr()), C.c_void_p(pix.data_ptr()),
                C.c_void_p(val.data_ptr()), n, 1 if on_dev else 0))
            self._keep = None if on_dev else ts
            return self
        off = np.ascontiguousarray(frame_off, dtype=np.int64)
        px = np.ascontiguousarray(pix, dtype=np.int32)
        vv = np.ascontiguousarray(val, dtype=np.uint8)
        if off.ndim != 1 or off.size < 2 or px.shape != vv.shape or off[-1] != px.size:
            raise ShapeError("load_events: frame_off must hold n + 1 offsets ending at len(pix)")
        _check(self.ctx.h, lib.xg_series_load_events(self.h, _ptr(off), _ptr(px), _ptr(vv),
                                                      off.size - 1, 0))
        self._keep = (off, px, vv)
        return self

    def ttc_raw_events_host(self, frame_off, pix, val, strict: bool = False, g2: bool = True,
                            store: bool = True) -> "FrameSeries":
        """load_events() + ttc_raw() for event lists in HOST memory, the PCIe
        transfer of each chunk of frames overlapped with the scatter and the
        Gram tiles it completes (xg_series_ttc_raw_events_host).  Pinned torch
        tensors (int64 / int32 / uint8) for full overlap, or numpy arrays."""
        flags = ((_abi.STRICT if strict else 0) | (0 if g2 else _abi.NO_G2)
                 | (0 if store else _abi.NO_STORE))
        if hasattr(frame_off, "data_ptr"):
            ts = (frame_off, pix, val)
            for t_, dt in zip(ts, ("torch.int64", "torch.int32", "torch.uint8")):
                if (str(t_.dtype) != dt or not t_.is_contiguous() or t_.dim() != 1
                        or t_.is_cuda):
                    raise ShapeError(f"ttc_raw_events_host: expected contiguous 1-D host {dt}")
            if pix.numel() != val.numel():
                raise ShapeError("ttc_raw_events_host: pix and val differ in length")
            ptrs = [C.c_void_p(t_.data_ptr()) for t_ in ts]
            n = frame_off.numel() - 1
            keep = ts
        else:
            off = np.ascontiguousarray(frame_off, dtype=np.int64)
            px = np.ascontiguousarray(pix, dtype=np.int32)
            vv = np.ascontiguousarray(val, dtype=np.uint8)
            if off.ndim != 1 or off.size < 2 or px.shape != vv.shape or off[-1] != px.size:
                raise ShapeError("ttc_raw_events_host: frame_off must hold n + 1 offsets ending "
                                 "at len(pix)")
            ptrs = [_ptr(off), _ptr(px), _ptr(vv)]
            n = off.size - 1
            keep = (off, px, vv)
        _check(self.ctx.h, lib.xg_series_ttc_raw_events_host(self.h, *ptrs, n, flags))
        self._keep = keep
        return self

    def ttc_raw(self, strict: bool = False, g2: bool = True, store: bool = True) -> "FrameSeries":
        """Raw TTC of every ring (ttc_raw, correlate.cpp:19-25).  store=False
        keeps only g2 (the TTC tiles never leave the chip)."""
        flags = ((_abi.STRICT if strict else 0) | (0 if g2 else _abi.NO_G2)
                 | (0 if store else _abi.NO_STORE))
        _check(self.ctx.h, lib.xg_ttc_raw(self.h, flags))
        return self

    def ttc_raw_host(self, frames, strict: bool = False, g2: bool = True,
                     store: bool = True) -> "FrameSeries":
        """load() + ttc_raw() for frames in HOST memory, with the PCIe transfer
        overlapped with ingest and the Gram (xg_series_ttc_raw_host).  Pass a
        pinned torch tensor (``pin_memory=True``) for full overlap; numpy
        arrays work too.  Same results as the two calls."""
        flags = ((_abi.STRICT if strict else 0) | (0 if g2 else _abi.NO_G2)
                 | (0 if store else _abi.NO_STORE))
        if hasattr(frames, "data_ptr"):
            n, _ = _tensor_frames(frames, self.ctx, self.layout.full_pixels, None, "ttc_raw_host",
                                  device_ok=False)
            _check(self.ctx.h, lib.xg_series_ttc_raw_host(self.h, C.c_void_p(frames.data_ptr()),
                                                          n, flags))
            self._keep = frames
            return self
        a = _as_counts_u8(frames)
        if a.ndim != 2 or a.shape[1] != self.layout.full_pixels:
            raise ShapeError(f"frames must be n x {self.layout.full_pixels}, got {a.shape}")
        _check(self.ctx.h, lib.xg_series_ttc_raw_host(self.h, _ptr(a), a.shape[0], flags))
        self._keep = a
        return self

    # ---------------------------------------------- split rings (multi-GPU)
    @property
    def partial_elems(self) -> int:
        """int32 values of one ring's packed Gram partial (upper pair tiles)."""
        return int(lib.xg_series_partial_elems(self.h))

    def export_partial(self, ring: int, gram=None, norm2=None):
        """This process's share of a split ring: (packed int32 Gram tiles,
        int64 |x_t|^2).  Pass CUDA torch tensors (int32 [partial_elems], int64
        [n_frames]) to export on the device; by default numpy host arrays."""
        on_dev = gram is not None and getattr(gram, "is_cuda", False)
        if gram is None:
            gram = np.empty(self.partial_elems, np.int32)
            norm2 = np.empty(self.n_frames, np.int64)
        self._check_partial(gram, norm2, on_dev)
        gp = gram.data_ptr() if on_dev else gram.ctypes.data
        npp = norm2.data_ptr() if on_dev else norm2.ctypes.data
        _check(self.ctx.h, lib.xg_series_export_partial(self.h, ring, C.c_void_p(gp),
                                                        C.c_void_p(npp), 1 if on_dev else 0))
        return gram, norm2

    def import_partial(self, ring: int, gram, norm2, strict: bool = False,
                       g2: bool = True) -> "FrameSeries":
        """Install the summed partials of a split ring (numpy or CUDA tensors)."""
        on_dev = getattr(gram, "is_cuda", False)
        if not on_dev:
            gram = np.ascontiguousarray(gram, dtype=np.int32)
            norm2 = np.ascontiguousarray(norm2, dtype=np.int64)
        self._check_partial(gram, norm2, on_dev)
        gp = gram.data_ptr() if on_dev else gram.ctypes.data
        npp = norm2.data_ptr() if on_dev else norm2.ctypes.data
        flags = (_abi.STRICT if strict else 0) | (0 if g2 else _abi.NO_G2)
        _check(self.ctx.h, lib.xg_series_import_partial(self.h, ring, C.c_void_p(gp),
                                                        C.c_void_p(npp), 1 if on_dev else 0,
                                                        flags))
        return self

    def _check_partial(self, gram, norm2, on_dev: bool) -> None:
        if on_dev:
            ok = (str(gram.dtype) == "torch.int32" and str(norm2.dtype) == "torch.int64"
                  and gram.is_contiguous() and norm2.is_contiguous()
                  and getattr(norm2, "is_cuda", False)
                  and gram.numel() == self.partial_elems and norm2.numel() == self.n_frames)
        else:
            ok = (isinstance(gram, np.ndarray) and isinstance(norm2, np.ndarray)
                  and gram.dtype == np.int32 and norm2.dtype == np.int64
                  and gram.flags.c_contiguous and norm2.flags.c_contiguous
                  and gram.size == self.partial_elems and norm2.size == self.n_frames)
        if not ok:
            raise ShapeError(f"split-ring partial must be int32[{self.partial_elems}] + "
                             f"int64[{self.n_frames}], contiguous, both host or both device")

    def compute_g2(self) -> "FrameSeries":
        """g2 of every ring from the current raw TTC (after ttc_raw(g2=False))."""
        _check(self.ctx.h, lib.xg_series_g2(self.h))
        return self

    def ttc(self, ring: int, dtype: str = "f64", out=None):
        """Full symmetric n x n TTC of one ring: "f64" C, "f32", or the exact
        int32 "gram".  ``out``: an optional preallocated n x n destination (a
        numpy array, or a torch tensor -- pinned host memory reads back at
        PCIe speed, a CUDA tensor is filled on the device)."""
        code = {"f64": _abi.F64, "f32": _abi.F32, "gram": _abi.I32_GRAM}[dtype]
        n = self.n_frames
        npd = {"f64": np.float64, "f32": np.float32, "gram": np.int32}[dtype]
        if out is None:
            out = np.empty((n, n), npd)
        if hasattr(out, "data_ptr"):
            tdt = {"f64": "torch.float64", "f32": "torch.float32", "gram": "torch.int32"}[dtype]
            if str(out.dtype) != tdt or not out.is_contiguous() or out.numel() != n * n:
                raise ShapeError(f"ttc out must be a contiguous {n} x {n} {tdt} tensor")
            on_dev = 1 if getattr(out, "is_cuda", False) else 0
            _check(self.ctx.h, lib.xg_series_get_ttc(self.h, ring, code, C.c_void_p(out.data_ptr()),
                                                     n, on_dev))
            return out
        if out.dtype != npd or out.shape != (n, n) or not out.flags.c_contiguous:
            raise ShapeError(f"ttc out must be a contiguous {n} x {n} {np.dtype(npd)} array")
        _check(self.ctx.h, lib.xg_series_get_ttc(self.h, ring, code, _ptr(out), n, 0))
        return out

    def g2(self, ring: int):
        """(lags [s], values, counts) like G2Curve (model.hpp:142-146)."""
        n = self.n_frames
        vals = np.empty(n, np.float64)
        cnt = np.empty(n, np.int64)
        _check(self.ctx.h, lib.xg_series_get_g2(self.h, ring, vals.ctypes.data_as(_abi.PD),
                                                cnt.ctypes.data_as(_abi.PI64)))
        lags = np.arange(n, dtype=np.float64) * self.frame_period
        return lags, vals, cnt

    def g2_all(self):
        """(lags, values [ring][n], counts [ring][n]) of every ring, one transfer."""
        n, q = self.n_frames, self.layout.n_rings
        vals = np.empty((q, n), np.float64)
        cnt = np.empty((q, n), np.int64)
        _check(self.ctx.h, lib.xg_series_get_g2_all(self.h, vals.ctypes.data_as(_abi.PD),
                                                    cnt.ctypes.data_as(_abi.PI64)))
        return np.arange(n, dtype=np.float64) * self.frame_period, vals, cnt

    def g2_device(self, compressed: bool = False):
        """Every ring's g2 values and pair counts as CUDA torch tensors
        [rings, ld] viewing the library's device buffers (no copy; valid
        until the series is recomputed; columns >= n_frames are padding)."""
        import torch

        v, c, ld = C.c_void_p(), C.c_void_p(), C.c_int64(0)
        _check(self.ctx.h, lib.xg_series_g2_device(self.h, 1 if compressed else 0, C.byref(v),
                                                   C.byref(c), C.byref(ld)))
        shape = (self.layout.n_rings, int(ld.value))
        return (torch.as_tensor(_DeviceArray(v.value, shape, "<f8", self), device="cuda"),
                torch.as_tensor(_DeviceArray(c.value, shape, "<i8", self), device="cuda"))

    def cg2_all(self):
        """(lags, values [ring][n], counts [ring][n]) of the compressed g2."""
        n, q = self.n_frames, self.layout.n_rings
        vals = np.empty((q, n), np.float64)
        cnt = np.empty((q, n), np.int64)
        for r in range(q):
            _, vals[r], cnt[r] = self.cg2(r)
        return np.arange(n, dtype=np.float64) * self.frame_period, vals, cnt

    # ------------------------------------------------------ compressed path
    def compress(self, basis: "Basis", strict: bool = False) -> "FrameSeries":
        """Rank-k projection of every ring (compress_series, compress.cpp:48-81)."""
        _check(self.ctx.h, lib.xg_compress(self.h, basis.h, _abi.STRICT if strict else 0))
        self.k = basis.k
        return self

    def rel_error(self) -> np.ndarray:
        """Per-ring ttc_rel_error(raw C, compressed C~) (correlate.cpp:87-108):
        the homomorphic path's deviation report, computed on the device."""
        out = np.empty(self.layout.n_rings, np.float64)
        _check(self.ctx.h, lib.xg_series_rel_error(self.h, out.ctypes.data_as(_abi.PD)))
        return out

    def write_xcmp(self, ring: int, path, encoder_hash: int, append: bool = False) -> None:
        """This ring's compressed rows as an XCMP store (io.cpp:319-441)."""
        _check(self.ctx.h, lib.xg_series_write_xcmp(self.h, ring, str(path).encode(),
                                                     int(encoder_hash), 1 if append else 0))

    def write_ttc(self, ring: int, path, dtype: str = "f64", compressed: bool = False) -> None:
        """Stream one ring's stored TTC to an XTTC tile file (upper triangle,
        row after row): raw as "f64" C or exact "gram" (int32); compressed as
        "f32" C~.  read_xttc() loads it back."""
        code = {"f64": 0, "f32": 1, "gram": 2}[dtype]
        _check(self.ctx.h, lib.xg_series_write_ttc(self.h, ring, 1 if compressed else 0, code,
                                                    str(path).encode()))

    def load_xfsr(self, path) -> "FrameSeries":
        """Load an XFSR frames file (u16/f32/f64 as the reference, or u8) of
        photon counts; the series takes the file's frame period."""
        per = C.c_double(0.0)
        _check(self.ctx.h, lib.xg_series_load_xfsr(self.h, str(path).encode(), C.byref(per)))
        self.frame_period = per.value
        return self

    def ttc_background(self, exclusion: int = 0, compressed: bool = False) -> np.ndarray:
        """Per-ring ttc_background (analysis.cpp:202-235) of the stored raw or
        compressed TTC, on the device: sigma of the entries with lag > exclusion."""
        out = np.empty(self.layout.n_rings, np.float64)
        _check(self.ctx.h, lib.xg_series_ttc_background(self.h, 1 if compressed else 0,
                                                         int(exclusion), out.ctypes.data_as(_abi.PD)))
        return out

    def fit_kww(self, min_lag: float, max_lag: float, compressed: bool = False):
        """Per-ring fit_kww (analysis.cpp:77-172) of the device g2 curves over
        lags [min_lag, max_lag] (lags in frame periods * frame_period).
        Returns (fits [rings x 4]: B, C, t0, residual rms; status [rings]:
        0 ok, 1 FitDegenerateError, 2 FitError (fit = last accepted iterate),
        3 ContractError (window too small / non-finite))."""
        q = self.layout.n_rings
        fits = np.zeros((q, 4), np.float64)
        st = np.zeros(q, np.int32)
        _check(self.ctx.h, lib.xg_series_fit_kww(self.h, 1 if compressed else 0,
                                                  float(self.frame_period), float(min_lag),
                                                  float(max_lag), fits.ctypes.data_as(_abi.PD),
                                                  st.ctypes.data_as(C.POINTER(C.c_int32))))
        return fits, st

    def build_basis(self, k: int, basis: "Basis | None" = None):
        """Per-ring encoding basis from this series' frames, built on the
        device (xg_series_build_basis; the reference's build_online_from_frames
        per ring, k = 0 -> build_offline).  Returns (V per ring in mask order,
        spectrum per ring, rank per ring); fills ``basis`` when given."""
        q = self.layout.n_rings
        n = self.n_frames
        rank = np.zeros(q, np.int64)
        sig = np.zeros((q, max(n, 1)), np.float64)
        vs = [np.empty((self.layout.ring_pixels(r), k if k > 0 else n), np.float64)
              for r in range(q)]
        ptrs = (_abi.PD * q)(*[v.ctypes.data_as(_abi.PD) for v in vs])
        _check(self.ctx.h, lib.xg_series_build_basis(
            self.h, int(k), ptrs, sig.ctypes.data_as(_abi.PD), sig.shape[1],
            rank.ctypes.data_as(_abi.PI64), basis.h if basis is not None else None))
        if k == 0:  # full rank: V was written with the ring's own rank as row length
            vs = [np.ascontiguousarray(v.ravel()[: v.shape[0] * int(rank[r])]
                                       .reshape(v.shape[0], int(rank[r])))
                  for r, v in enumerate(vs)]
        return vs, [sig[r, : int(rank[r])].copy() for r in range(q)], rank

    def compress_chunk(self, basis: "Basis", frames, first: bool = False,
                       strict: bool = False) -> "FrameSeries":
        """Append a chunk of frames and compress it (xg_series_compress_chunk):
        norms, coefficients and planes land at the next series rows; the
        frames are not kept.  ``first`` starts a new series."""
        flags = (_abi.CHUNK_FIRST if first else 0) | (_abi.STRICT if strict else 0)
        if hasattr(frames, "data_ptr"):
            n, on_dev = _tensor_frames(frames, self.ctx, self.layout.full_pixels, None,
                                       "compress_chunk")
            _check(self.ctx.h, lib.xg_series_compress_chunk(
                self.h, basis.h, C.c_void_p(frames.data_ptr()), n, 1 if on_dev else 0, flags))
            self._keep = None if on_dev else frames
        else:
            a = _as_counts_u8(frames)
            if a.ndim != 2 or a.shape[1] != self.layout.full_pixels:
                raise ShapeError(f"frames must be n x {self.layout.full_pixels}, got {a.shape}")
            _check(self.ctx.h, lib.xg_series_compress_chunk(self.h, basis.h, _ptr(a), a.shape[0],
                                                            0, flags))
        self.k = basis.k
        return self

    def ttc_compressed(self, mode: str = "f32", g2: bool = True,
                       store: bool = True, spectral: bool = False) -> "FrameSeries":
        """Homomorphic TTC C~ = Y Y^T of every ring (ttc_compressed,
        correlate.cpp:27-35). mode 'f32' (bf16x3 split, ~1e-6) or 'bf16';
        store=False keeps only g2.  spectral=True (with store=False): g2 from
        the coefficient series' autocorrelations by FFT, in f64, without
        forming any C~ tile (O(k T log T) instead of O(k T^2))."""
        flags = ((_abi.CMP_BF16 if mode == "bf16" else 0) | (0 if g2 else _abi.NO_G2)
                 | (0 if store else _abi.NO_STORE) | (_abi.G2_SPECTRAL if spectral else 0))
        _check(self.ctx.h, lib.xg_ttc_compressed(self.h, flags))
        return self

    def coeffs(self, ring: int):
        n, k = self.n_frames, self.k
        y = np.empty((n, k), np.float64)
        nr = np.empty(n, np.float64)
        _check(self.ctx.h, lib.xg_series_get_coeffs(self.h, ring, y.ctypes.data_as(_abi.PD),
                                                    nr.ctypes.data_as(_abi.PD)))
        return y, nr

    def cttc(self, ring: int, dtype: str = "f64") -> np.ndarray:
        n = self.n_frames
        out = np.empty((n, n), np.float64 if dtype == "f64" else np.float32)
        code = _abi.F64 if dtype == "f64" else _abi.F32
        _check(self.ctx.h, lib.xg_series_get_cttc(self.h, ring, code, _ptr(out), n, 0))
        return out

    def cg2(self, ring: int):
        n = self.n_frames
        vals = np.empty(n, np.float64)
        cnt = np.empty(n, np.int64)
        _check(self.ctx.h, lib.xg_series_get_cg2(self.h, ring, vals.ctypes.data_as(_abi.PD),
                                                 cnt.ctypes.data_as(_abi.PI64)))
        return np.arange(n, dtype=np.float64) * self.frame_period, vals, cnt

    def norms(self, ring: int):
        n = self.n_frames
        out = np.empty(n, np.float64)
        nz = C.c_int64(0)
        _check(self.ctx.h, lib.xg_series_get_norms(self.h, ring, out.ctypes.data_as(_abi.PD),
                                                   C.byref(nz)))
        return out, int(nz.value)


__all__ = [
    "Context", "RingLayout", "FrameSeries", "FrameStream", "Basis", "write_xfsr", "read_xfsr",
    "write_xcmp", "read_xttc", "write_xenc", "read_xenc", "content_hash", "Error", "ShapeError", "ContractError", "MaskError",
    "NormalizationError", "RankError", "BindingError", "FormatError", "DeviceError",
]


# ---------------------------------------------------------------- streaming
class FrameStream:
    """kHz streaming mode: frames pushed one at a time, each correlated
    against the whole history of every ring (raw exact column + optional
    compressed column) -- the device-resident replacement of the reference's
    compress_frame -> ttc_extend -> append loop (acceptance_main.cpp:329-353)."""

    def __init__(self, layout: RingLayout, max_frames: int, basis: "Basis | None" = None,
                 store_ttc: bool = False, raw: bool = True, frame_period: float = 1.0,
                 sparse: bool = False):
        """``sparse``: raw columns from the new frame's nonzero pixels over a
        pixel-major history (nnz * t bytes per frame instead of M * t; same
        results bitwise) -- the photon-event mode for low count rates."""
        self.layout, self.ctx, self.basis = layout, layout.ctx, basis
        self.frame_period = float(frame_period)
        flags = ((_abi.STREAM_STORE_TTC if store_ttc else 0) | (0 if raw else _abi.STREAM_NO_RAW)
                 | (_abi.STREAM_SPARSE if sparse else 0))
        h = C.c_void_p()
        _check(self.ctx.h, lib.xg_stream_create(self.ctx.h, layout.h, basis.h if basis else None,
                                                int(max_frames), flags, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib.xg_stream_destroy(self.h)
            self.h = None

    @property
    def n_frames(self) -> int:
        return int(lib.xg_stream_frames(self.h))

    def append_xcmp(self, ring: int, path, encoder_hash: int, from_frame: int = 0) -> None:
        """Append this ring's compressed rows [from_frame, t) to an XCMP store
        (CompressedFileAppender, io.cpp:368-441; created if missing)."""
        _check(self.ctx.h, lib.xg_stream_append_xcmp(self.h, ring, str(path).encode(),
                                                      int(encoder_hash), int(from_frame)))

    def push(self, frame) -> None:
        if hasattr(frame, "data_ptr"):
            _, on_dev = _tensor_frames(frame, self.ctx, self.layout.full_pixels, 1, "push")
            _check(self.ctx.h, lib.xg_stream_push(self.h, C.c_void_p(frame.data_ptr()),
                                                  1 if on_dev else 0))
            self._keep = None if on_dev else frame
            return
        a = _as_counts_u8(frame).ravel()
        if a.size != self.layout.full_pixels:
            raise ShapeError(f"frame must have {self.layout.full_pixels} pixels, got {a.size}")
        _check(self.ctx.h, lib.xg_stream_push(self.h, _ptr(a), 0))

    def push_many(self, frames) -> None:
        """Push n frames (n x full_pixels) in one library call: the same as n
        push() calls without the per-frame Python round trip."""
        if hasattr(frames, "data_ptr"):
            n, on_dev = _tensor_frames(frames, self.ctx, self.layout.full_pixels, None, "push_many")
            _check(self.ctx.h, lib.xg_stream_push_batch(self.h, C.c_void_p(frames.data_ptr()), n,
                                                        1 if on_dev else 0))
            self._keep = None if on_dev else frames
            return
        a = _as_counts_u8(frames)
        if a.ndim != 2 or a.shape[1] != self.layout.full_pixels:
            raise ShapeError(f"frames must be n x {self.layout.full_pixels}, got {a.shape}")
        _check(self.ctx.h, lib.xg_stream_push_batch(self.h, _ptr(a), a.shape[0], 0))

    def g2(self, ring: int, compressed: bool = False):
        n = self.n_frames
        vals = np.empty(n, np.float64)
        cnt = np.empty(n, np.int64)
        _check(self.ctx.h, lib.xg_stream_get_g2(self.h, ring, 1 if compressed else 0,
                                                vals.ctypes.data_as(_abi.PD),
                                                cnt.ctypes.data_as(_abi.PI64)))
        return np.arange(n, dtype=np.float64) * self.frame_period, vals, cnt

    def coeffs(self, ring: int):
        n, k = self.n_frames, self.basis.k
        y = np.empty((n, k), np.float64)
        nr = np.empty(n, np.float64)
        _check(self.ctx.h, lib.xg_stream_get_coeffs(self.h, ring, y.ctypes.data_as(_abi.PD),
                                                    nr.ctypes.data_as(_abi.PD)))
        return y, nr

    def ttc(self, ring: int, compressed: bool = False, dtype: str = "f64") -> np.ndarray:
        n = self.n_frames
        code = {"f64": _abi.F64, "f32": _abi.F32, "gram": _abi.I32_GRAM}[dtype]
        out = np.empty((n, n), {"f64": np.float64, "f32": np.float32, "gram": np.int32}[dtype])
        _check(self.ctx.h, lib.xg_stream_get_ttc(self.h, ring, 1 if compressed else 0, code,
                                                 _ptr(out), n))
        return out


def frames_to_events(frames):
    """Dense u8 frames (n x pixels, numpy) -> photon-event CSR (frame_off
    int64 [n + 1], pix int32, val uint8): the format event-mode detectors
    deliver (host-side format conversion for tests and benchmarks)."""
    a = np.ascontiguousarray(frames)
    f, p = np.nonzero(a)
    off = np.zeros(a.shape[0] + 1, np.int64)
    np.cumsum(np.bincount(f, minlength=a.shape[0]), out=off[1:])
    return off, p.astype(np.int32), a[f, p].astype(np.uint8)


# --------------------------------------------- reference-facing f64 functions
# One function per xpcs:: operator, same arguments and errors, computed on the
# GPU in the reference's exact floating-point order (k_exact.cu): the results
# are the reference's bits.  A Context (device selection) must exist.
def _f64check(rc: int) -> None:
    if rc == _abi.OK:
        return
    msg = lib.xg_f64_last_error().decode()
    payload = int(lib.xg_f64_last_payload())
    if rc == _abi.ERR_NORMALIZATION:
        raise NormalizationError(msg, payload)
    raise _ERRS.get(rc, DeviceError)(msg or f"status {rc}")


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def ttc_raw(x) -> np.ndarray:
    """xpcs::ttc_raw (correlate.cpp:19-25), bit-exact."""
    x = _d(x)
    n, m = x.shape
    out = np.empty((n, n))
    _f64check(lib.xg_f64_ttc_raw(x.ctypes.data_as(_abi.PD), n, m, out.ctypes.data_as(_abi.PD)))
    return out


def ttc_compressed(y):
    """xpcs::ttc_compressed (correlate.cpp:27-35) -> (G~, lossless), bit-exact."""
    y = _d(y)
    n, k = y.shape
    out = np.empty((n, n))
    ll = C.c_int(0)
    _f64check(lib.xg_f64_ttc_compressed(y.ctypes.data_as(_abi.PD), n, k,
                                        out.ctypes.data_as(_abi.PD), C.byref(ll)))
    return out, bool(ll.value)


def ttc_extend(g, y, row):
    """xpcs::ttc_extend (correlate.cpp:37-65) -> ((n+1)x(n+1), lossless)."""
    g, y, row = _d(g), _d(y), _d(row)
    n = g.shape[0]
    if y.shape[0] != n:
        raise ShapeError(f"ttc_extend: TTC covers {n} frames but store holds {y.shape[0]}")
    if row.size != y.shape[1]:
        raise ShapeError(f"ttc_extend: new row has {row.size} coefficients, store holds "
                         f"k = {y.shape[1]}")
    out = np.empty((n + 1, n + 1))
    ll = C.c_int(0)
    _f64check(lib.xg_f64_ttc_extend(g.ctypes.data_as(_abi.PD), n, y.ctypes.data_as(_abi.PD),
                                    y.shape[1], row.ctypes.data_as(_abi.PD),
                                    out.ctypes.data_as(_abi.PD), C.byref(ll)))
    return out, bool(ll.value)


def g2_from_ttc(g, frame_period: float = 1.0):
    """xpcs::g2_from_ttc (correlate.cpp:67-85) -> (lags, values, counts)."""
    g = _d(g)
    n = g.shape[0]
    lags, vals = np.empty(n), np.empty(n)
    cnt = np.empty(n, np.int64)
    _f64check(lib.xg_f64_g2_from_ttc(g.ctypes.data_as(_abi.PD), n, frame_period,
                                     lags.ctypes.data_as(_abi.PD), vals.ctypes.data_as(_abi.PD),
                                     cnt.ctypes.data_as(_abi.PI64)))
    return lags, vals, cnt


def compress_series(x, v):
    """xpcs::compress_series (compress.cpp:48-81) -> (coefficients, norms)."""
    x, v = _d(x), _d(v)
    n, m = x.shape
    if v.shape[0] != m:
        raise ShapeError(f"frame has {m} pixels, encoder expects {v.shape[0]}")
    k = v.shape[1]
    y, nr = np.empty((n, k)), np.empty(n)
    _f64check(lib.xg_f64_compress_series(x.ctypes.data_as(_abi.PD), n, m,
                                         v.ctypes.data_as(_abi.PD), k, y.ctypes.data_as(_abi.PD),
                                         nr.ctypes.data_as(_abi.PD)))
    return y, nr


def compress_frame(frame, v):
    """xpcs::compress_frame (compress.cpp:34-46) -> (coefficients, norm)."""
    frame, v = _d(frame).ravel(), _d(v)
    if v.shape[0] != frame.size:
        raise ShapeError(f"frame has {frame.size} pixels, encoder expects {v.shape[0]}")
    k = v.shape[1]
    y = np.empty(k)
    nr = C.c_double(0)
    _f64check(lib.xg_f64_compress_frame(frame.ctypes.data_as(_abi.PD), frame.size,
                                        v.ctypes.data_as(_abi.PD), k, y.ctypes.data_as(_abi.PD),
                                        C.byref(nr)))
    return y, nr.value


def ttc_rel_error(g, g_approx) -> float:
    """xpcs::ttc_rel_error (correlate.cpp:87-108)."""
    a, b = _d(g), _d(g_approx)
    if a.shape != b.shape:
        raise ShapeError(f"ttc_rel_error: sizes {a.shape[0]} vs {b.shape[0]}")
    out = C.c_double(0)
    _f64check(lib.xg_f64_ttc_rel_error(a.ctypes.data_as(_abi.PD), b.ctypes.data_as(_abi.PD),
                                       a.size, C.byref(out)))
    return out.value


# ------------------------------------------------------------ geometry / data
def annular_rings(height: int, width: int, n_rings: int) -> np.ndarray:
    """Equal-width annular q-rings: ring(p) =
    min(Q-1, floor(r Q / r_max)), r = distance to the detector centre
    ((W-1)/2, (H-1)/2), r_max = the corner distance.  Returns the ring index
    of every pixel (raster order); masks follow as ``ring == r``."""
    cy, cx = 0.5 * (height - 1), 0.5 * (width - 1)
    rmax = np.sqrt(cx * cx + cy * cy)
    yy, xx = np.meshgrid(np.arange(height, dtype=np.float64),
                         np.arange(width, dtype=np.float64), indexing="ij")
    r = np.sqrt((xx - cx) ** 2 + (yy - cy) ** 2)
    q = np.floor(r * n_rings / rmax).astype(np.int64)
    return np.minimum(q, n_rings - 1).astype(np.int32).ravel()


def synth_speckle(ctx: Context, out_device_ptr: int, n_frames: int, height: int, width: int,
                  n_rings: int, mu: float, seed: int, gamma_mode: int = 0,
                  gamma_a: float = 0.002) -> None:
    """Seeded synthetic speckle counts written straight into device memory
    (benchmark input generator, K8).  Returns once the frames are written:
    K8 runs on the library's stream, and callers read the buffer from torch's."""
    _check(ctx.h, lib.xg_synth_speckle(ctx.h, n_frames, height, width, n_rings, mu, gamma_mode,
                                       gamma_a, seed, C.c_void_p(out_device_ptr)))
    ctx.synchronize()
