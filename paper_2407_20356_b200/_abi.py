"""ctypes binding of the C ABI in include/xpcs_b200.h (libxpcs_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2407_20356_b200/csrc``).  There is no fallback: if the
library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XG_LIB_OVERRIDE") or os.path.join(HERE, "libxpcs_b200.so")  # override: dev A/B probes only
HEADER = os.path.join(os.path.dirname(HERE), "include", "xpcs_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a library first "
        "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback."
    )

lib = C.CDLL(LIB_PATH)

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
U32 = C.c_uint32
PI64 = C.POINTER(C.c_int64)
PI32 = C.POINTER(C.c_int32)
PD = C.POINTER(C.c_double)

_sigs = {
    "xg_version": (C.c_int, []),
    "xg_ctx_create": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "xg_ctx_destroy": (None, [P]),
    "xg_last_error": (C.c_char_p, [P]),
    "xg_last_error_payload": (I64, [P, PI32]),
    "xg_synchronize": (C.c_int, [P]),
    "xg_kernel_launches": (I64, [P]),
    "xg_layout_create": (C.c_int, [P, I64, I32, PI64, PI64, C.POINTER(P)]),
    "xg_layout_create_2d": (C.c_int, [P, I64, I64, I32, PI64, PI64, C.POINTER(P)]),
    "xg_layout_destroy": (None, [P]),
    "xg_layout_ring_pixels": (I64, [P, I32]),
    "xg_series_create": (C.c_int, [P, P, I64, C.POINTER(P)]),
    "xg_series_create2": (C.c_int, [P, P, I64, I64, C.POINTER(P)]),
    "xg_series_destroy": (None, [P]),
    "xg_series_load_frames": (C.c_int, [P, P, I64, C.c_int]),
    "xg_series_load_events": (C.c_int, [P, P, P, P, I64, C.c_int]),
    "xg_series_ttc_raw_events_host": (C.c_int, [P, P, P, P, I64, C.c_uint32]),
    "xg_ttc_raw": (C.c_int, [P, U32]),
    "xg_series_ttc_raw_host": (C.c_int, [P, P, I64, U32]),
    "xg_series_g2": (C.c_int, [P]),
    "xg_series_partial_elems": (I64, [P]),
    "xg_series_export_partial": (C.c_int, [P, I32, P, P, C.c_int]),
    "xg_series_import_partial": (C.c_int, [P, I32, P, P, C.c_int, U32]),
    "xg_series_get_ttc": (C.c_int, [P, I32, I32, P, I64, C.c_int]),
    "xg_series_get_g2": (C.c_int, [P, I32, PD, PI64]),
    "xg_series_get_g2_all": (C.c_int, [P, PD, PI64]),
    "xg_series_g2_device": (C.c_int, [P, I32, C.POINTER(P), C.POINTER(P), PI64]),
    "xg_series_rel_error": (C.c_int, [P, PD]),
    "xg_series_write_xcmp": (C.c_int, [P, I32, C.c_char_p, C.c_uint64, I32]),
    "xg_stream_append_xcmp": (C.c_int, [P, I32, C.c_char_p, C.c_uint64, I64]),
    "xg_series_load_xfsr": (C.c_int, [P, C.c_char_p, PD]),
    "xg_series_write_ttc": (C.c_int, [P, I32, I32, I32, C.c_char_p]),
    "xg_io_last_error": (C.c_char_p, []),
    "xg_io_last_payload": (I64, []),
    "xg_io_write_xcmp": (C.c_int, [C.c_char_p, I64, C.c_uint64, I64, PD, PD, I32]),
    "xg_io_write_xfsr_u8": (C.c_int, [C.c_char_p, P, I64, I64, C.c_double]),
    "xg_io_read_xfsr_u8": (C.c_int, [C.c_char_p, P, I64, PI64, PI64, PD]),
    "xg_io_write_xenc": (C.c_int, [C.c_char_p, I32, I64, I64, PD, I64, PD]),
    "xg_io_read_xenc": (C.c_int, [C.c_char_p, C.POINTER(I32), PI64, PI64, PI64, PD, PD]),
    "xg_series_ttc_background": (C.c_int, [P, I32, I64, PD]),
    "xg_series_fit_kww": (C.c_int, [P, I32, C.c_double, C.c_double, C.c_double, PD, C.POINTER(I32)]),
    "xg_series_build_basis": (C.c_int, [P, I32, C.POINTER(PD), PD, I64, PI64, P]),
    "xg_series_get_norms": (C.c_int, [P, I32, PD, PI64]),
    "xg_series_frames": (I64, [P]),
    "xg_synth_speckle": (C.c_int, [P, I64, I64, I64, I32, C.c_double, I32, C.c_double,
                                   C.c_uint64, P]),
    "xg_build_basis": (C.c_int, [PD, I64, I64, I32, PD, PD, PI64]),
    "xg_content_hash": (C.c_uint64, [PD, I64, I64, I32]),
    "xg_build_basis_batch": (C.c_int, [I32, C.POINTER(PD), I64, PI64, I32, C.POINTER(PD), I32,
                                       PI64]),
    "xg_stream_create": (C.c_int, [P, P, P, I64, U32, C.POINTER(P)]),
    "xg_stream_destroy": (None, [P]),
    "xg_stream_push": (C.c_int, [P, P, C.c_int]),
    "xg_stream_push_batch": (C.c_int, [P, P, I64, C.c_int]),
    "xg_stream_frames": (I64, [P]),
    "xg_stream_get_g2": (C.c_int, [P, I32, I32, PD, PI64]),
    "xg_stream_get_coeffs": (C.c_int, [P, I32, PD, PD]),
    "xg_stream_get_ttc": (C.c_int, [P, I32, I32, I32, P, I64]),
    "xg_f64_last_error": (C.c_char_p, []),
    "xg_f64_last_payload": (I64, []),
    "xg_f64_ttc_raw": (C.c_int, [PD, I64, I64, PD]),
    "xg_f64_ttc_compressed": (C.c_int, [PD, I64, I64, PD, C.POINTER(C.c_int)]),
    "xg_f64_ttc_extend": (C.c_int, [PD, I64, PD, I64, PD, PD, C.POINTER(C.c_int)]),
    "xg_f64_g2_from_ttc": (C.c_int, [PD, I64, C.c_double, PD, PD, PI64]),
    "xg_f64_compress_series": (C.c_int, [PD, I64, I64, PD, I64, PD, PD]),
    "xg_f64_compress_series_u8": (C.c_int, [P, I64, I64, PD, I64, PD, PD]),
    "xg_f64_compress_frame": (C.c_int, [PD, I64, PD, I64, PD, PD]),
    "xg_f64_ttc_rel_error": (C.c_int, [PD, PD, I64, PD]),
    "xg_basis_create": (C.c_int, [P, P, I32, I32, C.POINTER(P)]),
    "xg_basis_destroy": (None, [P]),
    "xg_basis_set_ring": (C.c_int, [P, I32, PD]),
    "xg_compress": (C.c_int, [P, P, U32]),
    "xg_series_compress_chunk": (C.c_int, [P, P, P, I64, C.c_int, U32]),
    "xg_ttc_compressed": (C.c_int, [P, U32]),
    "xg_series_get_coeffs": (C.c_int, [P, I32, PD, PD]),
    "xg_series_get_cttc": (C.c_int, [P, I32, I32, P, I64, C.c_int]),
    "xg_series_get_cg2": (C.c_int, [P, I32, PD, PI64]),
}

for _name, (_res, _args) in _sigs.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def header_symbols(path: str = HEADER) -> list[str]:
    """Every function the public header declares (for the export test)."""
    text = open(path).read()
    return sorted(set(re.findall(r"XG_API\s+[\w\s\*]+?\b(xg_\w+)\s*\(", text)))


# status codes (xg_status)
OK = 0
ERR_SHAPE = 1
ERR_CONTRACT = 2
ERR_MASK = 3
ERR_NORMALIZATION = 4
ERR_RANK = 5
ERR_BINDING = 6
ERR_FORMAT = 7
ERR_CUDA = 100
ERR_DEVICE = 101
ERR_INVALID = 102

F64, F32, I32_GRAM = 0, 1, 2
STRICT = 0x1
NO_G2 = 0x2
CMP_BF16 = 0x4
NO_STORE = 0x8
CHUNK_FIRST = 0x10
G2_SPECTRAL = 0x20
STREAM_STORE_TTC = 0x1
STREAM_NO_RAW = 0x2
STREAM_SPARSE = 0x4
