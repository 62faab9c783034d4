"""ctypes binding of the ddcca C ABI (include/ddcca.h).

The library is the only compute path: if it is missing or no CUDA device is
present, calls raise — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, DdccanetError, NumericalError, ShapeError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libddcca.so"

OK, ESHAPE, ECONFIG, ENUMERICAL, ECUDA = 0, 1, 2, 3, 4


class DeviceError(DdccanetError):
    """CUDA launch or runtime failure inside the ddcca library."""


class Geom(C.Structure):
    _fields_ = [("p", C.c_int), ("q", C.c_int), ("l1", C.c_int), ("l2", C.c_int),
                ("stride", C.c_int), ("zero_same", C.c_int)]


_vp = C.c_void_p
_i32, _i64, _f64, _sz = C.c_int, C.c_int64, C.c_double, C.c_size_t
_GP = C.POINTER(Geom)

_SIGNATURES = {
    "ddcca_version": (_i32, []),
    "ddcca_last_error": (C.c_char_p, []),
    "ddcca_payload_len": (_i64, [_i32, _i32]),
    "ddcca_moments_workspace": (_sz, [_GP, _i32, _i64, _i32]),
    "ddcca_moments_partial": (_i32, [_vp, _vp, _vp, C.POINTER(_i64), _i32, _GP, _i32, _i32, _vp, _vp, _sz, _vp]),
    "ddcca_moments_partial_ex": (_i32, [_vp, _vp, _vp, C.POINTER(_i64), _i32, _GP, _i32, _i32, _vp, _vp, _sz,
                                        _i32, _vp]),
    "ddcca_moments_tree": (_i32, [_vp, _i32, _i64, _vp, _vp]),
    "ddcca_accumulate_columns": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "ddcca_solve_workspace": (_sz, [_i32]),
    "ddcca_solve": (_i32, [_vp, _i32, _i32, _f64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ddcca_finalize": (_i32, [_vp, _i32, _i32, _f64, _vp, _vp, _vp]),
    "ddcca_sym_eig": (_i32, [_vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ddcca_pack_filters": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "ddcca_conv": (_i32, [_vp, _i64, _GP, _vp, _i32, _i32, _vp, _vp]),
    "ddcca_conv_hash": (_i32, [_vp, _i64, _GP, _vp, _i32, _i32, _vp, _vp]),
    "ddcca_block_hist": (_i32, [_vp, _i32, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i32,
                               _i64, _i64, _i64, _vp]),
    "ddcca_iq_expand": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _vp, _vp]),
    "ddcca_im2col": (_i32, [_vp, _i64, _GP, _i32, _vp, _vp]),
    "ddcca_sign_hash": (_i32, [_vp, _i64, _i32, _i64, _vp, _vp]),
    "ddcca_conv_hw": (_i32, [_vp, _i64, _GP, _vp, _i32, _i32, _vp, _vp]),
    "ddcca_conv_hist_hw": (_i32, [_vp, _i64, _GP, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i64, _i64, _i64, _vp]),
    "ddcca_conv_dev": (_i32, [_vp, _i64, _GP, _vp, _i32, _i32, _vp, _vp]),
    "ddcca_conv_hist_last_path": (_i32, []),
    "ddcca_conv_last_path": (_i32, []),
    "ddcca_conv_hist_dev": (_i32, [_vp, _i64, _GP, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i64, _i64, _i64, _vp]),
    "ddcca_nn_workspace": (_sz, [_i64, _i64]),
    "ddcca_nn_classify": (_i32, [_vp, _i64, _vp, _i64, _i64, _i32, _vp, _i32, _vp, _i32, _vp, _vp, _sz, _vp]),
    "ddcca_counts_to_u16": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp]),
    "ddcca_linear_classify": (_i32, [_vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ddcca_lbp": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp]),
    "ddcca_pgm_info": (_i32, [C.c_char_p, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i64)]),
    "ddcca_pgm_load_many": (_i32, [C.POINTER(C.c_char_p), _i64, _i32, _i32, _vp, _i32]),
    "ddcca_write_feature_csv": (_i32, [_vp, _i32, _i64, _i64, _i32, _i32, C.POINTER(C.c_char_p), C.POINTER(_i32),
                                       _i64, C.c_char_p, _i32]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise DeviceError(
            f"ddcca CUDA library not found at {p}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = load().ddcca_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == ESHAPE:
        raise ShapeError(msg)
    if rc == ECONFIG:
        raise ConfigError(msg)
    if rc == ENUMERICAL:
        raise NumericalError(msg)
    raise DeviceError(msg)


def status_error(code: int, what: str) -> None:
    """Raise the exception matching a device-side status word (0 = ok)."""
    if code == OK:
        return
    if code == ESHAPE:
        raise ShapeError(f"{what}: matrix is not symmetric")
    if code == ENUMERICAL:
        raise NumericalError(
            f"{what}: numerical failure (non-positive-definite input, Jacobi non-convergence "
            "or empty accumulator); is the ridge term missing?"
        )
    if code == ECONFIG:
        raise ConfigError(what)
    raise DeviceError(f"{what}: device status {code}")


def geom(p: int, q: int, l1: int, l2: int, stride: int = 1, padding: str = "zero_same") -> Geom:
    return Geom(int(p), int(q), int(l1), int(l2), int(stride), 1 if padding == "zero_same" else 0)


def ptr(t) -> C.c_void_p:
    """Device (or host) address of a torch tensor; None for None."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream) -> C.c_void_p:
    return C.c_void_p(stream.cuda_stream if stream is not None else 0)
