"""ctypes binding of ``libmgrit_b200.so`` (declared in ``include/mgrit_b200.h``).

The library is the only execution path of this package: there is no CPU or
PyTorch fallback.  If the shared object is missing or no CUDA device is
present, every compute call raises ``RuntimeError`` (loudly, by design).
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

from .errors import DimensionMismatchError, SingularOperatorError

# MGB_LIB selects an experimental build of the same library (tools/build_variant.sh)
_LIB_NAME = os.environ.get("MGB_LIB") or (
    "libmgrit_b200_trace.so" if os.environ.get("MGB_TRACE") else "libmgrit_b200.so")
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", _LIB_NAME)

MGB_OK, MGB_ERR_INVALID, MGB_ERR_DIMENSION, MGB_ERR_SINGULAR, MGB_ERR_CUDA, MGB_ERR_UNSUPPORTED = range(6)
MGB_STEP_STENCIL, MGB_STEP_RK_STAGED, MGB_STEP_SL_DIRECT, MGB_STEP_SL_GMRES = range(4)

_i32, _i64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_pf64, _pi64, _pi32 = ctypes.POINTER(_f64), ctypes.POINTER(_i64), ctypes.POINTER(_i32)


class StepDesc(ctypes.Structure):
    _fields_ = [
        ("kind", _i32), ("n_x", _i32), ("exact", _i32), ("repeat", _i32),
        ("n_taps", _i32), ("offsets", _pi64), ("weights", _pf64),
        ("n_taps2", _i32), ("offsets2", _pi64), ("weights2", _pf64),
        ("stages", _i32), ("implicit", _i32), ("rk_a", _pf64), ("rk_b", _pf64),
        ("gmres_tol", _f64), ("gmres_cap", _i32),
    ]


class RelaxArgs(ctypes.Structure):
    _fields_ = [
        ("n_intervals", _i64), ("k_global0", _i64), ("m", _i32), ("n_fsteps", _i32),
        ("c_src", ctypes.c_void_p), ("c_stride", _i64), ("c_src0", ctypes.c_void_p),
        ("e", ctypes.c_void_p), ("e_stride", _i64),
        ("c_out", ctypes.c_void_p), ("c_out_stride", _i64), ("c_last_out", ctypes.c_void_p),
        ("u", ctypes.c_void_p), ("write_f", _i32),
        ("g", ctypes.c_void_p), ("tail", _i32),
        ("tail_out", ctypes.c_void_p), ("tail_stride", _i64),
        ("cref", ctypes.c_void_p), ("cref_stride", _i64),
        ("cref_e", ctypes.c_void_p), ("cref_e_stride", _i64),
        ("partials", ctypes.c_void_p),
        ("stats_depth", ctypes.c_void_p), ("stats_res", ctypes.c_void_p),
        ("z_out", ctypes.c_void_p), ("z_stride", ctypes.c_int64),
    ]


#: every symbol the header declares (checked by tests/test_native_abi.py)
EXPORTED = ("mgb_step_create", "mgb_step_destroy", "mgb_step_layout",
            "mgb_step_reserve_workspace", "mgb_relax", "mgb_sum", "mgb_version",
            "mgb_last_error", "mgb_launch_count", "mgb_fp64_peak", "mgb_copy_rows")

_lib: Optional[ctypes.CDLL] = None


def lib_path() -> str:
    return _LIB_PATH


def load() -> ctypes.CDLL:
    """Load the shared library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"libmgrit_b200.so not built ({_LIB_PATH}); run "
                           "`python -c 'import __graft_entry__ as g; g.build()'` or `make`")
    lib = ctypes.CDLL(_LIB_PATH)
    lib.mgb_step_create.argtypes = [ctypes.POINTER(StepDesc), ctypes.POINTER(ctypes.c_void_p)]
    lib.mgb_step_create.restype = _i32
    lib.mgb_step_destroy.argtypes = [ctypes.c_void_p]
    lib.mgb_step_destroy.restype = None
    lib.mgb_step_layout.argtypes = [ctypes.c_void_p, _pi32, _pi32, _pi32]
    lib.mgb_step_layout.restype = _i32
    lib.mgb_step_reserve_workspace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.mgb_step_reserve_workspace.restype = _i32
    lib.mgb_relax.argtypes = [ctypes.c_void_p, ctypes.POINTER(RelaxArgs), ctypes.c_void_p]
    lib.mgb_relax.restype = _i32
    lib.mgb_sum.argtypes = [ctypes.c_void_p, _i64, ctypes.c_void_p, ctypes.c_void_p]
    lib.mgb_sum.restype = _i32
    lib.mgb_version.argtypes = []
    lib.mgb_version.restype = _i32
    lib.mgb_last_error.argtypes = []
    lib.mgb_last_error.restype = ctypes.c_char_p
    lib.mgb_launch_count.argtypes = []
    lib.mgb_launch_count.restype = _i64
    lib.mgb_fp64_peak.argtypes = [_i64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
    lib.mgb_fp64_peak.restype = _i32
    lib.mgb_copy_rows.argtypes = [ctypes.c_void_p, _i64, ctypes.c_void_p, _i64, _i64, _i64,
                                  ctypes.c_void_p]
    lib.mgb_copy_rows.restype = _i32
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map an MGB status code to the reference's exception types."""
    if rc == MGB_OK:
        return
    msg = load().mgb_last_error().decode(errors="replace")
    if rc == MGB_ERR_SINGULAR:
        raise SingularOperatorError(msg)
    if rc == MGB_ERR_DIMENSION:
        raise DimensionMismatchError(msg)
    if rc == MGB_ERR_INVALID:
        raise ValueError(msg)
    if rc == MGB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA failure in libmgrit_b200: {msg}")


def launch_count() -> int:
    return int(load().mgb_launch_count())
